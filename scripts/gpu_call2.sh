set -x
timeout 900 python -m pytest tests/test_gpu_degree.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4_radix.json 2> gpurun_out/c4_radix.err
python -c "
import json;d=json.load(open('gpurun_out/c4_radix.json'));print(d['ms_per_step'], d['stages_ms'], d['kernels']['prediction (k_degree, k_deg_hist)'])"
tail -5 gpurun_out/c4_radix.err
