set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./scripts/micro/l2_peaks > gpurun_out/l2_peaks.json 2> gpurun_out/l2_peaks.err
cat gpurun_out/l2_peaks.json
for w in 24 23 25; do
CC_DEG_WINDOW_LOG2=$w timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4_w$w.json 2> gpurun_out/c4_w$w.err
python -c "
import json;d=json.load(open('gpurun_out/c4_w$w.json'));print($w, d['ms_per_step'], d['stages_ms'], d['kernels']['prediction (k_degree, k_deg_hist)'])"
done
