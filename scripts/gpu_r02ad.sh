#!/bin/bash
# Round 2, session 6 call ad: long-row segment kernels with LU = 8 loads in flight per lane,
# k_pull0 with four gathers in flight, vectorised k_longlist -- parity (full parity file),
# C4 mode sv / C4 / C2 lines, C4-sv timeline
TAG=r02ad
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_c4sv.json
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2> gpurun_out/${TAG}_tl_c4sv.err; echo "tl c4sv rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_c4.json
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_c2.json
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_degree.py tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
