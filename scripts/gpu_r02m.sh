#!/bin/bash
# Round 2, session 5 call m: iteration-0 hot selection by distinct targets (C4 mode sv, C2, C4),
# balanced variant (gloo dist tests), renumbering; parity subset
TAG=r02m
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 1200 python -m pytest tests/test_dist_gpu.py -x -q -k "balanced or c1 or exclusion" > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
tail -3 gpurun_out/${TAG}_pytest_dist.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2>&1; echo "tl c4sv rc=$?"
