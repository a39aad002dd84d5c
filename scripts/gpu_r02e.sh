#!/bin/bash
# Round 2, session 3 call e: HEAD check (smoke, GPU suite, C4 + C2 bench lines)
TAG=r02e
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --config c4 --mode sv --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4sv.json 2> gpurun_out/${TAG}_bench_c4sv.err; echo "bench c4sv rc=$?"
