#!/bin/bash
# Round 2, session 5 call o: owner-computes slot exchange (NEXT-1) -- all dist tests (gloo, ranks
# sharing cuda:0); sort microbenchmark at the paper's 2e9 keys (NEXT-3)
TAG=r02o
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
tail -5 gpurun_out/${TAG}_pytest_dist.log
timeout 900 python scripts/sort_bench.py --n 2000000000 --reps 2 > gpurun_out/${TAG}_sort_2e9.json 2> gpurun_out/${TAG}_sort_2e9.err; echo "sort rc=$?"
tail -2 gpurun_out/${TAG}_sort_2e9.err
