#!/bin/bash
# Round 2, call c: row collapse -- parity (forced collapse, the csr engine's traces), benches.
TAG=r02c
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "collapse" > gpurun_out/${TAG}_pytest_collapse.log 2>&1; echo "collapse rc=$?"; tail -15 gpurun_out/${TAG}_pytest_collapse.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_pytest_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/${TAG}_pytest_parity.log
for c in c2 c3 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --config c4 --mode sv --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4sv.json 2> gpurun_out/${TAG}_bench_c4sv.err; echo "bench c4 sv rc=$?"
