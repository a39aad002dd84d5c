#!/bin/bash
# Round 2, call b: new parity tests (full-size goldens, bfs+sv, K-S gate, 8 ranks, NCCL-owned
# world 1, failure agreement) and compute-sanitizer memcheck / racecheck / synccheck / initcheck.
TAG=r02b
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_full or gate_ks" > gpurun_out/${TAG}_pytest_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/${TAG}_pytest_parity.log
timeout 900 python -m pytest tests/test_dist_gpu.py -m gpu -x -q > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "dist rc=$?"; tail -3 gpurun_out/${TAG}_pytest_dist.log
for tool in memcheck racecheck synccheck initcheck; do
  Q=""; [ $tool != memcheck ] && Q="--quick"
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python scripts/sanitize_run.py $Q > gpurun_out/${TAG}_san_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/${TAG}_san_$tool.log
done
