#!/bin/bash
# Quick iteration on the GPU box: csr parity tests, a C2 bench line, optional ncu capture.
# usage: bash scripts/gpu_iter.sh <tag> [ncu-kernel-regex]
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${PYK:-csr}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2>gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -2 gpurun_out/${TAG}_bench.err
if [ -n "$2" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
  $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$2" -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-2} \
    -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
fi
