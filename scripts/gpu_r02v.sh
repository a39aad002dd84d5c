#!/bin/bash
# Round 2, session 5 call v: group and subgroup bucketing staged in shared memory (coalesced runs)
TAG=r02v
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; echo "$c rc=$?"; done
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2>&1; echo "tl rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "config or trace or collapse or straddle or ragged or c4 or u64 or csr" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q -k "c1 or exchange or balanced" > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
tail -2 gpurun_out/${TAG}_pytest_dist.log
