#!/bin/bash
# Round 2, session 5 call y: 256-bit edge loads in the degree pass and the BFS level (4 edges
# per thread step)
TAG=r02y
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4_$i.json 2> gpurun_out/${TAG}_c4_$i.err; echo "c4 rc=$?"; done
timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
timeout 1200 python -m pytest tests/test_gpu_degree.py tests/test_gpu_spec.py tests/test_gpu_parity.py -x -q -k "not radix and not u64_relabel" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q -k "bfs or c1 or degree" > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
tail -2 gpurun_out/${TAG}_pytest_dist.log
