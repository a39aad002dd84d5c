#!/bin/bash
# Round 2, session 3 call i: hub cache v2 (2^15 tags, 2 blocks/SM, branch-free loads), edge-partitioned
# multi-rank BFS; C4 A/B, ncu of level 2, dist + spec + parity tests
TAG=r02i
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_c4_hub.json 2> gpurun_out/${TAG}_c4_hub.err; echo "bench hub rc=$?"
CC_BFS_HUB=0 timeout 600 $B > gpurun_out/${TAG}_c4_nohub.json 2>/dev/null; echo "bench nohub rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level_hub" -s 0 -c 1 -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "rmat or c4 or gate or hand or exhaustive or config" > gpurun_out/${TAG}_pytest2.log 2>&1; echo "pytest2 rc=$?"
tail -3 gpurun_out/${TAG}_pytest2.log
