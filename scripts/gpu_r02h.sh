#!/bin/bash
# Round 2, session 3 call h: fire-and-forget BFS claims; C4 A/B (spec, hub), ncu of level 2 both ways, GPU suite
TAG=r02h
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_c4_both.json 2> gpurun_out/${TAG}_c4_both.err; echo "bench both rc=$?"
CC_SPEC_MIN_EDGES=1000000000000 timeout 600 $B > gpurun_out/${TAG}_c4_nospec.json 2>/dev/null; echo "bench nospec rc=$?"
CC_BFS_HUB=0 timeout 600 $B > gpurun_out/${TAG}_c4_nohub.json 2>/dev/null; echo "bench nohub rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_deg_part|k_bfs_level" -s 0 -c 4 -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
CC_BFS_HUB=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level" -s 1 -c 1 -o gpurun_out/${TAG}_prof_nohub -f $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
