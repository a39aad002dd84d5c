#!/bin/bash
# Round 2, session 3 call g: spec-root + hub-cache tests, C4 bench with each ablation, ncu of deg_part / hub level
TAG=r02g
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_c4_both.json 2> gpurun_out/${TAG}_c4_both.err; echo "bench both rc=$?"
CC_SPEC_MIN_EDGES=1000000000000 timeout 600 $B > gpurun_out/${TAG}_c4_nospec.json 2>/dev/null; echo "bench nospec rc=$?"
CC_BFS_HUB=0 timeout 600 $B > gpurun_out/${TAG}_c4_nohub.json 2>/dev/null; echo "bench nohub rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_deg_part|k_bfs_level|k_deg_sample" -s 0 -c 5 -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
CC_SPEC_MIN_EDGES=1000000000000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_deg_part" -s 0 -c 1 -o gpurun_out/${TAG}_prof_nospec -f $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2 rc=$?"
