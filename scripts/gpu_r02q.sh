#!/bin/bash
# Round 2, session 5 call q: ncu full set (with source) of C4's degree pass and BFS level 2
TAG=r02q
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/${TAG}_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_deg_part|k_deg_count" -c 2 -o gpurun_out/${TAG}_deg $CMD > gpurun_out/${TAG}_ncu_deg.log 2>&1; echo "ncu deg rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_bfs_level" -s 2 -c 1 -o gpurun_out/${TAG}_bfs $CMD > gpurun_out/${TAG}_ncu_bfs.log 2>&1; echo "ncu bfs rc=$?"
for r in deg bfs; do
  ncu -i gpurun_out/${TAG}_$r.ncu-rep --page details --csv > gpurun_out/${TAG}_${r}_details.csv 2>/dev/null
done
python profiles/stalls.py gpurun_out/${TAG}_deg.ncu-rep k_deg_part 0 30 > gpurun_out/${TAG}_deg_stalls.txt 2>&1
python profiles/srclines.py gpurun_out/${TAG}_deg.ncu-rep k_deg_part 30 > gpurun_out/${TAG}_deg_src.txt 2>&1
python profiles/stalls.py gpurun_out/${TAG}_bfs.ncu-rep k_bfs_level 0 30 > gpurun_out/${TAG}_bfs_stalls.txt 2>&1
