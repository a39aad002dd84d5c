#!/bin/bash
# Round 2, session 7 call ai: ncu --set full of the C4 mode-sv row passes after iteration 0
# (evidence for the next step): iteration 1's pass A (k_rowpass<true,false,true,true>, launch
# 3 of a run's 14 row-pass launches) and iteration 2's pass A (the hot variant, launch 6);
# one warm-up run first (14 launches)
TAG=r02ai
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
CMD="python scripts/pullw_ab.py --windows 24 --reps 1 --out gpurun_out/${TAG}_ab.json"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rowpass -s 17 -c 1 -o gpurun_out/${TAG}_rowpassA1 -f $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu A1 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rowpass -s 20 -c 1 -o gpurun_out/${TAG}_rowpassA2 -f $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu A2 rc=$?"
tail -2 gpurun_out/${TAG}_ncu1.log gpurun_out/${TAG}_ncu2.log
