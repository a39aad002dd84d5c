#!/bin/bash
# Round 2, call d: ncu --set full of the collapse kernel (C2) and of C4 mode=sv row pass B (iteration 0)
TAG=r02d
mkdir -p gpurun_out
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_collapse" -s 3 -c 1 -o gpurun_out/${TAG}_collapse -f $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:k_rowpass" -s 84 -c 12 -o gpurun_out/${TAG}_rowpass_c2 -f $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2 rc=$?"
CMD4="python bench.py --config c4 --mode sv --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-profile"
ncu --set full --clock-control none --import-source on -k "regex:k_rowpass" -s 36 -c 2 -o gpurun_out/${TAG}_rowpass_c4sv -f $CMD4 > gpurun_out/${TAG}_ncu3.log 2>&1; echo "ncu3 rc=$?"
