CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_deg_part" -s 1 -c 1 -o gpurun_out/prof_deg2 -f $CMD > gpurun_out/ncu1.log 2>&1
tail -n 3 gpurun_out/ncu1.log
