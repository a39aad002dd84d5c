# ncu --set full of the C4 prediction and BFS kernels (one launch each); read with ncu -i here
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_deg_part|k_deg_count" -s 2 -c 2 -o gpurun_out/prof_deg -f $CMD > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level" -s 6 -c 2 -o gpurun_out/prof_bfs -f $CMD > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
