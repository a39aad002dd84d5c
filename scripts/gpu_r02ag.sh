#!/bin/bash
# Round 2, session 7 call ag: iteration 0's pull by id windows of U (CC_PULLW) -- parity of the
# windowed pull, A/B of the window size on C4 mode sv in one process, timeline, bench lines,
# one ncu --set full capture of iteration 0's pass B (k_rowpass<false,true,true,true>)
TAG=r02ag
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pull" > gpurun_out/${TAG}_pytest_pull.log 2>&1; echo "pytest pull rc=$?"
tail -2 gpurun_out/${TAG}_pytest_pull.log
timeout 1500 python scripts/pullw_ab.py --windows 0,24,23,25,22,0,24 --envs "CC_HOT_A=31;CC_HOT_A=12;CC_HOT_B=31;CC_HOT_B=10;CC_HOT_B=4" --out gpurun_out/${TAG}_pullw_ab.json > gpurun_out/${TAG}_pullw_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/${TAG}_pullw_ab.log | tail -8
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > gpurun_out/${TAG}_tl_c4sv.log 2> gpurun_out/${TAG}_tl_c4sv.err; echo "tl c4sv rc=$?"
head -12 gpurun_out/${TAG}_tl_c4sv.log
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_c4sv.json | head -2
CMD="python scripts/pullw_ab.py --windows 24 --reps 1 --out gpurun_out/${TAG}_ncu_ab.json"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_rowpass -s 14 -c 1 -o gpurun_out/${TAG}_rowpassB0 -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log
# the build as the driver will see it: default line, C2 / C3 lines, C4 launch list, full GPU suite
timeout 300 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_bench_default.json | head -4
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"; python scripts/show_bench.py gpurun_out/${TAG}_bench_$c.json | head -2; done
timeout 600 python scripts/timeline.py --config c2 --out gpurun_out/${TAG}_tl_c2.json > gpurun_out/${TAG}_tl_c2.log 2>&1; echo "tl c2 rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for c in c2 c3 c4; do timeout 900 python scripts/traffic.py --config $c > gpurun_out/${TAG}_traffic_$c.log 2>&1; echo "traffic $c rc=$?"; done
timeout 1500 python scripts/traffic.py --config c4 --mode sv > gpurun_out/${TAG}_traffic_c4sv.log 2>&1; echo "traffic c4sv rc=$?"
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
