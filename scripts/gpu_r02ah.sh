#!/bin/bash
# Round 2, session 7 call ah: final HEAD verification (pull windows, tile skip, cc_approx_diameter, NVTX)
# default -- smoke, full GPU suite, traffic.json regenerated, the default bench line as the
# driver runs it, C2 / C3 / C4-sv lines, reference arm, C4 ncu launch list
TAG=r02ah
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
# traffic.json first, so the bench lines below read this build's DRAM bytes
for c in c2 c3 c4; do timeout 900 python scripts/traffic.py --config $c > gpurun_out/${TAG}_traffic_$c.log 2>&1; echo "traffic $c rc=$?"; done
timeout 1500 python scripts/traffic.py --config c4 --mode sv > gpurun_out/${TAG}_traffic_c4sv.log 2>&1; echo "traffic c4sv rc=$?"
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
timeout 300 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
for c in c2 c3; do timeout 300 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"; done
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4sv.json 2> gpurun_out/${TAG}_bench_c4sv.err; echo "bench c4sv rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "bench ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c4.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
