#!/bin/bash
# Round 2, session 5 call s: fused BFS level epilogue + deg_order + collapse HW red; parity of the
# BFS / spec / degree paths; traffic.json regenerated (c2, c3, c4, c4 mode sv); the default
# bench line as the driver runs it; ncu launch list of that command
TAG=r02s
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_degree.py -x -q -k "bfs or spec or c4 or rmat or renumber or config or degree or collapse or ecc" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
for c in c2 c3 c4; do timeout 900 python scripts/traffic.py --config $c > gpurun_out/${TAG}_traffic_$c.log 2>&1; echo "traffic $c rc=$?"; done
timeout 1500 python scripts/traffic.py --config c4 --mode sv > gpurun_out/${TAG}_traffic_c4sv.log 2>&1; echo "traffic c4sv rc=$?"
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
timeout 300 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4sv.json 2> gpurun_out/${TAG}_bench_c4sv.err; echo "bench c4sv rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c4.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
