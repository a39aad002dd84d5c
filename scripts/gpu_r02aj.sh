#!/bin/bash
# Round 2, session 7 call aj: pass A's relabel gathers used after the tile's first barrier
# (LATE in k_rowpass) -- C2 / C3 / C4-sv / default lines and timelines against call ah's,
# then the full GPU suite on this build
TAG=r02aj
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"; python scripts/show_bench.py gpurun_out/${TAG}_bench_$c.json | sed -n 2,2p; done
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4sv.json 2> gpurun_out/${TAG}_bench_c4sv.err; echo "bench c4sv rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_bench_c4sv.json | sed -n 2,2p
timeout 300 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_bench_default.json | sed -n 2,2p
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > gpurun_out/${TAG}_tl_c4sv.log 2>&1; echo "tl c4sv rc=$?"
sed -n 2,12p gpurun_out/${TAG}_tl_c4sv.log
timeout 600 python scripts/timeline.py --config c2 --out gpurun_out/${TAG}_tl_c2.json > gpurun_out/${TAG}_tl_c2.log 2>&1; echo "tl c2 rc=$?"
sed -n 2,6p gpurun_out/${TAG}_tl_c2.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
