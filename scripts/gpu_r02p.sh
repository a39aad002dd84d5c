#!/bin/bash
# Round 2, session 5 call p: collapse scheduled from iteration 0 (C4 mode sv), C3 / C5 lines,
# ncu full sets of C2's collapse and CSR bucket kernels
TAG=r02p
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c3.json 2> gpurun_out/${TAG}_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err; echo "c5 rc=$?"
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_collapse|k_bucket|k_place" -c 4 -o gpurun_out/${TAG}_c2_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_c2_full.ncu-rep --page details --csv > gpurun_out/${TAG}_c2_full_details.csv 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "collapse or config or trace or c4" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
