#!/bin/bash
# Round 2, session 5 call x: 256-bit group stores in the degree pass (C4); ncu of C2's collapse
TAG=r02x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4b.json 2> gpurun_out/${TAG}_c4b.err; echo "c4b rc=$?"
timeout 600 python -m pytest tests/test_gpu_degree.py tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_collapse" -c 1 -o gpurun_out/${TAG}_collapse $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_deg_part" -c 1 -o gpurun_out/${TAG}_degpart python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2 rc=$?"
