#!/bin/bash
# Round 2, session 3 call f: speculative root level (tests + C4 bench), ncu of BFS level 2 and deg_part
TAG=r02f
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_spec.py tests/test_gpu_degree.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rmat or c4 or gate" > gpurun_out/${TAG}_pytest2.log 2>&1; echo "pytest2 rc=$?"
tail -3 gpurun_out/${TAG}_pytest2.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err; echo "bench c4 rc=$?"
CMD="python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level|k_deg_part" -s 4 -c 3 -o gpurun_out/${TAG}_prof -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
