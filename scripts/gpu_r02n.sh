#!/bin/bash
# Round 2, session 5 call n: collapse after iteration 1, min_visited / fused BFS labels / vectorised
# root count; C4, C4-sv, C2 lines, C2 + C4 timelines; GPU parity subset
TAG=r02n
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv.json 2> gpurun_out/${TAG}_c4sv.err; echo "c4sv rc=$?"
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 300 python scripts/timeline.py --config c2 --out gpurun_out/${TAG}_tl_c2.json > /dev/null 2>&1; echo "tl c2 rc=$?"
timeout 300 python scripts/timeline.py --config c4 --out gpurun_out/${TAG}_tl_c4.json > /dev/null 2>&1; echo "tl c4 rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
