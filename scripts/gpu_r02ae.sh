#!/bin/bash
# Round 2, session 6 call ae: k_place -- subgroup size adapted to the tuples per id (C4 mode
# sv: 2^7 ids instead of 2^11, so subgroups stage in shared memory) and R of unstaged short
# rows written a warp per row; A/B against CC_SUBG=11; parity
TAG=r02ae
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
for sg in "" 11; do
  CC_SUBG=$sg timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv_$sg.json 2> gpurun_out/${TAG}_c4sv_$sg.err; echo "c4sv $sg rc=$?"
  python scripts/show_bench.py gpurun_out/${TAG}_c4sv_$sg.json | head -2
done
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2> gpurun_out/${TAG}_tl_c4sv.err; echo "tl c4sv rc=$?"
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; echo "$c rc=$?"; python scripts/show_bench.py gpurun_out/${TAG}_$c.json | head -2; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_c4.json | head -2
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
