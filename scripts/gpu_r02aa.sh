#!/bin/bash
# Round 2, session 5 call aa: iteration 0's pass A by pull -- parity (pull vs push vs oracle,
# full parity file), C2 / C3 / C4-sv / C4 lines with and without (CC_PULL0=0)
TAG=r02aa
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
for p0 in 1 0; do
  for c in c2 c3; do CC_PULL0=$p0 timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${c}_p$p0.json 2> gpurun_out/${TAG}_${c}_p$p0.err; echo "$c p$p0 rc=$?"; done
  CC_PULL0=$p0 timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv_p$p0.json 2> gpurun_out/${TAG}_c4sv_p$p0.err; echo "c4sv p$p0 rc=$?"
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 300 python scripts/timeline.py --config c2 --out gpurun_out/${TAG}_tl_c2.json > /dev/null 2>&1; echo "tl rc=$?"
