#!/bin/bash
# Round 2, session 6 call ac: degree pass with predicated ring stores on full rounds (default)
# against the branched insert (CC_DEG_LEGACY=1): degree/spec parity, C4 and C2 lines, twice each
TAG=r02ac
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_degree.py tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for lg in 0 1; do
    CC_DEG_LEGACY=$lg timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4_l${lg}_$rep.json 2> gpurun_out/${TAG}_c4_l${lg}_$rep.err; echo "c4 l$lg rc=$?"
    python -c "
import json;d=json.load(open('gpurun_out/${TAG}_c4_l${lg}_$rep.json'));print('c4 legacy=$lg', d['ms_per_step'], d.get('stages_ms'))"
  done
done
CC_DEG_LEGACY=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c4 or gate or degree" > gpurun_out/${TAG}_pytest2.log 2>&1; echo "pytest2 rc=$?"
tail -2 gpurun_out/${TAG}_pytest2.log
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err; echo "c2 rc=$?"
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2> gpurun_out/${TAG}_tl_c4sv.err; echo "tl c4sv rc=$?"
timeout 300 python scripts/timeline.py --config c4 --out gpurun_out/${TAG}_tl_c4.json > /dev/null 2>&1; echo "tl c4 rc=$?"
