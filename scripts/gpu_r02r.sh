#!/bin/bash
# Round 2, session 5 call r: block-wide decoupled look-back (collapse / compact / CSR offsets /
# relabel rank), k_bucket at 4 blocks/SM -- C2, C3, C4, C5/16 lines; parity subset; collapse ncu
TAG=r02r
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
for c in c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; echo "$c rc=$?"
done
timeout 300 python scripts/timeline.py --config c2 --out gpurun_out/${TAG}_tl_c2.json > /dev/null 2>&1; echo "tl c2 rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_degree.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_collapse|k_bucket" -c 2 -o gpurun_out/${TAG}_c2_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
python profiles/srclines.py gpurun_out/${TAG}_c2_full.ncu-rep k_collapse 20 > gpurun_out/${TAG}_collapse_src.txt 2>&1
