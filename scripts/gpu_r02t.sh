#!/bin/bash
# Round 2, session 5 call t: ncu full set (with source) of the CSR build kernels on C4 mode sv
TAG=r02t
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
CMD="python bench.py --config c4 --mode sv --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_bucket|k_place" -c 3 -o gpurun_out/${TAG}_csr $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/${TAG}_csr.ncu-rep --page details --csv > gpurun_out/${TAG}_csr_details.csv 2>/dev/null
for k in "k_bucket<" k_bucket2 k_place; do
  python profiles/srclines.py gpurun_out/${TAG}_csr.ncu-rep "$k" 25 > "gpurun_out/${TAG}_src_${k//</}.txt" 2>&1
done
