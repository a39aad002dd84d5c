#!/bin/bash
# Round 2, session 3 call j: hot-variant selection on the current iteration's slot targets (CC_HOT_SEL)
# C4 mode=sv and C2 A/B; L2 metrics of the C4 sv row passes
TAG=r02j
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_dist_gpu.py tests/test_gpu_spec.py -x -q > gpurun_out/${TAG}_pytest_dist.log 2>&1; echo "pytest dist rc=$?"
tail -3 gpurun_out/${TAG}_pytest_dist.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2>/dev/null; echo "c4 rc=$?"
for sel in 0 1; do
  CC_HOT_SEL=$sel timeout 900 python bench.py --config c4 --mode sv --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4sv_sel$sel.json 2>/dev/null; echo "c4sv sel=$sel rc=$?"
  CC_HOT_SEL=$sel timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2_sel$sel.json 2>/dev/null; echo "c2 sel=$sel rc=$?"
done
for ab in "8 6" "10 8" "9 5"; do
  set -- $ab
  CC_HOT_SEL=1 CC_HOT_A=$1 CC_HOT_B=$2 timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c2_sel1_$1_$2.json 2>/dev/null; echo "c2 $1 $2 rc=$?"
done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
CMD="python bench.py --config c4 --mode sv --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
for sel in 0 1; do
  CC_HOT_SEL=$sel timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"k_rowpass|k_pstat|k_long|k_collapse" -c 24 $CMD > gpurun_out/${TAG}_c4sv_l2_sel$sel.csv 2>/dev/null; echo "ncu sel=$sel rc=$?"
done
CC_HOT_SEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config or trace or regression or collapse" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv $CMD > gpurun_out/${TAG}_c4sv_launches.csv 2>/dev/null; echo "ncu launches rc=$?"
