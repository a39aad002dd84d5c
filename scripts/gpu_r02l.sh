#!/bin/bash
# Round 2, session 5 call l: remainder renumbering (parity + C4 line), C4 / C4-sv kernel timelines,
# C4-sv per-launch DRAM and L2 metrics
TAG=r02l
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "renumber or rmat_bfs or c4_full or config_full or trace_parity" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4.json 2> gpurun_out/${TAG}_c4.err; echo "c4 rc=$?"
timeout 300 python scripts/timeline.py --config c4 --out gpurun_out/${TAG}_tl_c4.json > /dev/null 2>&1; echo "tl c4 rc=$?"
timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv.json > /dev/null 2>&1; echo "tl c4sv rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_red.sum,lts__t_requests_srcunit_tex_op_atom.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
CMD="python bench.py --config c4 --mode sv --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile"
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"k_rowpass|k_long|k_place|k_bucket|k_rows|k_fill|k_pstat|k_collapse|k_compact" -c 60 $CMD > gpurun_out/${TAG}_c4sv_l2.csv 2>/dev/null; echo "ncu rc=$?"
