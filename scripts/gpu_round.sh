#!/bin/bash
# One gpurun call: GPU parity tests, bench lines, ncu launch list + one --set full capture.
# usage (from the repo root on the GPU box): bash scripts/gpu_round.sh <tag> [pytest-args]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
nproc >> gpurun_out/${TAG}_gpu.txt; lscpu | grep "Model name" >> gpurun_out/${TAG}_gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for c in ${BENCH_CONFIGS:-c2 c4 c5}; do
  timeout 600 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
CMD="python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${NCU_KERNELS:-k_rowpass|k_pstat1|k_place|k_bucket2}" -s ${NCU_SKIP:-60} -c ${NCU_COUNT:-8} \
  -o gpurun_out/${TAG}_full_c2 $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
# kernel timelines (CUPTI), DRAM traffic per row-pass launch, L2 request rates
python scripts/timeline.py --out gpurun_out/${TAG}_tl_c2.json > /dev/null 2>&1
python scripts/timeline.py --config c4 --out gpurun_out/${TAG}_tl_c4.json > /dev/null 2>&1
python scripts/traffic.py > gpurun_out/${TAG}_traffic.log 2>&1; cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,lts__t_requests_op_red_lookup_hit.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_read.sum,lts__t_sectors_op_read.sum"
ncu --metrics $M --clock-control none --csv -k 'regex:k_rowpass' -s 84 -c 28 python scripts/timeline.py --out gpurun_out/l2x.json > gpurun_out/${TAG}_l2_c2.csv 2>/dev/null
echo "extras done"
