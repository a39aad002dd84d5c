timeout 900 python -m pytest tests/test_gpu_degree.py -x -q 2>&1 | tail -3
bash scripts/gpu_ncu_deg.sh
