timeout 900 python -m pytest tests/test_gpu_degree.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gate or degree or c4_full or rmat" 2>&1 | tail -5
python scripts/timeline.py --config c4 --out gpurun_out/tl_c4.json 2>&1 | grep -v Warn | head -16
