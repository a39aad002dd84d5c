timeout 900 python -m pytest tests/test_gpu_degree.py -x -q 2>&1 | tail -3
python scripts/timeline.py --config c4 --op degrees --out gpurun_out/tl_c4d.json 2>&1 | grep -v Warn | head -6
