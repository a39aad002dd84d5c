#!/bin/bash
# C4 prediction time vs degree-counter window (experiment)
for w in 22 23 24 25 26; do
  CC_DEG_WINDOW_LOG2=$w timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/degw_$w.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/degw_$w.json').read().strip().splitlines()[-1]);print($w, d['stages_ms'], d['ms_per_step'])"
done
