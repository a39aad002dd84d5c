#!/bin/bash
# Round 2, session 7 call ak: does the windowed pull change iteration 1's pass A?  Two C4 mode-sv
# timelines on one box, CC_PULLW=0 against the default, same build
TAG=r02ak
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
for w in 0 24 0 24; do
  CC_PULLW=$w timeout 600 python scripts/timeline.py --config c4 --mode sv --out gpurun_out/${TAG}_tl_c4sv_w$w.json > gpurun_out/${TAG}_tl_w$w.log 2>&1; echo "tl w=$w rc=$?"
  grep -E "span_us|k_rowpass|k_pull0" gpurun_out/${TAG}_tl_w$w.log | cut -c1-110
done
