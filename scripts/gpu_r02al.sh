#!/bin/bash
# Round 2, session 7 call al: last check of the committed HEAD (comment-only changes since call
# aj's build): build + smoke, the pull / eccentricity parity tests, the default bench line
TAG=r02al
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -x -q -k "pull or eccentricity or abi or c1" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
python scripts/show_bench.py gpurun_out/${TAG}_bench_default.json | sed -n 2,5p | cut -c1-150
