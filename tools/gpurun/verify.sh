#!/bin/bash
# Round-start verification: GPU tests, smoke, bench, then sanitizers on small inputs.
mkdir -p gpurun_out
export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/bench.json
if [ "$1" = "san" ]; then bash tools/gpurun/sanitize.sh; cat gpurun_out/sanitize_summary.txt; fi
