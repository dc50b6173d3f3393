#!/bin/bash
# compute-sanitizer over tools/sanitize.py (small inputs, every kernel family)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize.py --quick > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
done
