#!/bin/bash
# C6 fused multi-operator (experiments only): final numbers + tests
export DATABIN_NO_BUILD=1
python -m pytest tests/test_multi.py -x -q 2>&1 | tail -1
python tools/multi_bench.py --rows 46875,131072,262144,1000000,24000000 --steps 20 --warmup 3 > gpurun_out/multi_final4.txt 2>&1
grep -o "\"mode\": \"[a-z]*\", \"rows\": [0-9]*, \"ms_per_step\": [0-9.]*, \"rows_per_s\": [0-9.e+]*, \"bin_updates_per_s\": [0-9.e+]*, \"launches_per_step\": [0-9.]*" gpurun_out/multi_final4.txt
