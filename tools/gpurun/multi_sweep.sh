#!/bin/bash
# C6 fused multi-operator (experiments only): previous library vs current + the tests
export DATABIN_NO_BUILD=1
for rep in 1 2; do
for lib in paper_2310_02926_b200/variants/head.so paper_2310_02926_b200/libdatabin.so; do
  echo "$lib $(DATABIN_LIB=$lib python tools/multi_bench.py --rows 46875,262144,524288,1000000,24000000 --steps 20 --warmup 3 2>&1 | grep -o "\"mode\": \"fused\", \"rows\": [0-9]*, \"ms_per_step\": [0-9.]*" | grep -o "ms_per_step\": [0-9.]*" | tr "\n" " ")"
done; done
python -m pytest tests/test_multi.py -x -q 2>&1 | tail -1
DATABIN_MULTI_FILTER_RPB=0 python -m pytest tests/test_multi.py -x -q 2>&1 | tail -1
python tools/multi_bench.py --steps 20 --warmup 3 > gpurun_out/multi_final3.txt 2>&1
