#!/bin/bash
# partition route A/B (experiments only): tests, then C4 / C2 / C5 bench, current library vs variants/head.so
export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_exact.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for wl in c4 c2 c5; do
  st=100; [ $wl = c4 ] && st=10
  for rep in 1 2; do for v in default head; do
    if [ $v = head ]; then export DATABIN_LIB=paper_2310_02926_b200/variants/head.so; else unset DATABIN_LIB; fi
    timeout 300 python bench.py --workload $wl --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/pab.json')); print('$wl $v', round(d['ms_per_step'],4))"
  done; done
done
unset DATABIN_LIB
DATABIN_PART_TIMING=1 timeout 300 python bench.py --workload c4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -E "part timing"
