#!/bin/bash
# TMA-staged partition refine A/B (experiments only)
export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_gpu_exact.py -q -x -p no:cacheprovider 2>&1 | tail -1
b() { timeout 300 python bench.py --workload $1 --steps $2 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))"; }
for rep in 1 2; do for v in default head; do
  [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so
  echo "$v c4 $(b c4 10) c5 $(b c5 100) c2 $(b c2 100)"
done; done
for v in default head; do
  [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so
  echo "$v $(DATABIN_PART_TIMING=1 timeout 300 python bench.py --workload c4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -E 'part timing' | cut -c30-)"
done
