#!/bin/bash
# finalize skips the loads of empty bins: A/B (experiments only)
export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests/test_multi.py tests/test_gpu_parity.py tests/test_gpu_group.py -q -x -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for v in default head; do
  [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so
  echo "$v c6 $(python tools/multi_bench.py --rows 46875,1000000 --steps 50 --warmup 5 2>&1 | grep -o '"mode": "fused", "rows": [0-9]*, "ms_per_step": [0-9.]*' | grep -o 'ms_per_step": [0-9.]*' | tr '\n' ' ') c3 $(timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))")"
done; done
