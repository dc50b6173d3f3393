#!/bin/bash
# DB_LD_STREAM A/B (experiments only): deterministic C3, auto-bounds C3, window route C2, sequential C6 (k_bin general)
export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
b() { timeout 300 python bench.py --workload $1 --steps $2 --warmup 3 --no-e2e --no-cpu-baseline $3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))"; }
for rep in 1 2; do for v in default old; do
  [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so
  echo "$v det $(b c3 20 --deterministic) | bounds-auto $(b c3 100 --bounds-auto) | c6seq $(python tools/multi_bench.py --rows 24000000 --steps 5 --warmup 2 2>&1 | grep -o '"mode": "sequential", "rows": [0-9]*, "ms_per_step": [0-9.]*' | grep -o 'ms_per_step": [0-9.]*')"
done; done
