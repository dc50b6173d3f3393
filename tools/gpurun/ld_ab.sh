#!/bin/bash
# load cache-hint A/B (experiments only): C3 (k_bin_fast), C4/C2/C5 (partition reduce), C6 (multi)
export DATABIN_NO_BUILD=1
b() { timeout 300 python bench.py --workload $1 --steps $2 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['ms_per_launch'],4))"; }
for rep in 1 2; do
  for v in default fcg; do [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; echo "c3 $v $(b c3 100)"; done
  for v in default rcg; do [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; echo "c4 $v $(b c4 10) | c2 $(b c2 100) | c5 $(b c5 100)"; done
  for v in default mcg; do [ $v = default ] && unset DATABIN_LIB || export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; echo "c6 $v $(python tools/multi_bench.py --rows 1000000,24000000 --steps 10 --warmup 3 2>&1 | grep -o '"mode": "fused", "rows": [0-9]*, "ms_per_step": [0-9.]*' | grep -o 'ms_per_step": [0-9.]*' | tr '\n' ' ')"; done
done
