#!/bin/bash
# k_part_keys load-cache-hint A/B on C4 (experiments only): in-pipeline kernel times + DRAM bytes of one launch
export DATABIN_NO_BUILD=1
for v in default kldcg kldg kldlu; do
  if [ $v = default ]; then unset DATABIN_LIB; else export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; fi
  echo "$v $(DATABIN_PART_TIMING=1 timeout 300 python bench.py --workload c4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | grep -E 'part timing' | cut -c30-)"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:k_part_keys -s 2 -c 1 python bench.py --workload c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "duration|bytes|sectors"
done
