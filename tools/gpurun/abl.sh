#!/bin/bash
# ablation variants: time (bench) + LSU breakdown (ncu) for each
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ "$v" = "default" ]; then unset DATABIN_LIB; else export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; fi
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/abl_$v.json 2> gpurun_out/abl_$v.err
  python -c "import json; d=json.load(open('gpurun_out/abl_$v.json')); print('$v', round(d['value']/1e9,1), 'G/s bin', round(d['roofline']['ms_per_launch'],4), d['window'])" 2>&1 | tail -1
  if [ "${NCU:-1}" = "1" ]; then TAG=$v bash tools/gpurun/ncu_lsu.sh > /dev/null; grep -E "lsu_wavefronts.sum|lgds.sum|shared.sum |op_atom.sum|op_ld.sum|op_st.sum|duration|inst_executed.sum " gpurun_out/ncu_lsu_$v.log | awk '{print "   ", $1, $NF}'; fi
done
