# A/B of build variants on the bench workload (kernel-level numbers only)
export DATABIN_NO_BUILD=1
for v in default $VARIANTS; do
  if [ "$v" = "default" ]; then unset DATABIN_LIB; else export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; fi
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value']/1e9,1), 'G/s step', round(d['ms_per_step'],4), 'bin', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), d['window'])" 2>&1 | tail -1
done
