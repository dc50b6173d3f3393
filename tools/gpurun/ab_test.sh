#!/bin/bash
# parity subset of the default build, then A/B of the variants on the bench workload(s)
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${TESTS} > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/ab_tests.log
for wl in ${WLS:-c3}; do
for v in default $VARIANTS; do
  if [ "$v" = "default" ]; then unset DATABIN_LIB; else export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; fi
  for rep in 1 2; do
  timeout 300 python bench.py --workload $wl --steps 100 --warmup 5 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab_${wl}_$v.json 2> gpurun_out/ab_${wl}_$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_${wl}_$v.json')); print('$wl $v', round(d['value']/1e9,1), 'G/s step', round(d['ms_per_step'],4), 'bin', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), d['window'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
done
