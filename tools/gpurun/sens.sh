#!/bin/bash
# sensitivity of the C3 bin kernel to the requested ops and a loads-only build
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
run() {  # tag, extra env/args
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $2 > gpurun_out/sens_$1.json 2> gpurun_out/sens_$1.err
  python -c "import json; d=json.load(open('gpurun_out/sens_$1.json')); print('$1', round(d['value']/1e9,1), 'G/s bin', round(d['roofline']['ms_per_launch'],4), d['roofline']['kernel'], d['window'])" 2>&1 | tail -1
}
run full ""
run sum "--ops sum,avg"
run mm "--ops min,max"
run cnt "--ops none"
DATABIN_LIB=paper_2310_02926_b200/variants/loads.so run loads ""
for v in $VARIANTS; do DATABIN_LIB=paper_2310_02926_b200/variants/$v.so run $v ""; done
