# per-workload kernel timings on 1 GPU (no e2e / cpu baseline)
export DATABIN_NO_BUILD=1
for wl in ${WLS:-c2 c3 c4 c5}; do
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/wl_$wl.json 2> gpurun_out/wl_$wl.err
  python -c "import json; d=json.load(open('gpurun_out/wl_$wl.json')); print('$wl', round(d['value']/1e9,2), 'G/s step', round(d['ms_per_step'],4), 'bin', round(d['roofline']['ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), d.get('window'), d.get('profile_ms'))" 2>&1 | tail -1
done
