export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "det or we or c1 or c2 or c3 or random or ragged or zero or dyadic" 2>&1 | tail -3; echo
EXTRA=--deterministic WLS="c3 c2" STEPS=5 bash tools/gpurun/run_wl.sh
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --deterministic"
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_det.csv $B > /dev/null 2>&1; echo ncu=$?
