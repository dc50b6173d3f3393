# GPU round: parity tests, bench, launch list, ncu full of the bin kernel
export DATABIN_NO_BUILD=1
TAG=${TAG:-r}
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 200 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench=$?
B="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin -s 2 -c 1 -o gpurun_out/prof_kbin_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1; echo full=$?
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log
