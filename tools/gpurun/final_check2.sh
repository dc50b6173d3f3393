#!/bin/bash
# Round-end check (final code): GPU tests, smoke, bench (driver's flags), reference arm, launch list, ncu --set full of k_bin_fast
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1; echo gputest=$?; tail -2 gpurun_out/final_gputest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final_smoke.log
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench=$?
timeout 300 python bench.py --gpus 1 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/final_bench100.json 2>> gpurun_out/final_bench.err; echo bench100=$?
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_ref.json 2>> gpurun_out/final_bench.err; echo ref=$?
B="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $B > gpurun_out/final_ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bin_fast -s 3 -c 1 -o gpurun_out/final_kbin -f $B > gpurun_out/final_ncu_full.log 2>&1; echo ncufull=$?
python tools/bench_lines.py gpurun_out/final_bench.json gpurun_out/final_bench100.json
