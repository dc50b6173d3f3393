#!/bin/bash
# ncu evidence for the bench kernel: launch list of the bench command + one --set full capture of k_bin_fast
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/fp_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fp_launches.csv $B > gpurun_out/fp_ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bin_fast -s 2 -c 1 -o gpurun_out/fp_kbin $B > gpurun_out/fp_ncu_full.log 2>&1; echo full=$?
