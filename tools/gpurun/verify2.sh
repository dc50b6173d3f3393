#!/bin/bash
# GPU tests (incl. the full-size C4 check), bench with the new cpu_baseline, host info
mkdir -p gpurun_out
export DATABIN_NO_BUILD=1
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
tail -25 gpurun_out/gputest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc=$?"
cat gpurun_out/host.txt
