#!/bin/bash
# NVLink data counters (nvidia-smi nvlink -gt d, per link, KiB) around a 2-GPU bench of K steps:
# bytes the peer combine moves per step (ncu cannot replay a kernel that spins on another GPU's flags)
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
nvidia-smi nvlink -gt d > gpurun_out/nvl_before.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29741 bench.py --gpus 2 --steps 1000 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/nvl_bench.json 2> gpurun_out/nvl.err; echo bench=$?
nvidia-smi nvlink -gt d > gpurun_out/nvl_after.txt 2>&1
head -20 gpurun_out/nvl_after.txt
