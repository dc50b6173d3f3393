#!/bin/bash
# Scaling record as the driver runs it (C3 strong, N = 1, 2, 4 on one box) + weak / exact at N=4 + C4 at N=1/4
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 > gpurun_out/sf_n1.json 2> gpurun_out/sf.err; echo n1=$?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --steps 100 --warmup 5 > gpurun_out/sf_n$N.json 2>> gpurun_out/sf.err; echo n$N=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 4 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --scaling weak > gpurun_out/sf_n4_weak.json 2>> gpurun_out/sf.err; echo weak=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29732 bench.py --gpus 4 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --exact > gpurun_out/sf_n4_exact.json 2>> gpurun_out/sf.err; echo exact=$?
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --exact > gpurun_out/sf_n1_exact.json 2>> gpurun_out/sf.err; echo exact1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29733 bench.py --gpus 4 --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sf_c4_n4.json 2>> gpurun_out/sf.err; echo c4=$?
DATABIN_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29734 tools/trace_combine.py 2>&1 | grep "barrier" | tail -4
python tools/bench_lines.py gpurun_out/sf_n1.json gpurun_out/sf_n2.json gpurun_out/sf_n4.json gpurun_out/sf_n4_weak.json gpurun_out/sf_n1_exact.json gpurun_out/sf_n4_exact.json gpurun_out/sf_c4_n4.json
