#!/bin/bash
# 4-GPU box: multi-GPU parity (peer + NVLS), GPU tests incl. the 2-GPU ones, bench N=2/4 at the driver's flags, reference arm at N=4
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tools/mgpu_check.py > gpurun_out/f4_mgpu_peer.log 2>&1; echo mgpu_peer=$?; tail -2 gpurun_out/f4_mgpu_peer.log
DATABIN_COMBINE=nvls timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29742 tools/mgpu_check.py > gpurun_out/f4_mgpu_nvls.log 2>&1; echo mgpu_nvls=$?; tail -2 gpurun_out/f4_mgpu_nvls.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/f4_gputest.log 2>&1; echo gputest=$?; tail -3 gpurun_out/f4_gputest.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2975$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/f4_n$N.json 2>> gpurun_out/f4.err; echo n$N=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29759 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/f4_ref_n4.json 2>> gpurun_out/f4.err; echo ref4=$?
python tools/bench_lines.py gpurun_out/f4_n2.json gpurun_out/f4_n4.json gpurun_out/f4_ref_n4.json
