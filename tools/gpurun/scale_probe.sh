#!/bin/bash
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
python tools/nvls_probe.py > gpurun_out/nvls_probe.txt 2>&1; cat gpurun_out/nvls_probe.txt
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --cpu-seconds 2 > gpurun_out/scale_n1.json 2> gpurun_out/scale.err; echo n1=$?
for N in 2 4; do
  NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 100 --warmup 5 --no-e2e > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err; echo n$N=$?
  DATABIN_COMBINE=nccl NCCL_DEBUG=INFO timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 100 --warmup 5 --no-e2e > gpurun_out/scale_nccl_n$N.json 2> gpurun_out/scale_nccl_n$N.err; echo nccl n$N=$?
done
grep -i "nvls" gpurun_out/scale_nccl_n4.err | head -5
python tools/bench_lines.py gpurun_out/scale_n1.json gpurun_out/scale_n2.json gpurun_out/scale_n4.json gpurun_out/scale_nccl_n2.json gpurun_out/scale_nccl_n4.json
