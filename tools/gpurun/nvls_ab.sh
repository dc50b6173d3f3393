#!/bin/bash
# NVLS vs IPC-peer combine at N GPUs: parity check (NVLS default), bench both, combine phase trace
export DATABIN_NO_BUILD=1
N=${N:-2}
mkdir -p gpurun_out
if [ "${CHECK:-1}" = "1" ]; then
DATABIN_COMBINE=${CHECK_COMBINE:-nvls} timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 tools/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo mgpu_check=$? ok=$(grep -c '"ok"' gpurun_out/mgpu_check_$N.log) fail=$(grep -c FAIL gpurun_out/mgpu_check_$N.log)
fi
for mode in nvls peer nccl; do
  env_c="DATABIN_COMBINE=$mode"
  env $env_c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/nab_${mode}_n$N.json 2> gpurun_out/nab_n$N.err
  python tools/bench_lines.py gpurun_out/nab_${mode}_n$N.json | cut -c1-200
done
DATABIN_COMBINE=nvls DATABIN_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29631 tools/trace_combine.py 2>&1 | grep "barrier" | tail -4
