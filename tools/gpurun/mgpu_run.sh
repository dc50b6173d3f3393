# N-GPU round: NCCL parity check + bench at N (launched as the driver does)
export DATABIN_NO_BUILD=1
N=${N:-2}
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo mgpu_check=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --scaling weak > gpurun_out/bench_n${N}_weak.json 2>> gpurun_out/bench_n$N.err; echo bench_weak=$?
cat gpurun_out/mgpu_check_$N.log | grep -E "case|Error|FAIL" | head -20
if [ "${C4:-0}" = "1" ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $N --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_c4.json 2>> gpurun_out/bench_n$N.err; echo bench_c4=$?
fi
python tools/bench_lines.py gpurun_out/bench_n$N.json gpurun_out/bench_n${N}_weak.json gpurun_out/bench_n${N}_c4.json
if [ "${AB_NCCL:-0}" = "1" ]; then
DATABIN_COMBINE=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_nccl.json 2>> gpurun_out/bench_n$N.err; echo bench_nccl=$?
python tools/bench_lines.py gpurun_out/bench_n${N}_nccl.json
fi
if [ "${AB_PEER:-0}" = "1" ]; then
DATABIN_COMBINE=peer timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_peer.json 2>> gpurun_out/bench_n$N.err; echo bench_peer=$?
python tools/bench_lines.py gpurun_out/bench_n${N}_peer.json
fi
