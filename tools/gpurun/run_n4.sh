export DATABIN_NO_BUILD=1
N=4
for b in 1 0; do
DATABIN_COMBINE_BULK=$b timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$b bench.py --gpus $N --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_bulk$b.json 2>/dev/null; echo bulk=$b; python tools/bench_lines.py gpurun_out/bench_n${N}_bulk$b.json
DATABIN_COMBINE_BULK=$b timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$b bench.py --gpus $N --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_c4_bulk$b.json 2>/dev/null; python tools/bench_lines.py gpurun_out/bench_n${N}_c4_bulk$b.json
done
