export DATABIN_NO_BUILD=1
N=${N:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tools/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo mgpu_check=$?; grep -c '"ok"' gpurun_out/mgpu_check_$N.log; grep -v '"ok"' gpurun_out/mgpu_check_$N.log | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/trace_combine.py 2>&1 | grep "trace" | grep "rank 0" | tail -3
for b in 1 0; do
DATABIN_COMBINE_BULK=$b timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$b bench.py --gpus $N --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_n${N}_bulk$b.json 2>/dev/null; echo bulk=$b; python tools/bench_lines.py gpurun_out/bench_n${N}_bulk$b.json
done
