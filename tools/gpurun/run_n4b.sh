export DATABIN_NO_BUILD=1
N=4
for v in default cb512 cb128; do
  if [ "$v" = "default" ]; then unset DATABIN_LIB; else export DATABIN_LIB=paper_2310_02926_b200/variants/$v.so; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $N --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bn4_$v.json 2>/dev/null; echo $v; python tools/bench_lines.py gpurun_out/bn4_$v.json
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29525 bench.py --gpus $N --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bn4c4_$v.json 2>/dev/null; python tools/bench_lines.py gpurun_out/bn4c4_$v.json
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/mgpu_check.py > gpurun_out/mgpu_check_4.log 2>&1; echo mgpu_check=$?; grep -c '"ok"' gpurun_out/mgpu_check_4.log
