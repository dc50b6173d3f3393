export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/b1.json 2>gpurun_out/b1.err; python tools/bench_lines.py gpurun_out/b1.json
N=2; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $N --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/b2.json 2> gpurun_out/b2.err; python tools/bench_lines.py gpurun_out/b2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/mgpu_check.py > gpurun_out/mgpu_check_2.log 2>&1; echo mgpu_check=$?; grep -c '"ok"' gpurun_out/mgpu_check_2.log
