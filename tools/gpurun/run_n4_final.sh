# 4-GPU round: fan-in parity + placement study (incl. 3:1 fan-in), multi-GPU parity, C3 strong/weak/exact
export DATABIN_NO_BUILD=1
N=${N:-4}
timeout 600 python -m pytest tests/test_gpu_shards.py tests/test_gpu_placement_study.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_n$N.log 2>&1; echo pytest=$?
timeout 900 python tools/placement_study.py --n 50000000 --steps 100 > gpurun_out/placement_n$N.jsonl 2> gpurun_out/placement_n$N.err; echo study=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo mgpu_check=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo bench=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --scaling weak > gpurun_out/bench_n${N}_weak.json 2>> gpurun_out/bench_n$N.err; echo weak=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --exact > gpurun_out/bench_n${N}_exact.json 2>> gpurun_out/bench_n$N.err; echo exact=$?
tail -2 gpurun_out/pytest_n$N.log; grep -c '"ok"' gpurun_out/mgpu_check_$N.log; grep -E "FAIL|rror" gpurun_out/mgpu_check_$N.log | head -3
