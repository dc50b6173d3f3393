# Scaling sequence as the driver runs it (C3 strong, N = 1, 2, 4 on one box) + C4 at N=4 + exact at each N
export DATABIN_NO_BUILD=1
timeout 300 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 > gpurun_out/scale_n1.json 2> gpurun_out/scale.err; echo n1=$?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 100 --warmup 5 > gpurun_out/scale_n$N.json 2>> gpurun_out/scale.err; echo n$N=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_c4_n4.json 2>> gpurun_out/scale.err; echo c4=$?
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scale_c4_n1.json 2>> gpurun_out/scale.err; echo c4n1=$?
python tools/bench_lines.py gpurun_out/scale_n1.json gpurun_out/scale_n2.json gpurun_out/scale_n4.json gpurun_out/scale_c4_n4.json gpurun_out/scale_c4_n1.json
