#!/bin/bash
# 2-GPU box, final code: all GPU tests (incl. the 2-GPU ones), multi-GPU parity at N=2, smoke, bench N=1 / N=2 at the
# driver's flags, C4 / C5 / C2 bench lines, launch list
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/fc3_gputest.log 2>&1; echo gputest=$?; tail -2 gpurun_out/fc3_gputest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 tools/mgpu_check.py > gpurun_out/fc3_mgpu.log 2>&1; echo mgpu=$? ok=$(grep -c '"status": "ok"' gpurun_out/fc3_mgpu.log)
timeout 300 python __graft_entry__.py smoke > gpurun_out/fc3_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/fc3_smoke.log
timeout 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fc3_bench.json 2> gpurun_out/fc3.err; echo bench=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29762 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/fc3_bench_n2.json 2>> gpurun_out/fc3.err; echo bench2=$?
for wl in c4 c5 c2; do st=100; [ $wl = c4 ] && st=10; timeout 300 python bench.py --workload $wl --steps $st --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fc3_$wl.json 2>> gpurun_out/fc3.err; echo $wl=$?; done
python tools/bench_lines.py gpurun_out/fc3_bench.json gpurun_out/fc3_bench_n2.json gpurun_out/fc3_c4.json gpurun_out/fc3_c5.json gpurun_out/fc3_c2.json
