set -x
export DATABIN_NO_BUILD=1
timeout 600 python -m pytest tests/test_gpu_placement.py tests/test_gpu_placement_study.py -x -q 2>&1 | tail -5
timeout 900 python tools/placement_study.py --n 50000000 --steps 100 > gpurun_out/placement.jsonl 2> gpurun_out/placement.err; echo rc=$?
cat gpurun_out/placement.jsonl
export CUDA_VISIBLE_DEVICES=0
VARIANTS="gfoff" bash tools/gpurun/ab.sh
BENCH_ARGS="--workload c5" VARIANTS="gfoff" bash tools/gpurun/ab.sh
