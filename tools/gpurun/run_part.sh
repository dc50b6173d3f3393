export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q 2>&1 | tail -5
WLS="c2 c4 c5" STEPS=20 bash tools/gpurun/run_wl.sh
bash tools/gpurun/prof_part.sh
