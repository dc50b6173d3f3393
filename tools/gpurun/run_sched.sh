export DATABIN_NO_BUILD=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 500 python tools/trace_bin.py 2>&1 | grep -E "trace|---" | grep -v "ticket 1 \|ticket 2 \|ticket 3 \|ticket 4 "
VARIANTS="tp2 tp8 tp16" bash tools/gpurun/ab.sh
