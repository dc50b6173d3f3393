# ncu --set full of the given kernels (regex) on a workload: KREGEX, WL, TAG
export DATABIN_NO_BUILD=1
B="python bench.py --workload ${WL:-c5} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain_full.log 2>&1 || { echo plain failed; exit 1; }
for k in $KREGEX; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-3} -c 1 -o gpurun_out/prof_${TAG}_$k $B > gpurun_out/ncu_full_${TAG}_$k.log 2>&1; echo $k full=$?
done
