# launch lists (per-kernel device time) of the partition route on C5 / C2 / C4
export DATABIN_NO_BUILD=1
for wl in c5 c2; do
  B="python bench.py --workload $wl --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $B > gpurun_out/plain_$wl.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum --clock-control none --csv --log-file gpurun_out/launches_part_$wl.csv $B > gpurun_out/ncu_launch_$wl.log 2>&1; echo $wl launches=$?
done
B="python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum --clock-control none --csv --log-file gpurun_out/launches_part_c4.csv $B > gpurun_out/ncu_launch_c4.log 2>&1; echo c4 launches=$?
