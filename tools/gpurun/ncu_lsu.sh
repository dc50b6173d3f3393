#!/bin/bash
# LSU wavefront breakdown of the bin kernel on a workload (WL), one launch
export DATABIN_NO_BUILD=1
mkdir -p gpurun_out
B="python bench.py --workload ${WL:-c3} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
M=l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,smsp__inst_executed.sum,smsp__inst_executed_op_shared_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_red.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:${K:-k_bin} -s 3 -c 1 $B > gpurun_out/ncu_lsu_${TAG:-x}.log 2>&1; echo ncu=$?
