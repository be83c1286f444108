#!/bin/bash
# ncu evidence for the bench kernel (B200_PROFILING.md recipe), reduced on the
# GPU box to small files under gpurun_out/:
#   <tag>_launches.csv   per-launch gpu__time_duration of `bench.py` (launch list)
#   <tag>_kernel.csv     one config-4 sweep launch: DRAM / L2 traffic, issue,
#                        instruction-cache and stall metrics
# usage: tools/ncu_bench.sh TAG   (run after bench.py has exited 0 without ncu)
set -u
TAG=${1:-r2}
O=gpurun_out
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu --c5-stride 0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches.csv \
    python bench.py $ARGS > $O/${TAG}_launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__icc_request_hit_rate.pct,sm__warps_active.avg.per_cycle_active
M=$M,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warp_latency_per_inst_issued.ratio
M=$M,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum
ncu --metrics $M --clock-control none -k regex:kvsim_sweep -s 1 -c 1 --csv --log-file $O/${TAG}_kernel.csv \
    python bench.py $ARGS > $O/${TAG}_kernel.log 2>&1
echo ncu_rc=$?
