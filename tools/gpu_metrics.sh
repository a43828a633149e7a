#!/bin/bash
# quick pipe-utilisation metrics of one score_kernel launch for each library variant given
cd "$(dirname "$0")/.."
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio
for v in "$@"; do
  lib=""; [ "$v" != base ] && lib=tmp_ab/$v/libvdb200.so
  VD_LIB=$lib ncu --metrics $M --clock-control none -k regex:score_kernel -s 5 -c 1 python bench.py --steps 3 --warmup 3 --no-cpu --screen-ligands 0 2>&1 | grep -E "^\s+[a-z_]+__" | awk -v v=$v '{print v, $1, $NF}'
done
