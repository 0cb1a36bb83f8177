#!/bin/bash
# Targeted ncu counters (SURVEY §8(d) list) for the three hot kernels, one launch each:
# hist (C2, 2048 frames), fused hist+ds (C4, 1024 frames), ds-only (C4, 1024 frames).
# Summarised by tools/ncu_summarize.py into gpurun_out/ncu_counters_*.json.
mkdir -p gpurun_out
[ -f paper_1805_07339_b200/libscn.so ] || make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,\
sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,\
l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,\
smsp__inst_executed_op_global_st.sum,smsp__inst_executed_op_global_red.sum,sm__inst_executed_pipe_tma.sum,\
sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,\
smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,\
smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,\
lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
run() {  # name frames cfg op
  REPS=1 timeout 600 ncu --metrics $M --clock-control none -k regex:hist_tma_kernel -s 1 -c 1 --csv \
    --log-file gpurun_out/ncu_counters_$1.csv python tools/hist_tune.py shots $2 $3 $4 > gpurun_out/ncu_counters_$1.log 2>&1
  echo "$1 rc=$?"
  python tools/ncu_summarize.py gpurun_out/ncu_counters_$1.csv $1 $2 $3 $4 > gpurun_out/ncu_counters_$1.json
  cat gpurun_out/ncu_counters_$1.json
}
run hist 2048 C2 hist
run histds 1024 C4 histds
run ds 1024 C4 ds
