#!/bin/bash
# ncu counters of the kernels added late in round 2: K2b, fused kVarBins, fused kVarRaw
set -u
O=${NCU_OUT:-gpurun_out/r02/ncu_new}
mkdir -p $O
SHA=$(python -c "import paper_1805_07339_b200 as s; print(s.scn_version().split(', ')[1].rstrip(')'))")
echo "library sha $SHA"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,\
sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,\
l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,\
smsp__inst_executed_op_global_st.sum,smsp__inst_executed_op_global_red.sum,sm__inst_executed_pipe_tma.sum,\
sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,\
smsp__inst_executed_op_match.sum,smsp__inst_executed_op_shfl.sum,\
smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,\
smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_drain.ratio,smsp__average_warp_latency_issue_stalled_membar.ratio,\
lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
run() {  # name frames cfg op bins shape impl
  REPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 --csv \
    --log-file $O/counters_$1.csv python tools/hist_tune.py shots $2 $3 $4 --bins $5 --shape "$6" --impl $7 --reps 1 \
    > $O/counters_$1.log 2>&1
  echo "$1 rc=$?"
  python tools/ncu_summarize.py $O/counters_$1.csv $1 $2 $3 $4 $5 "$6" $SHA > $O/counters_$1.json
}
run hist_b5_k2b 2048 C2 hist 5 "" 0
run histds_b5_bins 1024 C4 histds 5 "" 0
run histds_b100_raw 1024 C4 histds 100 "" 0
run histds_b5_bins_1366 2048 C4 histds 5 1366x768 0
run histds_b100_raw_1366 2048 C4 histds 100 1366x768 0
ls -la $O
