#!/bin/bash
# r02 ncu evidence for the HEAD kernels: targeted counters (SURVEY §8(d) list) per kernel /
# shape, full-set captures for roofline.traffic (with the library's git SHA), and the launch
# list of the default bench command. Summaries land in gpurun_out/r02/ncu/.
set -u
O=${NCU_OUT:-gpurun_out/r02/ncu}
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
run hist 2048 C2 hist 0 "" 0
run histds 1024 C4 histds 0 "" 0
run ds 1024 C4 ds 0 "" 0
run hist_b100 2048 C2 hist 100 "" 0
run hist_b256 2048 C2 hist 256 "" 0
run histds_1366 2048 C4 histds 0 1366x768 0
run ds_1366 2048 C4 ds 0 1366x768 0
run histds_854 4096 C4 histds 0 854x480 0
run hist_k2a 128 C2 hist 0 "" 1
run hist_k2ap 512 C2 hist 0 "" 2
REPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 --csv \
  --log-file $O/counters_hist_joint8.csv python bench.py --joint 8 --frames 2048 --steps 1 --warmup 3 > $O/counters_hist_joint8.log 2>&1
python tools/ncu_summarize.py $O/counters_hist_joint8.csv hist_joint8 2048 C2 hist 0 "" $SHA > $O/counters_hist_joint8.json
REPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 --csv \
  --log-file $O/counters_hist_joint3.csv python bench.py --joint 3 --frames 2048 --steps 1 --warmup 3 > $O/counters_hist_joint3.log 2>&1
python tools/ncu_summarize.py $O/counters_hist_joint3.csv hist_joint3 2048 C2 hist 0 "" $SHA > $O/counters_hist_joint3.json
# full-set captures of the two headline kernels -> traffic summaries (bytes per frame, SHA)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_hist \
  python tools/hist_tune.py shots 2048 C2 hist --reps 1 > $O/full_hist.log 2>&1; echo "full hist $?"
python tools/ncu_traffic.py $O/full_hist.ncu-rep hist 2048 6220800 $SHA $O/ncu_hist_summary.json \
  "hist_tma_kernel<0,16>, C2 shape, 2048 frames/launch"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds \
  python tools/hist_tune.py shots 1024 C4 histds --reps 1 > $O/full_histds.log 2>&1; echo "full histds $?"
python tools/ncu_traffic.py $O/full_histds.ncu-rep histds 1024 6220800 $SHA $O/ncu_histds_summary.json \
  "hist_tma_kernel<2,8> fused hist+downsample, C4 shape, 1024 frames/launch"
# launch list of the default bench command (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --frames 4096 > $O/launches_bench.log 2>&1; echo "launches $?"
ls -la $O
for s in 1366x768 854x480; do
  run histds_gen_$s 1024 C4 histds 0 $s 0
  run ds_gen_$s 1024 C4 ds 0 $s 0
done
# traffic summaries for the other configs' frame sizes (C3 640x360 hist, C5 4K fused)
timeout 900 ncu --set full --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_hist_c3 \
  python tools/hist_tune.py shots 8192 C3 hist --reps 1 > $O/full_hist_c3.log 2>&1; echo "full hist c3 $?"
python tools/ncu_traffic.py $O/full_hist_c3.ncu-rep hist 8192 691200 $SHA $O/ncu_hist_c3_summary.json \
  "hist_tma_kernel<0,16>, C3 shape 640x360, 8192 frames/launch"
timeout 900 ncu --set full --clock-control none -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds_4k \
  python tools/hist_tune.py shots 512 C5 histds --reps 1 > $O/full_histds_4k.log 2>&1; echo "full histds 4k $?"
python tools/ncu_traffic.py $O/full_histds_4k.ncu-rep histds 512 24883200 $SHA $O/ncu_histds_4k_summary.json \
  "hist_tma_kernel<2,8> fused hist+downsample, C5 shape 3840x2160, 512 frames/launch"
