#!/bin/bash
# refresh every bench line under profiles/ (N = 1)
mkdir -p gpurun_out/prof
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
B="timeout 900 python bench.py"
$B --config C3 --cpu-seconds 5 > gpurun_out/prof/bench_C3.json 2>/dev/null; echo "C3 $?"
$B --config C4 --cpu-seconds 5 > gpurun_out/prof/bench_C4.json 2>/dev/null; echo "C4 $?"
$B --config C5 --frames 4096 --steps 10 --cpu-seconds 5 --e2e-frames 64 > gpurun_out/prof/bench_C5.json 2>/dev/null; echo "C5 $?"
$B --config C3 --graph e > gpurun_out/prof/bench_C3_graph_e.json 2>/dev/null; echo "C3e $?"
$B --cuts 16 --no-cpu-baseline --no-e2e > gpurun_out/prof/bench_C2_cuts16.json 2>/dev/null; echo "cuts $?"
$B --montage 8 --steps 10 > gpurun_out/prof/bench_C2_montage8.json 2>/dev/null; echo "montage $?"
$B --bins 256 --no-cpu-baseline --no-e2e > gpurun_out/prof/bench_C2_bins256.json 2>/dev/null; echo "bins256 $?"
$B --frames 2048 --no-cpu-baseline --no-e2e > gpurun_out/prof/bench_C2_2048f_shard_proxy.json 2>/dev/null; echo "proxy $?"
for m in uniform constant xgrad; do $B --mode $m --no-cpu-baseline --no-e2e > gpurun_out/prof/bench_C2_$m.json 2>/dev/null; echo "$m $?"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof/prof_histds \
   python bench.py --config C4 --steps 1 --warmup 2 --frames 1024 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_full_ds.log 2>&1; echo "ncu ds $?"
$B --config C5 --round-frames 3584 --steps 5 --warmup 2 > gpurun_out/prof/bench_C5_rounds.json 2>/dev/null; echo "C5 rounds $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof/prof_c5 \
   python bench.py --config C5 --steps 1 --warmup 2 --frames 512 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c5.log 2>&1; echo "ncu c5 $?"
bash tools/gpu_ncu_metrics.sh > gpurun_out/prof/ncu_metrics.log 2>&1; echo "ncu metrics $?"
