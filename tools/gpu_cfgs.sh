#!/bin/bash
# bench lines for every config at N=1 (C5 limited to the frames one GPU holds with its ds output)
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in C2 C3 C4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; cat gpurun_out/bench_$c.json | cut -c1-400; done
timeout 900 python bench.py --config C5 --frames 4096 --steps 5 --warmup 3 --cpu-seconds 5 --e2e-frames 64 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"; cut -c1-400 gpurun_out/bench_C5.json; tail -3 gpurun_out/bench_C5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof_histds \
   python bench.py --config C4 --steps 1 --warmup 2 --frames 1024 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_ds.log 2>&1; echo "ncu full rc=$?"
