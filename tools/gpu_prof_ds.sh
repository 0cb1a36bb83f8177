#!/bin/bash
mkdir -p gpurun_out/prof
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof/prof_histds8 \
   python bench.py --config C4 --steps 1 --warmup 2 --frames 1024 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_ds8.log 2>&1; echo "ncu ds $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof/prof_c5 \
   python bench.py --config C5 --steps 1 --warmup 2 --frames 512 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c5.log 2>&1; echo "ncu c5 $?"
