#!/bin/bash
# ncu --set full of the histogram kernel on C3 (640x360, stride-30 sparse rows)
mkdir -p gpurun_out/prof
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 2 -c 1 -o gpurun_out/prof/prof_c3 \
   python bench.py --config C3 --steps 1 --warmup 2 --frames 8192 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_c3.log 2>&1; echo "ncu c3 $?"
