#!/bin/bash
# ncu source-level capture of the fused realigning kernel (1366x768) for per-instruction counts
O=gpurun_out/r02/srcprof; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds_1366 \
  python tools/hist_tune.py shots 512 C4 histds --shape 1366x768 --reps 1 > $O/full_histds_1366.log 2>&1; echo "gen histds $?"
ncu -i $O/full_histds_1366.ncu-rep --page source --csv --print-source sass > $O/src_sass.csv 2>&1; echo "src $?"
ls -la $O
