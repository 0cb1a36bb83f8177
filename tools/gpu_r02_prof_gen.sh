O=gpurun_out/r02/ncu
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_histds_1366 \
  python tools/hist_tune.py shots 512 C4 histds --shape 1366x768 --reps 1 > $O/full_histds_1366.log 2>&1; echo "gen histds $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hist_tma_kernel -s 3 -c 1 -o $O/full_ds_1366 \
  python tools/hist_tune.py shots 512 C4 ds --shape 1366x768 --reps 1 > $O/full_ds_1366.log 2>&1; echo "gen ds $?"
