#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/tune.jsonl; : > $OUT
for w in 8 16 24; do for t in 15360 23040 30720 33792; do
  SCN_HIST_WARPS=$w SCN_HIST_TILE=$t timeout 120 python tools/hist_tune.py shots 4096 >> $OUT 2>>gpurun_out/tune.err
done; done
for m in uniform constant xgrad; do timeout 120 python tools/hist_tune.py $m 4096 >> $OUT 2>>gpurun_out/tune.err; done
timeout 120 python tools/hist_tune.py shots 36864 C3 >> $OUT 2>>gpurun_out/tune.err
cat $OUT
