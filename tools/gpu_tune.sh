#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/tune2.jsonl; : > $OUT
for w in 16 8; do for t in 24576 30720 32256 36864 43008 49152 64512; do
  SCN_HIST_WARPS=$w SCN_HIST_TILE=$t timeout 120 python tools/hist_tune.py shots 4096 >> $OUT 2>>gpurun_out/tune.err
done; done
for t in 32256 43008 64512; do SCN_HIST_TILE=$t timeout 120 python tools/hist_tune.py shots 36864 C3 >> $OUT 2>>gpurun_out/tune.err; done
cat $OUT
