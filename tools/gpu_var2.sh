#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/var2.jsonl; : > $OUT
for rep in 1 2; do for v in 0 1 2 3; do SCN_HIST_VAR=$v REPS=15 timeout 200 python tools/hist_tune.py shots 8192 >> $OUT 2>>gpurun_out/tune.err; done; done
cat $OUT
