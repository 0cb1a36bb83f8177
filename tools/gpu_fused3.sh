#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/f3.jsonl; : > $OUT
for t in 23040 34560 46080 57600; do SCN_FUSED_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "C4 histds t=$t" >> $OUT; done
for t in 23040 46080; do SCN_FUSED_TILE=$t REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "C5 histds t=$t" >> $OUT; done
for t in 11520 23040 34560 46080; do SCN_DS_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "C4 ds t=$t" >> $OUT; done
for w in 8 16; do SCN_FUSED_WARPS=$w REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "C4 ds w=$w" >> $OUT; done
cat $OUT
