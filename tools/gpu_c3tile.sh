#!/bin/bash
# C3 (640x360, F = 691,200 = 16.07 default tiles): balanced tile sizes vs the default 43,008
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/c3tile.jsonl; : > $OUT
for rep in 1 2; do
for t in 43008 40704 38400 34560; do
echo "{\"tile\": $t}" >> $OUT
SCN_HIST_TILE=$t REPS=8 timeout 300 python tools/hist_tune.py shots 36864 C3 hist >> $OUT 2>>gpurun_out/c3tile.err
done; done
