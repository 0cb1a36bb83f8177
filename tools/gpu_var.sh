#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/var.jsonl; : > $OUT
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/var_clocks.csv &
SMI=$!
for f in 4096 8192 16384; do REPS=20 timeout 200 python tools/hist_tune.py shots $f >> $OUT 2>>gpurun_out/tune.err; done
kill $SMI
cat $OUT
