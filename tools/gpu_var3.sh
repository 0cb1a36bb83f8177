#!/bin/bash
mkdir -p gpurun_out
make -j8 all micro > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/var3_clocks.csv &
SMI=$!
./tools/micro/k0 40 > gpurun_out/var3.txt
sleep 2
REPS=40 timeout 200 python tools/hist_tune.py shots 8192 >> gpurun_out/var3.txt 2>>gpurun_out/tune.err
kill $SMI
cat gpurun_out/var3.txt
