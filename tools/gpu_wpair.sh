#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -m gpu -q -x > gpurun_out/pytest_wp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_wp.log
OUT=gpurun_out/wp.jsonl; : > $OUT
for rep in 1 2; do for v in 0 8; do SCN_HIST_VAR=$v REPS=15 timeout 200 python tools/hist_tune.py shots 8192 C2 >> $OUT 2>>gpurun_out/tune.err; echo "var=$v" >> $OUT; done; done
for v in 0 8; do SCN_HIST_VAR=$v REPS=15 timeout 200 python tools/hist_tune.py uniform 8192 C2 >> $OUT 2>>gpurun_out/tune.err; echo "var=$v uniform" >> $OUT; done
REPS=10 timeout 200 python tools/hist_tune.py shots 36864 C3 >> $OUT 2>>gpurun_out/tune.err; echo "C3" >> $OUT
REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "C4 histds" >> $OUT
REPS=10 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "C5 histds" >> $OUT
cat $OUT
