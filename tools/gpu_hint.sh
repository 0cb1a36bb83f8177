#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_TMA_HINT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c1 or small_shapes" > gpurun_out/pytest_hint.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_hint.log
OUT=gpurun_out/hint.jsonl; : > $OUT
for rep in 1 2; do for h in 0 1; do
SCN_TMA_HINT=$h REPS=40 timeout 300 python tools/hist_tune.py shots 8192 C2 >> $OUT 2>>gpurun_out/tune.err; echo "hint=$h C2" >> $OUT
SCN_TMA_HINT=$h REPS=15 timeout 300 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "hint=$h C4" >> $OUT
done; done
cat $OUT
