#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -m gpu -q -x -k "downsample or small_shapes or content or c4 or c5 or host or n1" > gpurun_out/pytest_ds.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ds.log
OUT=gpurun_out/ds.jsonl; : > $OUT
for t in 34560 46080 57600 64512; do SCN_FUSED_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; done
for t in 23040 34560 46080 64512; do SCN_FUSED_TILE=$t REPS=10 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; done
cat $OUT
