#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for v in 0 1; do SCN_DS_VAR=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "downsample or small_shapes or content or c4 or c5 or host" > gpurun_out/pytest_ds$v.log 2>&1; echo "pytest dsvar=$v rc=$?"; tail -1 gpurun_out/pytest_ds$v.log; done
OUT=gpurun_out/ds.jsonl; : > $OUT
for v in 0 1; do for t in 46080 64512; do
SCN_DS_VAR=$v SCN_FUSED_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err
SCN_DS_VAR=$v SCN_FUSED_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err
SCN_DS_VAR=$v SCN_FUSED_TILE=$t REPS=10 timeout 200 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err
done; done
cat $OUT
