#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_next.py tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/pytest_f2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_f2.log
OUT=gpurun_out/f2.jsonl; : > $OUT
for rep in 1 2; do
REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "C4 histds" >> $OUT
REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "C5 histds" >> $OUT
REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "C4 ds" >> $OUT
SCN_FUSED_TILE=34560 REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "C4 histds t34560" >> $OUT
done
cat $OUT
