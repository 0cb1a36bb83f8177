#!/bin/bash
# PRMT table layout (default) vs the previous layout (SCN_HIST_VAR=64): parity, then A/B timings
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_prmt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_prmt.log
OUT=gpurun_out/prmt.jsonl; : > $OUT
for rep in 1 2 3; do for v in 64 0; do
SCN_HIST_VAR=$v REPS=15 timeout 300 python tools/hist_tune.py shots 8192 C2 hist >> $OUT 2>>gpurun_out/tune.err; echo "var=$v C2 hist 8192" >> $OUT
SCN_HIST_VAR=$v REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "var=$v C4 histds" >> $OUT
done; done
SCN_HIST_VAR=0 REPS=15 timeout 300 python tools/hist_tune.py uniform 8192 C2 hist >> $OUT 2>>gpurun_out/tune.err; echo "var=0 C2 hist uniform" >> $OUT
SCN_HIST_VAR=0 REPS=15 timeout 300 python tools/hist_tune.py constant 8192 C2 hist >> $OUT 2>>gpurun_out/tune.err; echo "var=0 C2 hist constant" >> $OUT
cat $OUT | cut -c1-150
