#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_variants.py -m gpu -q -k "DS_VAR" > gpurun_out/pytest_dsv.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_dsv.log
OUT=gpurun_out/dsv.jsonl; : > $OUT
for rep in 1 2; do for v in 1 2; do
SCN_DS_VAR=$v REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "dsv=$v C4 histds" >> $OUT
SCN_DS_VAR=$v REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "dsv=$v C5 histds" >> $OUT
SCN_DS_VAR=$v REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "dsv=$v C4 ds" >> $OUT
done; done
cat $OUT
