#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_gpu_variants.py -m gpu -q > gpurun_out/pytest_var.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_var.log
OUT=gpurun_out/match.jsonl; : > $OUT
for m in shots uniform constant; do SCN_HIST_IMPL=match REPS=5 timeout 300 python tools/hist_tune.py $m 1024 C2 >> $OUT 2>>gpurun_out/tune.err; echo "match $m" >> $OUT; done
REPS=5 timeout 300 python tools/hist_tune.py shots 1024 C2 >> $OUT 2>>gpurun_out/tune.err; echo "pairs shots" >> $OUT
cat $OUT
