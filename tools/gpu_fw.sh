#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_next.py -m gpu -q -x > gpurun_out/pytest_fw.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_fw.log
OUT=gpurun_out/fw.jsonl; : > $OUT
for w in 8 16; do SCN_FUSED_WARPS=$w REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "ds w=$w C4" >> $OUT; done
cat $OUT
