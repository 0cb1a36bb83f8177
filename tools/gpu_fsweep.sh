#!/bin/bash
# fused split-layout sweep: consumer warps x tile size on C4 / C5
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/fsweep.jsonl; : > $OUT
for rep in 1 2; do
for w in 8 12 16; do
for ct in "C5 2048 0" "C5 2048 23040" "C4 4096 0" "C4 4096 34560"; do
set -- $ct
echo "{\"warps\": $w, \"cfg\": \"$1\", \"tile\": $3}" >> $OUT
if [ $3 = 0 ]; then SCN_FUSED_WARPS=$w REPS=6 timeout 300 python tools/hist_tune.py shots $2 $1 histds >> $OUT 2>>gpurun_out/fsweep.err
else SCN_FUSED_TILE=$3 SCN_FUSED_WARPS=$w REPS=6 timeout 300 python tools/hist_tune.py shots $2 $1 histds >> $OUT 2>>gpurun_out/fsweep.err; fi
done; done; done
SCN_FUSED_WARPS=16 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_shapes or content or sampling" > gpurun_out/pytest_w16.log 2>&1; echo "w16 parity rc=$?"; tail -1 gpurun_out/pytest_w16.log
SCN_FUSED_WARPS=12 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_shapes or content or sampling" > gpurun_out/pytest_w12.log 2>&1; echo "w12 parity rc=$?"; tail -1 gpurun_out/pytest_w12.log
