#!/bin/bash
# downsample-only kernel sweep (warps x tile) + the sanitizer tests
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q > gpurun_out/pytest_san.log 2>&1; echo "san rc=$?"; tail -1 gpurun_out/pytest_san.log
OUT=gpurun_out/dsonly.jsonl; : > $OUT
for rep in 1 2; do
for w in 8 16; do
for t in 0 23040 34560 64512; do
for cf in "C4 4096" "C5 2048"; do
set -- $cf
echo "{\"warps\": $w, \"tile\": $t, \"cfg\": \"$1\"}" >> $OUT
if [ $t = 0 ]; then SCN_FUSED_WARPS=$w REPS=6 timeout 300 python tools/hist_tune.py shots $2 $1 ds >> $OUT 2>>gpurun_out/dsonly.err
else SCN_DS_TILE=$t SCN_FUSED_WARPS=$w REPS=6 timeout 300 python tools/hist_tune.py shots $2 $1 ds >> $OUT 2>>gpurun_out/dsonly.err; fi
done; done; done; done
