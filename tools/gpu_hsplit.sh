#!/bin/bash
# hist-only kernel: split layout (SCN_HIST_SPLIT=1) x tile size vs the default 96 KB table
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/pytest_hsplit.log 2>&1; echo "variants rc=$?"; tail -1 gpurun_out/pytest_hsplit.log
OUT=gpurun_out/hsplit.jsonl; : > $OUT
for rep in 1 2; do
for cfg in "0 43008" "1 43008" "1 33792" "1 30720" "1 23040"; do
set -- $cfg
for cm in "C2 8192 shots" "C3 36864 shots" "C2 8192 uniform"; do
set -- $1 $2 $cm
echo "{\"split\": $1, \"tile\": $2, \"cfg\": \"$3\", \"mode\": \"$5\"}" >> $OUT
SCN_HIST_SPLIT=$1 SCN_HIST_TILE=$2 REPS=8 timeout 300 python tools/hist_tune.py $5 $4 $3 hist >> $OUT 2>>gpurun_out/hsplit.err
done; done; done
