#!/bin/bash
# ring-depth cap (SCN_MAX_STAGES) on the downsample-only and histogram kernels
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_MAX_STAGES=3 timeout 600 python tests/helpers/variant_parity.py > gpurun_out/st_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/st_parity.log | cut -c1-80
OUT=gpurun_out/stages.jsonl; : > $OUT
for rep in 1 2 3; do
for st in 0 3 2; do
for cm in "C4 4096 ds" "C5 2048 ds" "C2 8192 hist" "C3 36864 hist"; do
set -- $st $cm
echo "{\"cap\": $1, \"cfg\": \"$2\", \"op\": \"$4\"}" >> $OUT
SCN_MAX_STAGES=$1 REPS=6 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/stages.err
done; done; done
