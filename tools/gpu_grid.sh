#!/bin/bash
# persistent-CTA count sweep (SCN_GRID): fewer SMs streaming, each with the same 3-stage ring
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_GRID=100 timeout 600 python tests/helpers/variant_parity.py > gpurun_out/grid_parity.log 2>&1; echo "parity rc=$?"
OUT=gpurun_out/grid.jsonl; : > $OUT
for rep in 1 2; do
for g in 0 144 136 128 112 96; do
for cm in "C2 8192 hist" "C3 36864 hist" "C4 4096 histds" "C5 2048 histds"; do
set -- $g $cm
echo "{\"grid\": $1, \"cfg\": \"$2\", \"op\": \"$4\"}" >> $OUT
SCN_GRID=$1 REPS=5 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/grid.err
done; done; done
