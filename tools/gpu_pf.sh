#!/bin/bash
# L2 bulk prefetch P tiles ahead of the TMA ring (SCN_L2_PREFETCH=P) on every config
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_L2_PREFETCH=3 timeout 600 python tests/helpers/variant_parity.py > gpurun_out/pf_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/pf_parity.log
OUT=gpurun_out/pf.jsonl; : > $OUT
for rep in 1 2; do
for P in 0 1 2 3 6; do
for cm in "C2 8192 hist" "C3 36864 hist" "C4 4096 histds" "C5 2048 histds"; do
set -- $P $cm
echo "{\"pf\": $1, \"cfg\": \"$2\", \"op\": \"$4\"}" >> $OUT
SCN_L2_PREFETCH=$1 REPS=6 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/pf.err
done; done; done
