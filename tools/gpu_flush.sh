#!/bin/bash
# flush without zeroing (default: cumulative lane counters, per-row previous sums in registers)
# vs the previous flush that re-zeroes the table (SCN_FLUSH_ZERO=1), + full GPU parity
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_flush.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_flush.log
OUT=gpurun_out/flush.jsonl; : > $OUT
for rep in 1 2 3; do
for z in 0 1; do
for cm in "C3 36864 hist" "C2 8192 hist" "C4 4096 histds" "C5 2048 histds"; do
set -- $z $cm
echo "{\"zero\": $1, \"cfg\": \"$2\", \"op\": \"$4\"}" >> $OUT
SCN_FLUSH_ZERO=$1 REPS=6 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/flush.err
done; done; done
