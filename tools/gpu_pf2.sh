#!/bin/bash
# confirm: fused default (1 tile of L2 prefetch) vs SCN_L2_PREFETCH=0; ds-only with 0 / 1
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_pf2.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_pf2.log
OUT=gpurun_out/pf2.jsonl; : > $OUT
for rep in 1 2 3; do
for P in def 0; do
for cm in "C4 4096 histds" "C5 2048 histds" "C4 4096 ds" "C2 8192 hist"; do
set -- $P $cm
echo "{\"pf\": \"$1\", \"cfg\": \"$2\", \"op\": \"$4\"}" >> $OUT
if [ $1 = def ]; then REPS=6 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/pf2.err
else SCN_L2_PREFETCH=$1 REPS=6 timeout 300 python tools/hist_tune.py shots $3 $2 $4 >> $OUT 2>>gpurun_out/pf2.err; fi
done; done
echo "{\"pf\": \"1\", \"cfg\": \"C4\", \"op\": \"ds\"}" >> $OUT
SCN_L2_PREFETCH=1 REPS=6 timeout 300 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/pf2.err
done
