#!/bin/bash
# fused hist+downsample: split ring layout (default) vs the previous 96 KB table layout, same session
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_split.log
OUT=gpurun_out/split.jsonl; : > $OUT
for rep in 1 2; do
for sp in 1 0; do
for cfgop in "C5 histds 2048" "C4 histds 4096" "C5 histds_xgrad 2048"; do
set -- $cfgop
op=$2; mode=shots; [ $op = histds_xgrad ] && { op=histds; mode=uniform; }
echo "{\"split\": $sp, \"cfg\": \"$1\", \"op\": \"$op\", \"mode\": \"$mode\"}" >> $OUT
SCN_FUSED_SPLIT=$sp REPS=8 timeout 300 python tools/hist_tune.py $mode $3 $1 $op >> $OUT 2>>gpurun_out/split.err
done; done; done
for t in 23040 34560; do
echo "{\"split\": 1, \"tile\": $t, \"cfg\": \"C4\", \"op\": \"histds\", \"mode\": \"shots\"}" >> $OUT
SCN_FUSED_TILE=$t REPS=8 timeout 300 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/split.err
done
