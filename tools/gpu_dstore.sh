#!/bin/bash
# downsample output by TMA bulk stores (SCN_DS_STORE=1, default) vs per-thread STG (0):
# parity of every ds path, then C4/C5 fused and C4 ds-only timings, alternating
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvcc -o /tmp/smembase tools/micro/smembase.cu -gencode arch=compute_100a,code=sm_100a && /tmp/smembase
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_next.py -m gpu -q -x > gpurun_out/pytest_dstore.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_dstore.log
OUT=gpurun_out/dstore.jsonl; : > $OUT
for rep in 1 2; do for v in 0 1; do
SCN_DS_STORE=$v REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "store=$v C4 histds" >> $OUT
SCN_DS_STORE=$v REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "store=$v C5 histds" >> $OUT
SCN_DS_STORE=$v REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "store=$v C4 ds" >> $OUT
done; done
cat $OUT | cut -c1-200
