#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_next.py tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/pytest_f4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_f4.log
OUT=gpurun_out/f4.jsonl; : > $OUT
for rep in 1 2; do
REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 histds >> $OUT 2>>gpurun_out/tune.err; echo "C4 histds" >> $OUT
REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 histds >> $OUT 2>>gpurun_out/tune.err; echo "C5 histds" >> $OUT
REPS=10 timeout 200 python tools/hist_tune.py shots 4096 C4 ds >> $OUT 2>>gpurun_out/tune.err; echo "C4 ds" >> $OUT
REPS=8 timeout 300 python tools/hist_tune.py shots 2048 C5 ds >> $OUT 2>>gpurun_out/tune.err; echo "C5 ds" >> $OUT
done
timeout 900 python bench.py --config C4 --cpu-seconds 5 > gpurun_out/bench_C4.json 2>/dev/null; echo "C4 bench $?"
timeout 1200 python bench.py --config C5 --round-frames 3584 --steps 5 --warmup 2 > gpurun_out/bench_C5_rounds.json 2>/dev/null; echo "C5 bench $?"
timeout 900 python bench.py --config C5 --frames 4096 --steps 10 --cpu-seconds 5 --e2e-frames 64 > gpurun_out/bench_C5.json 2>/dev/null; echo "C5b $?"
cat $OUT
