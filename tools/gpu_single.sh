#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_n4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_n4.log
SCN_HIST_SINGLE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_shapes or content or c1" > gpurun_out/pytest_single.log 2>&1; echo "pytest single rc=$?"; tail -1 gpurun_out/pytest_single.log
OUT=gpurun_out/single.jsonl; : > $OUT
for sg in 0 1; do for t in 43008 64512; do SCN_HIST_SINGLE=$sg SCN_HIST_TILE=$t REPS=15 timeout 200 python tools/hist_tune.py shots 8192 C2 >> $OUT 2>>gpurun_out/tune.err; echo "single=$sg tile=$t" >> $OUT; done; done
for b in 256 64; do timeout 600 python bench.py --config C2 --bins $b --frames 4096 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_b$b.json 2> gpurun_out/bench_C2_b$b.err; python -c "
import json; d=json.load(open('gpurun_out/bench_C2_b$b.json')); r=d['roofline']; print('bins', $b, round(d['value']), round(r['achieved']), round(r['frac'],3), d['config']['hist_variant'])" >> $OUT; done
cat $OUT
