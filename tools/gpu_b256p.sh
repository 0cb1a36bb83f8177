#!/bin/bash
# NEXT N4: B = 256 PRMT table layout (default) vs the previous shifted-key layout (SCN_HIST_VAR=64)
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/pytest_b256.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_b256.log
OUT=gpurun_out/b256.jsonl; : > $OUT
for rep in 1 2 3; do
for v in 0 64; do
for m in shots uniform; do
SCN_HIST_VAR=$v timeout 600 python bench.py --bins 256 --frames 4096 --mode $m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); r=d['roofline']
print(json.dumps({'var': $v, 'mode': '$m', 'GBps': r['achieved'], 'ms': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $OUT
done; done; done
timeout 600 python bench.py --bins 256 --no-cpu-baseline --no-e2e > gpurun_out/bench_b256_full.json 2>/dev/null; echo "full $?"
