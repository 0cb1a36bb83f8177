#!/bin/bash
# ring-depth cap for the kernels whose smaller tables leave room for > 3 stages (bins != 16, 256)
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
OUT=gpurun_out/stages2.jsonl; : > $OUT
for rep in 1 2; do
for b in 64 32 128 8 100; do
for st in 0 3; do
SCN_MAX_STAGES=$st timeout 600 python bench.py --bins $b --frames 4096 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); r=d['roofline']
print(json.dumps({'bins': $b, 'cap': $st, 'GBps': r['achieved'], 'ms': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $OUT
done; done; done
