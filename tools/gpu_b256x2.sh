#!/bin/bash
# NEXT N4: B = 256 two-block table (SCN_HIST_B256X2=1, every byte one PRMT, 3 x 31,728-B stages)
# vs the default one-block table (channel 2 PRMT + IMAD, 3 x 43,008-B stages)
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_HIST_B256X2=1 timeout 600 python tests/helpers/variant_parity.py > gpurun_out/vp_b256x2.log 2>&1; echo "vp rc=$?"; tail -1 gpurun_out/vp_b256x2.log
: timeout 1200 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/pytest_b256x2.log 2>&1; echo "variants rc=$?"; tail -1 gpurun_out/pytest_b256x2.log
OUT=gpurun_out/b256x2.jsonl; : > $OUT
for rep in 1 2 3; do
for v in 0 1; do
for m in shots uniform; do
SCN_HIST_B256X2=$v timeout 600 python bench.py --bins 256 --frames 4096 --mode $m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); r=d['roofline']
print(json.dumps({'x2': $v, 'mode': '$m', 'frames': 4096, 'GBps': r['achieved'], 'ms': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $OUT
done; done; done
for v in 0 1; do
SCN_HIST_B256X2=$v timeout 600 python bench.py --bins 256 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); r=d['roofline']
print(json.dumps({'x2': $v, 'mode': 'shots', 'frames': 16384, 'GBps': r['achieved'], 'ms': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $OUT
done
