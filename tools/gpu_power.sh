#!/bin/bash
# sustained C2 bench (40 steps) with consumers spinning on the full barrier (default) vs parked
# with a suspend hint (SCN_CONS_SUSPEND=1): does the spin cost power / clock under sw_power_cap?
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SCN_CONS_SUSPEND=1 timeout 600 python tests/helpers/variant_parity.py > gpurun_out/pw_parity.log 2>&1; echo "parity rc=$?"
OUT=gpurun_out/power.jsonl; : > $OUT
for rep in 1 2 3; do
for v in 0 1; do
SCN_CONS_SUSPEND=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); r=d['roofline']
print(json.dumps({'suspend': $v, 'value': d['value'], 'GBps': r['achieved'], 'ms': d['ms_per_step'], 'min_ms': d['step_ms_min'], 'med_ms': d['step_ms_median'], 'clocks': d['clocks']}))" >> $OUT
done; done
