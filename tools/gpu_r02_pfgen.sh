#!/bin/bash
# fused kVarGen: L2 bulk-prefetch distance (tuning build)
O=${OUT:-gpurun_out/r02/pfgen}; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480; do for pf in 0 1 2 3; do
  SCN_LIB=tuning SCN_L2_PREFETCH=$pf $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null
done; done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/pfgen")+"/tune.jsonl"):
    d=json.loads(l); print(d['width'], d['knobs'], round(d['GBps']))
PY
