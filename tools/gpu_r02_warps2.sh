#!/bin/bash
# kVarGen consumer-warp sweep after the half-lane block / staged ds stores (tuning build)
O=${OUT:-gpurun_out/r02/warps2}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240; do for op in histds ds; do
  $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null
  for wp in 12 16 20 24; do SCN_LIB=tuning SCN_GEN_WARPS=$wp $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null; done
done; done
for wp in 16 20 24; do SCN_LIB=tuning SCN_GEN_WARPS=$wp SCN_GEN_STAGE=0 $T 2048 C4 ds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null; done
done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/warps2")+"/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['knobs'], round(d['GBps']))
PY
