#!/bin/bash
# fused kVarGen: bigger tiles on a 2-stage ring vs the 3-stage default (tuning build)
O=${OUT:-gpurun_out/r02/twostage}; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do
  for sh in 854x480 1366x768 426x240; do W=${sh%x*}; $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null; done
  for rows in 20 22 24; do SCN_LIB=tuning SCN_GEN_HALF=0 SCN_FUSED_TILE=$((rows * 854 * 3)) $T 2048 C4 histds --shape 854x480 >> $O/tune.jsonl 2>/dev/null; done
  for rows in 12 14; do SCN_LIB=tuning SCN_GEN_HALF=0 SCN_FUSED_TILE=$((rows * 1366 * 3)) $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null; done
  for rows in 16; do SCN_LIB=tuning SCN_GEN_HALF=0 SCN_GEN_WARPS=16 SCN_FUSED_TILE=$((rows * 1366 * 3)) $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null; done
  for rows in 40 44 48; do SCN_LIB=tuning SCN_GEN_HALF=0 SCN_FUSED_TILE=$((rows * 426 * 3)) $T 2048 C4 histds --shape 426x240 >> $O/tune.jsonl 2>/dev/null; done
done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/twostage")+"/tune.jsonl"):
    d=json.loads(l); print(d['width'], d['knobs'], round(d['GBps']))
PY
