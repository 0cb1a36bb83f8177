#!/bin/bash
# fused raw-key hist + downsample: consumer warps (tuning build)
O=${OUT:-gpurun_out/r02/fraw2}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
T="python tools/hist_tune.py shots"
for r in 1 2; do for b in 100; do
  for wp in 0 12 16; do SCN_LIB=tuning SCN_GEN_WARPS=$wp $T 1024 C4 histds --bins $b >> $O/tune.jsonl 2>/dev/null; done
  for wp in 0 16; do SCN_LIB=tuning SCN_GEN_WARPS=$wp $T 2048 C4 histds --bins $b --shape 1366x768 >> $O/tune.jsonl 2>/dev/null; done
  SCN_LIB=tuning SCN_FUSED_RAW=0 $T 1024 C4 histds --bins $b >> $O/tune.jsonl 2>/dev/null
done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/fraw2")+"/tune.jsonl"):
    d=json.loads(l); print(d['width'], d['bins'], d['knobs'], round(d['GBps']), round(d['ms'],3))
PY
