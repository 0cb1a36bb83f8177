#!/bin/bash
# fused kVarGen: ring depth x tile rows x warps (tuning build)
O=${OUT:-gpurun_out/r02/stages3}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480; do W=${sh%x*}
  $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null
  for wp in 12 16; do for cfg in "8 4" "6 5" "6 4" "10 3" "4 6"; do set -- $cfg
    SCN_LIB=tuning SCN_GEN_WARPS=$wp SCN_FUSED_TILE=$(($1 * W * 3)) SCN_MAX_STAGES=$2 $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null
  done; done
done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/stages3")+"/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['knobs'], round(d['GBps']))
PY
