#!/bin/bash
# fused kVarGen: warps x staged stores (tuning build)
O=${OUT:-gpurun_out/r02/warps3}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 600 env SCN_LIB=tuning SCN_GEN_STAGE=2 python -m pytest tests/test_gpu_gen.py -x -q -p no:cacheprovider > $O/pytest_stage2.log 2>&1; echo "pytest stage2 rc=$?"; tail -1 $O/pytest_stage2.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240 1280x720; do
  for wp in 12 16; do for st in 1 2; do SCN_LIB=tuning SCN_GEN_WARPS=$wp SCN_GEN_STAGE=$st $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null; done; done
done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/warps3")+"/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['knobs'], round(d['GBps']))
PY
