#!/bin/bash
# kVarGen staged bulk-store output: parity, sanitizers, A/B against the direct cross-lane stores
O=${OUT:-gpurun_out/r02/stage}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -x -q -p no:cacheprovider > $O/sanitizer.log 2>&1; echo "sanitizer rc=$?"; tail -2 $O/sanitizer.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240; do for op in histds ds; do
  $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_GEN_STAGE=0 $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null
  [ $sh = 1366x768 ] && [ $op = histds ] && SCN_LIB=tuning SCN_GEN_STAGE=0 SCN_FUSED_TILE=32784 $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null
done; done
for op in histds ds; do $T 1024 C4 $op --offset 4 >> $O/tune.jsonl 2>/dev/null; SCN_LIB=tuning SCN_GEN_STAGE=0 $T 1024 C4 $op --offset 4 >> $O/tune.jsonl 2>/dev/null; done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/stage")+"/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['knobs'], round(d['GBps']))
PY
