#!/bin/bash
# half-lane 64 KB key block for the realigning fused kernel: parity, sanitizers, tile A/B
O=${OUT:-gpurun_out/r02/half}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -x -q -p no:cacheprovider > $O/sanitizer.log 2>&1; echo "sanitizer rc=$?"; tail -2 $O/sanitizer.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480; do
  $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null
  W=${sh%x*}
  for rows in 10 8; do SCN_LIB=tuning SCN_FUSED_TILE=$((rows * W * 3)) $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null; done
  for wp in 16; do SCN_LIB=tuning SCN_GEN_WARPS=$wp $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null; done
done
for op in histds; do $T 1024 C4 $op --offset 4 >> $O/tune.jsonl 2>/dev/null; done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/half")+"/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['knobs'], round(d['GBps']))
PY
