#!/bin/bash
# fused hist + downsample at B > 16 (raw byte keys, half-lane block): parity, sanitizers, A/B vs two passes
O=${OUT:-gpurun_out/r02/fraw}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_gen.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sanitizer.py tests/test_gpu_variants.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for b in 32 100 256; do
  $T 1024 C4 histds --bins $b >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_FUSED_RAW=0 $T 1024 C4 histds --bins $b >> $O/tune.jsonl 2>/dev/null
  $T 2048 C4 histds --bins $b --shape 1366x768 >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_FUSED_RAW=0 $T 2048 C4 histds --bins $b --shape 1366x768 >> $O/tune.jsonl 2>/dev/null
done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/fraw")+"/tune.jsonl"):
    d=json.loads(l); print(d['width'], d['bins'], d['knobs'], round(d['GBps']), round(d['ms'],3))
PY
