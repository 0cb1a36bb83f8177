#!/bin/bash
# K2b (pair keys of SIMD bins for B < 16 not dividing 16): parity + A/B against K2r (tuning knob)
O=${OUT:-gpurun_out/r02/k2b}; mkdir -p $O
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_variants.py -q -p no:cacheprovider -k "bin or fuzz or variant" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for b in 3 5 12 15 16 100; do
  SCN_LIB=tuning $T 4096 C2 hist --bins $b >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_PAIR_BINS=0 $T 4096 C2 hist --bins $b >> $O/tune.jsonl 2>/dev/null
done; done
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/k2b")+"/tune.jsonl"):
    d=json.loads(l); print(d['bins'], d['variant'], d['knobs'], round(d['GBps']))
PY
