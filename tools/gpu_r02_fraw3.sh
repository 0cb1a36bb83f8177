#!/bin/bash
# fused raw keys on the split table (full-lane channels 0/1) vs the half-lane block (old lib): parity + A/B
O=${OUT:-gpurun_out/r02/fraw3}; mkdir -p $O
P=paper_1805_07339_b200
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
cp $P/libscn.so $P/libscn_ab_new.so
timeout 1200 python -m pytest tests/test_gpu_gen.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sanitizer.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
T="python tools/hist_tune.py shots"
for r in 1 2; do for v in old new; do cp $P/libscn_ab_$v.so $P/libscn.so
  for b in 32 100 256; do $T 1024 C4 histds --bins $b | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl 2>/dev/null; done
  $T 256 C5 histds --bins 100 | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl 2>/dev/null
done; done
cp $P/libscn_ab_new.so $P/libscn.so
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/fraw3")+"/tune.jsonl"):
    d=json.loads(l); print(d['ab'], d['cfg'], d['bins'], round(d['GBps']))
PY
