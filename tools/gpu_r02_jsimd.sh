#!/bin/bash
# joint-colour SIMD binning (non-power-of-2 J): parity + same-box A/B old/new library
O=${OUT:-gpurun_out/r02/jsimd}; mkdir -p $O
P=paper_1805_07339_b200
make -j8 all > $O/make.log 2>&1 || { tail $O/make.log; exit 1; }
cp $P/libscn.so $P/libscn_ab_new.so
timeout 900 python -m pytest tests/test_gpu_joint.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for r in 1 2; do for v in old new; do cp $P/libscn_ab_$v.so $P/libscn.so
  for j in ${JS:-3 5 7 8}; do timeout 300 python bench.py --joint $j --frames 4096 --steps 20 | sed "s/^{/{\"ab\": \"$v\", /" >> $O/bench.jsonl 2>/dev/null; done
done; done
cp $P/libscn_ab_new.so $P/libscn.so
python - <<'PY'
import json,os
for l in open(os.environ.get("OUT","gpurun_out/r02/jsimd")+"/bench.jsonl"):
    d=json.loads(l); print(d['ab'], d['config']['joint_bins'], round(d['value']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])
PY
