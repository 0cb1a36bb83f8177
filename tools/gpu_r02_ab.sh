# A/B of two product-library builds: paper_1805_07339_b200/libscn_ab_{old,new}.so swapped in turn
O=gpurun_out/r02/ab; mkdir -p $O
P=paper_1805_07339_b200
T="python tools/hist_tune.py shots"
for r in 1 2 3; do for v in old new; do
  cp $P/libscn_ab_$v.so $P/libscn.so
  for b in 100 256; do $T 4096 C2 hist --bins $b | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl; done
  $T 16384 C3 hist --bins 100 | sed "s/^{/{\"ab\": \"$v\", /" >> $O/tune.jsonl
done; done
cp $P/libscn_ab_new.so $P/libscn.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "bin or small_shapes" 2>&1 | tail -1
python - <<'PY'
import json
for l in open("gpurun_out/r02/ab/tune.jsonl"):
    d=json.loads(l); print(d['ab'], d['cfg'], d['bins'], round(d['GBps']))
PY
