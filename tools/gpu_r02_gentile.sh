O=gpurun_out/r02/gentile; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do
for t in 0 24588 32784 45078 57372; do
  SCN_LIB=tuning SCN_FUSED_TILE=$t $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_FUSED_TILE=$t SCN_GEN_WARPS=16 $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null
done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/gentile/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['knobs'], round(d['GBps']))
PY
