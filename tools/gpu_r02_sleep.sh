O=gpurun_out/r02/sleep; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do for c in 0 100 1000; do for pz in 0 1000; do
  SCN_LIB=tuning SCN_CONS_SLEEP=$c SCN_PROD_SLEEP=$pz $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_CONS_SLEEP=$c SCN_PROD_SLEEP=$pz $T 1024 C4 histds >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_CONS_SLEEP=$c SCN_PROD_SLEEP=$pz $T 4096 C2 hist --bins 100 >> $O/tune.jsonl 2>/dev/null
done; done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/sleep/tune.jsonl"):
    d=json.loads(l); k=d['knobs']; print(d['op'], d['width'], d['bins'], k.get('SCN_CONS_SLEEP'), k.get('SCN_PROD_SLEEP'), round(d['GBps']))
PY
