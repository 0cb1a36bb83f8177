O=gpurun_out/r02/balance; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2 3; do for b in 0 1; do
  SCN_LIB=tuning SCN_HIST_BALANCE=$b $T 4096 C2 hist >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_HIST_BALANCE=$b $T 16384 C3 hist >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_HIST_BALANCE=$b $T 4096 C2 hist --bins 100 >> $O/tune.jsonl 2>/dev/null
done; done
SCN_LIB=tuning SCN_HIST_BALANCE=1 timeout 300 python tests/helpers/variant_parity.py | tail -1
python - <<'PY'
import json
for l in open("gpurun_out/r02/balance/tune.jsonl"):
    d=json.loads(l); print(d['cfg'], d['bins'], d['knobs'].get('SCN_HIST_BALANCE'), round(d['GBps']), round(d['ms'],3))
PY
