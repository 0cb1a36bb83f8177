O=gpurun_out/r02/warps; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do for w in 8 16 20; do
  SCN_LIB=tuning SCN_HIST_WARPS=$w $T 4096 C2 hist --bins 100 >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_HIST_WARPS=$w $T 4096 C2 hist >> $O/tune.jsonl 2>/dev/null
done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/warps/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['bins'], d['knobs'].get('SCN_HIST_WARPS',''), round(d['GBps']))
PY
