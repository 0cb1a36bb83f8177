O=gpurun_out/r02/genw; mkdir -p $O
T="python tools/hist_tune.py shots"
for r in 1 2; do for w in 12 16; do for sh in 1366x768 854x480; do for op in histds ds; do
  SCN_LIB=tuning SCN_GEN_WARPS=$w $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null; done; done; done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/genw/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['knobs'].get('SCN_GEN_WARPS'), round(d['GBps']))
PY
