O=gpurun_out/r02/gen2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gen.py -x -q -p no:cacheprovider 2>&1 | tail -2
T="python tools/hist_tune.py shots"
for r in 1 2; do
for sh in 1366x768 854x480; do
  for op in ds histds; do $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null; done
done
for op in ds histds; do $T 1024 C4 $op --offset 4 >> $O/tune.jsonl 2>/dev/null; $T 1024 C4 $op >> $O/tune.jsonl 2>/dev/null; done
$T 4096 C2 hist >> $O/tune.jsonl 2>/dev/null
for ns in 200 1000 5000; do SCN_LIB=tuning SCN_PROD_SLEEP=$ns $T 4096 C2 hist >> $O/tune.jsonl 2>/dev/null; SCN_LIB=tuning SCN_PROD_SLEEP=$ns $T 1024 C4 histds >> $O/tune.jsonl 2>/dev/null; SCN_LIB=tuning SCN_PROD_SLEEP=$ns $T 2048 C4 histds --shape 1366x768 >> $O/tune.jsonl 2>/dev/null; done
done
python - <<'PY'
import json
for l in open("gpurun_out/r02/gen2/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], d['knobs'].get('SCN_PROD_SLEEP',''), round(d['GBps']))
PY
