O=gpurun_out/r02/raw2; mkdir -p $O
SCN_LIB=tuning SCN_RAW2=1 timeout 600 python tests/helpers/variant_parity.py 2>&1 | tail -1
T="python tools/hist_tune.py shots"
for r in 1 2 3; do for v in 0 1; do
  SCN_LIB=tuning SCN_RAW2=$v $T 4096 C2 hist --bins 100 >> $O/tune.jsonl 2>/dev/null
  SCN_LIB=tuning SCN_RAW2=$v $T 16384 C3 hist --bins 256 >> $O/tune.jsonl 2>/dev/null
done; done
# sustained: 40 launches of 8192 frames each (~50 GB per launch)
for v in 0 1 0 1; do SCN_LIB=tuning SCN_RAW2=$v REPS=40 $T 8192 C2 hist --bins 100 --reps 40 >> $O/sustained.jsonl 2>/dev/null; done
python - <<'PY'
import json, statistics
for fn in ("tune", "sustained"):
    for l in open(f"gpurun_out/r02/raw2/{fn}.jsonl"):
        d=json.loads(l); print(fn, d['cfg'], d['bins'], d['knobs'].get('SCN_RAW2'), round(d['GBps']), "mean-ms", round(statistics.mean(d['all']),3), "min", d['min_ms'])
PY
