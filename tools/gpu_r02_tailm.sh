O=gpurun_out/r02/tailm; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider 2>&1 | tail -1
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240; do $T 2048 C4 histds --shape $sh >> $O/tune.jsonl 2>/dev/null; done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/tailm/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], round(d['GBps']))
PY
