O=gpurun_out/r02/gen5; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gen.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider 2>&1 | tail -2
T="python tools/hist_tune.py shots"
for r in 1 2; do for sh in 1366x768 854x480 426x240; do for op in histds ds; do $T 2048 C4 $op --shape $sh >> $O/tune.jsonl 2>/dev/null; done; done
for op in histds ds; do $T 1024 C4 $op --offset 4 >> $O/tune.jsonl 2>/dev/null; done; done
python - <<'PY'
import json
for l in open("gpurun_out/r02/gen5/tune.jsonl"):
    d=json.loads(l); print(d['op'], d['width'], d['offset'], round(d['GBps']))
PY
