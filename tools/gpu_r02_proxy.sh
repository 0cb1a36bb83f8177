# per-GPU shard sizes of the strong-scaling run (N = 2, 4, 8, 16 -> 8192 .. 1024 frames) on one GPU
mkdir -p gpurun_out/r02
for f in 8192 4096 2048 1024; do timeout 300 python bench.py --frames $f --no-cpu-baseline --no-e2e > gpurun_out/r02/proxy_$f.json 2>/dev/null; done
for f in 8192 4096 2048 1024; do python - $f <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads(open(f"gpurun_out/r02/proxy_{f}.json").read())
b = d["breakdown"]
print(f, round(d["value"]), round(d["ms_per_step"], 4), round(b["overhead_ms"][0] * 1000, 1), "us", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
