# Is the sustained (power-capped) rate a property of HBM streaming itself? A pure TMA read of
# the same ring shape (no histogram work) vs the histogram kernel, both for ~40 back-to-back
# launches, with nvidia-smi clocks/power sampled alongside.
O=gpurun_out/r02/power; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 200 > $O/smi_read.csv &
S=$!
./tools/micro/k0 40 > $O/k0_sustained.json
kill $S
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 200 > $O/smi_hist.csv &
S=$!
REPS=40 python tools/hist_tune.py shots 8192 C2 hist --reps 40 > $O/hist_sustained.json
kill $S
python - <<'PY'
import json, statistics, csv
k = json.load(open("gpurun_out/r02/power/k0_sustained.json"))
v = k["sustained_tma_read_GBps"]
print("pure TMA read GB/s: median", round(statistics.median(v)), "first", round(v[0]), "last", round(v[-1]))
h = json.loads(open("gpurun_out/r02/power/hist_sustained.json").read())
F = 6220800 * 8192
r = [F / (t / 1e3) / 1e9 for t in h["all"]]
print("hist GB/s: median", round(statistics.median(r)), "first", round(r[0]), "last", round(r[-1]))
for fn in ("smi_read", "smi_hist"):
    rows = [x for x in csv.reader(open(f"gpurun_out/r02/power/{fn}.csv"))]
    clk = [float(x[0].split()[0]) for x in rows if x and x[0].strip()[0].isdigit()]
    pw = [float(x[1].split()[0]) for x in rows if len(x) > 1 and x[1].strip()[0].isdigit()]
    cap = sum(1 for x in rows if len(x) > 2 and "Active" in x[2])
    print(fn, "sm MHz median", statistics.median(clk), "min", min(clk), "power W median", statistics.median(pw), "max", max(pw), "capped samples", cap, "/", len(rows))
PY
