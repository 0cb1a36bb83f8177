"""Tuning sweep for the histogram kernel (not part of the product): times
scn_run_histogram on C2-shaped frames for one knob setting (env SCN_HIST_WARPS /
SCN_HIST_TILE are read by libscn.so) and content mode; prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1805_07339_b200 as scn  # noqa: E402
import scn_harness  # noqa: E402
import scn_synth  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "shots"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    cfg = sys.argv[3] if len(sys.argv) > 3 else "C2"
    op = sys.argv[4] if len(sys.argv) > 4 else "hist"
    wl = scn_synth.WORKLOADS[cfg]
    pl = scn_harness.plan(wl)
    frames = min(frames, len(pl[1]))
    job = scn_harness.DeviceJob(wl, 0, frames, with_halo=False, spec=wl.spec(mode=mode), plan_=pl)
    out = job.alloc_outputs(("hist", "downsample"), wl.bins)
    st = torch.cuda.current_stream()

    def call():
        if op == "hist":
            scn.scn_run_histogram(job.seq, 0, frames, wl.bins, out["hist"], st)
        elif op == "histds":
            scn.scn_run_hist_downsample(job.seq, 0, frames, wl.bins, out["hist"], out["ds"], st)
        else:
            scn.scn_run_downsample(job.seq, 0, frames, out["ds"], st)

    for _ in range(3):
        call()
    ts = []
    for _ in range(int(os.environ.get("REPS", "7"))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        call()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    per = wl.frame_bytes * (1.0 if op == "hist" else 1.25)  # algorithmic bytes: read F (+ write F/4)
    gbs = frames * per / (ms / 1e3) / 1e9
    print(json.dumps({"cfg": cfg, "op": op, "fused_tile": os.environ.get("SCN_FUSED_TILE", ""), "mode": mode, "frames": frames, "warps": os.environ.get("SCN_HIST_WARPS", "16"),
                      "tile": os.environ.get("SCN_HIST_TILE", "30720"), "ms": ms, "GBps": gbs,
                      "min_ms": min(ts), "all": [round(x, 3) for x in ts]}), flush=True)
    job.close()


if __name__ == "__main__":
    main()
