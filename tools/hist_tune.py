"""Kernel timing for measurement runs (not part of the product): times one library call
(hist | histds | ds) over `frames` sampled frames of a config, optionally at another frame
size, bin count or histogram impl, and prints one JSON line with the median rate in
algorithmic GB/s. The measurement build's SCN_* knobs apply with SCN_LIB=tuning.

    python tools/hist_tune.py MODE FRAMES CFG OP [--bins B] [--shape WxH] [--impl I] [--reps R] [--offset O]
"""
import argparse
import dataclasses
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
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", nargs="?", default="shots")
    ap.add_argument("frames", nargs="?", type=int, default=4096)
    ap.add_argument("cfg", nargs="?", default="C2")
    ap.add_argument("op", nargs="?", default="hist", choices=["hist", "histds", "ds"])
    ap.add_argument("--bins", type=int, default=0)
    ap.add_argument("--shape", default="")
    ap.add_argument("--impl", type=int, default=0)
    ap.add_argument("--reps", type=int, default=int(os.environ.get("REPS", "7")))
    ap.add_argument("--offset", type=int, default=0, help="byte offset of the downsample output (alignment)")
    a = ap.parse_args()
    wl = scn_synth.WORKLOADS[a.cfg]
    if a.bins:
        wl = dataclasses.replace(wl, bins=a.bins)
    if a.shape:
        w, h = (int(x) for x in a.shape.lower().split("x"))
        wl = dataclasses.replace(wl, width=w, height=h)
    scn.scn_set_hist_impl(a.impl)
    pl = scn_harness.plan(wl)
    frames = min(a.frames, len(pl[1]))
    job = scn_harness.DeviceJob(wl, 0, frames, with_halo=False, spec=wl.spec(mode=a.mode), plan_=pl)
    out = job.alloc_outputs(("hist",), wl.bins)
    dsb = frames * (wl.height // 2) * (wl.width // 2) * 3
    ds = torch.empty(dsb + 16, dtype=torch.uint8, device="cuda") if a.op != "hist" else None
    dptr = ds.data_ptr() + a.offset if ds is not None else None
    st = torch.cuda.current_stream()

    def call():
        if a.op == "hist":
            scn.scn_run_histogram(job.seq, 0, frames, wl.bins, out["hist"], st)
        elif a.op == "histds":
            scn.scn_run_hist_downsample(job.seq, 0, frames, wl.bins, out["hist"], dptr, st)
        else:
            scn.scn_run_downsample(job.seq, 0, frames, dptr, st)

    for _ in range(3):
        call()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        call()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    F = wl.frame_bytes
    alg = frames * F + (dsb if a.op != "hist" else 0) + (frames * 3 * wl.bins * 4 if a.op != "ds" else 0)
    print(json.dumps({"cfg": a.cfg, "op": a.op, "mode": a.mode, "frames": frames, "width": wl.width,
                      "height": wl.height, "bins": wl.bins, "impl": a.impl, "offset": a.offset,
                      "variant": scn.scn_hist_variant(wl.bins), "ms": ms, "GBps": alg / (ms / 1e3) / 1e9,
                      "min_ms": min(ts), "all": [round(x, 3) for x in ts], "library": scn.scn_version(),
                      "knobs": {k: v for k, v in os.environ.items() if k.startswith("SCN_")}}), flush=True)
    job.close()


if __name__ == "__main__":
    main()
