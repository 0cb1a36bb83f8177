#!/usr/bin/env python3
"""Film summary on a synthetic film, through the public API only (the paper's data-mining
flow): HIST + [-1,0] shot-diff over every frame, the bounded-state adaptive cut
detector (warmup W), then a second job that gathers the first frame of every shot and
tiles their 2x downsamples into a montage, written as a binary PPM.

    python examples/shot_montage.py --frames 2000 --cols 8 --out montage.ppm
    python examples/shot_montage.py --joint 4          # shots scored on 64-bin joint-colour histograms
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_07339_b200 as scn  # noqa: E402
import scn_harness  # noqa: E402
import scn_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=2000)
    ap.add_argument("--cols", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=16, help="adaptive detector window W")
    ap.add_argument("--out", default="montage.ppm")
    ap.add_argument("--joint", type=int, default=0,
                    help="J > 0: score shots on joint-colour histograms (J bins per channel, J^3 bins)")
    a = ap.parse_args()

    wl = scn_synth.WORKLOADS["C2"]                       # 1920x1080 synthetic film
    plan = tuple(x[: a.frames] for x in scn_harness.plan(wl))
    M = len(plan[1])
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, plan_=plan)   # frames resident in HBM

    # job 1: HIST + shot-diff, then the bounded-state detector (cut if D > 4 x mean of last W + W*H/8)
    if a.joint:  # NEXT N4's joint-colour variant: J^3 counters per frame, the same [-1,0] stencil
        J = a.joint
        hist = torch.empty((M, J ** 3), dtype=torch.int32, device="cuda")
        diff = torch.empty(M, dtype=torch.int32, device="cuda")
        scratch = torch.empty(J ** 3, dtype=torch.int32, device="cuda")
        scn.scn_run_hist_shotdiff_joint(job.seq, 0, M, J, hist, diff, scratch)
    else:
        out = job.alloc_outputs(("hist", "shotdiff"), wl.bins)
        scn.scn_run_hist_shotdiff(job.seq, 0, M, wl.bins, out["hist"], out["diff"], out["scratch"])
        diff = out["diff"]
    cuts = torch.empty(M, dtype=torch.uint8, device="cuda")
    scn.scn_run_adaptive_cuts(job.seq, 0, M, a.warmup, diff, 4, 1, wl.width * wl.height // 8, cuts)
    starts = [0] + (torch.nonzero(cuts).flatten().cpu().numpy()).tolist()

    # job 2: gather the first frame of every shot, downsample into montage tiles
    kseq = scn.scn_seq_gather_positions(job.seq, np.array(sorted(set(starts)), dtype=np.int64))
    k = scn.scn_seq_length(kseq)
    ws = torch.empty(max(scn.scn_seq_device_bytes(kseq), 16), dtype=torch.uint8, device="cuda")
    scn.scn_seq_upload(kseq, ws, ws.numel())
    oh, ow = wl.height // 2, wl.width // 2
    canvas = torch.empty((-(-k // a.cols) * oh, a.cols * ow, 3), dtype=torch.uint8, device="cuda")
    scn.scn_run_montage(kseq, 0, k, a.cols, canvas, a.cols * ow * 3)
    img = canvas.cpu().numpy()
    with open(a.out, "wb") as f:
        f.write(f"P6 {img.shape[1]} {img.shape[0]} 255\n".encode())
        f.write(img.tobytes())
    print(f"{M} frames, {k} shots -> {a.out} ({img.shape[1]}x{img.shape[0]})")
    scn.scn_seq_destroy(kseq)
    job.close()


if __name__ == "__main__":
    main()
