"""Small workload exercising every kernel once, for compute-sanitizer (T4):
memcheck / racecheck / synccheck must report 0 errors. Also checks parity."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import scn_harness  # noqa: E402
import scn_synth  # noqa: E402
from scn_synth import Workload  # noqa: E402


def check(wl, ops, bins, fused=True, host=False):
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    b, e = M // 3, M
    job = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl)
    out = job.alloc_outputs(ops, bins)
    if host:
        hj = scn_harness.HostJob(wl, b, e, with_halo=True, plan_=pl, staging_frames=2)
        hj.run(out, ops, bins, stream=torch.cuda.current_stream(), copy_stream=torch.cuda.Stream())
    else:
        job.run(out, ops, bins, fused=fused)
    torch.cuda.synchronize()
    H, D, DS = oracle.run(wl.spec(), pl[0], pl[1], pl[2], b, e, bins, want_ds="downsample" in ops)
    n = e - b
    if "hist" in ops:
        assert (out["hist"].cpu().numpy().view(np.uint32)[:n] == H).all()
    if "shotdiff" in ops:
        assert (out["diff"].cpu().numpy().view(np.uint32)[:n] == D).all()
    if "downsample" in ops:
        assert (out["ds"].cpu().numpy()[:n] == DS).all()
    job.close()


def main():
    w1 = Workload("san1", 64, 36, 2, 20, ("stride", 1), (), spec_kw={"len_min": 3, "len_max": 7})
    w2 = Workload("san2", 67, 9, 1, 12, ("stride", 2), (), spec_kw={"len_min": 3, "len_max": 7})
    check(w1, ("hist", "shotdiff"), 16)
    check(w1, ("hist", "shotdiff"), 16, fused=False)
    check(w1, ("hist", "downsample"), 16)
    check(w1, ("downsample",), 16, fused=False)
    check(w2, ("hist", "shotdiff"), 5)
    check(w2, ("hist", "downsample"), 64)
    check(w1, ("hist", "shotdiff", "downsample"), 16, host=True)
    check(w1, ("hist", "shotdiff"), 256)   # NEXT N4 (single shifted key, B = 256)
    check(w1, ("hist", "shotdiff"), 64)
    # fused split layout with several row-pair tiles per frame (24-row tiles, 4-row tail)
    w3 = Workload("san3", 640, 100, 1, 6, ("stride", 1), (), spec_kw={"len_min": 2, "len_max": 4})
    check(w3, ("hist", "downsample"), 16)
    # realigning row-pair kernels (kVarGen): odd widths, several tiles per frame, odd output offsets
    check(w2, ("hist", "downsample"), 16)
    w4 = Workload("san4", 854, 30, 1, 4, ("stride", 1), (), spec_kw={"len_min": 2, "len_max": 4})
    check(w4, ("hist", "downsample"), 16)
    check(w4, ("downsample",), 16, fused=False)
    unaligned_out(w4)
    # the half-lane fused layout (1366 wide: 12-row tiles, 16 warps) and the staged bulk-store
    # downsample over several tiles with an odd last row
    w5 = Workload("san5", 1366, 29, 1, 3, ("stride", 1), (), spec_kw={"len_min": 2, "len_max": 3})
    check(w5, ("hist", "downsample"), 16)
    check(w5, ("downsample",), 16, fused=False)
    # fused hist + downsample at B < 16 not dividing 16 (K2b bins): aligned, realigning, half-lane
    check(w1, ("hist", "downsample"), 5)
    check(w4, ("hist", "downsample"), 12)
    check(w5, ("hist", "downsample"), 3)
    # ... and B > 16 (raw byte keys in the half-lane block; B = 256 emits value rows directly)
    check(w1, ("hist", "downsample"), 100)
    check(w4, ("hist", "downsample"), 256)
    check(w5, ("hist", "downsample"), 37)
    # the north_star's K2a and K2a' (per-warp bins, __match_any_sync)
    import paper_1805_07339_b200 as scn
    for impl in (1, 2):
        scn.scn_set_hist_impl(impl)
        check(w1, ("hist", "shotdiff"), 16)
    scn.scn_set_hist_impl(0)
    joint(w2, 4)
    joint(w1, 3)
    next_rows()
    print("sanitize_run ok")


def joint(wl, j):
    import paper_1805_07339_b200 as scn
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=False, plan_=pl)
    out = torch.empty((M, j ** 3), dtype=torch.int32, device="cuda")
    scn.scn_run_histogram_joint(job.seq, 0, M, j, out, job.stream)
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint32) == oracle.run_joint(wl.spec(), pl[0], pl[1], 0, M, j)).all()
    job.close()
    # joint shot-diff over a shard that needs its [-1,0] halo
    b = M // 2
    job = scn_harness.DeviceJob(wl, b, M, with_halo=True, plan_=pl)
    H = torch.empty((M - b, j ** 3), dtype=torch.int32, device="cuda")
    D = torch.empty(M - b, dtype=torch.int32, device="cuda")
    scratch = torch.empty(j ** 3, dtype=torch.int32, device="cuda")
    scn.scn_run_hist_shotdiff_joint(job.seq, b, M, j, H, D, scratch, job.stream)
    torch.cuda.synchronize()
    rh, rd = oracle.run_joint_diff(wl.spec(), pl[0], pl[1], pl[2], b, M, j)
    assert (H.cpu().numpy().view(np.uint32) == rh).all() and (D.cpu().numpy().view(np.uint32) == rd).all()
    job.close()


def unaligned_out(wl):
    import paper_1805_07339_b200 as scn
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=False, plan_=pl)
    _, _, DS = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 0, M, 16, want_ds=True)
    nb = M * (wl.height // 2) * (wl.width // 2) * 3
    buf = torch.zeros(nb + 16, dtype=torch.uint8, device="cuda")
    hist = torch.empty((M, 3, 16), dtype=torch.int32, device="cuda")
    scn.scn_run_hist_downsample(job.seq, 0, M, 16, hist, buf.data_ptr() + 3, job.stream)
    scn.scn_run_downsample(job.seq, 0, M, buf.data_ptr() + 3, job.stream)
    torch.cuda.synchronize()
    assert (buf.cpu().numpy()[3:3 + nb] == DS.reshape(-1)).all()
    job.close()


def next_rows():
    import paper_1805_07339_b200 as scn
    # N2: stencil before sampling
    w = Workload("sanN2", 48, 20, 2, 30, ("stride", 4), (), spec_kw={"len_min": 3, "len_max": 7})
    job = scn_harness.StencilJob(w, -1)
    out = job.alloc_outputs()
    job.run(out)
    torch.cuda.synchronize()
    ref = oracle.stencil_then_sample(w.spec(), job.part, job.row, -1, w.rows_per_video, 16)
    assert (out["diff"].cpu().numpy().view(np.uint32)[: job.M] == ref).all()
    job.close()
    # N3: adaptive cuts with warmup on a shard
    w = Workload("sanN3", 64, 36, 2, 40, ("stride", 1), (), spec_kw={"len_min": 5, "len_max": 12})
    pl = scn_harness.plan(w)
    M = len(pl[1])
    meta = scn_harness._build_seq(w)
    b, e = M // 2 + 3, M
    wb = scn.scn_seq_warmup_begin(meta, b, 4)
    scn.scn_seq_destroy(meta)
    job = scn_harness.DeviceJob(w, wb, e, with_halo=True, plan_=pl)
    o = job.alloc_outputs(("hist", "shotdiff"), 16)
    job.run(o, ("hist", "shotdiff"), 16)
    c = torch.empty(e - b, dtype=torch.uint8, device="cuda")
    scn.scn_run_adaptive_cuts(job.seq, b, e, 4, o["diff"], 4, 1, 64 * 36 // 8, c)
    torch.cuda.synchronize()
    _, D, _ = oracle.run(w.spec(), pl[0], pl[1], pl[2], 0, M, 16)
    assert (c.cpu().numpy() == oracle.adaptive_cuts(D, pl[2], 4, 4, 1, 64 * 36 // 8)[b:e]).all()
    job.close()
    # N1: montage (aligned and unaligned canvases)
    for ww, cols in ((64, 3), (40, 2)):
        w = Workload("sanN1", ww, 22, 1, 60, ("stride", 1), (), spec_kw={"len_min": 8, "len_max": 20})
        pl = scn_harness.plan(w)
        job = scn_harness.DeviceJob(w, 0, len(pl[1]), with_halo=True, plan_=pl)
        canvas, pos = scn_harness.shot_montage(job, cols, ww * 22)
        ref = oracle.montage(w.spec(), pl[0][pos], pl[1][pos], cols)
        assert (canvas.cpu().numpy() == ref).all()
        job.close()


if __name__ == "__main__":
    main()
