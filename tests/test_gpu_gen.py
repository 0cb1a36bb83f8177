"""The realigning row-pair kernels (kVarGen): any frame width (W % 16 != 0, odd W, W < 16)
and any output alignment, for the fused HIST + downsample and the downsample-only calls,
bit-exact against the oracle; bytes outside the output range stay untouched."""
import numpy as np
import pytest
import torch

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _job(w, h, frames, mode="shots"):
    wl = Workload(f"gen{w}x{h}", w, h, 2, frames, ("stride", 1), ("hist", "downsample"),
                  spec_kw={"len_min": 2, "len_max": 5})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    spec = wl.spec(mode=mode)
    H, _, DS = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, 16, want_ds=True)
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=False, spec=spec, plan_=pl)
    return wl, job, M, H, DS


# (1366, 37): the half-lane fused layout (12-row tiles, 16 warps) over 4 tiles, the last one odd
@pytest.mark.parametrize("w,h", [(1366, 24), (1366, 37), (854, 33), (426, 18), (67, 41), (17, 5), (15, 9), (3, 3),
                                 (2, 2), (1920, 17), (33, 64)])
@pytest.mark.parametrize("offset", [0, 1, 2, 4, 5])
def test_unaligned_widths_and_outputs(w, h, offset):
    wl, job, M, H, DS = _job(w, h, 7)
    nbytes = M * (h // 2) * (w // 2) * 3
    for fused in (True, False):
        buf = torch.full((nbytes + 64,), 0xAB, dtype=torch.uint8, device="cuda")
        hist = torch.empty((M, 3, 16), dtype=torch.int32, device="cuda")
        ptr = buf.data_ptr() + offset
        if fused:
            scn.scn_run_hist_downsample(job.seq, 0, M, 16, hist, ptr, job.stream)
        else:
            scn.scn_run_downsample(job.seq, 0, M, ptr, job.stream)
        torch.cuda.synchronize()
        got = buf.cpu().numpy()
        np.testing.assert_array_equal(got[offset:offset + nbytes], DS.reshape(-1), err_msg=f"fused={fused}")
        assert (got[:offset] == 0xAB).all() and (got[offset + nbytes:] == 0xAB).all()
        if fused:
            np.testing.assert_array_equal(hist.cpu().numpy().view(np.uint32), H)
    job.close()


@pytest.mark.parametrize("w,h", [(1366, 768), (854, 480)])
def test_common_unaligned_resolutions_full_frames(w, h):
    wl, job, M, H, DS = _job(w, h, 3, mode="uniform")
    out = job.alloc_outputs(("hist", "downsample"), 16)
    job.run(out, ("hist", "downsample"), 16)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["hist"].cpu().numpy().view(np.uint32)[:M], H)
    np.testing.assert_array_equal(out["ds"].cpu().numpy()[:M], DS)
    job.run(out, ("downsample",), 16, fused=False)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out["ds"].cpu().numpy()[:M], DS)
    job.close()


@pytest.mark.parametrize("w,cols,pad", [(1366, 3, 1), (96, 5, 3), (854, 2, 0)])
def test_montage_unaligned_canvas(w, cols, pad):
    wl, job, M, H, DS = _job(w, 10, 4)
    oh, ow3 = 5, (w // 2) * 3
    pitch = cols * ow3 + pad
    rows = -(-M // cols) * oh
    canvas = torch.full((rows * pitch + 16,), 7, dtype=torch.uint8, device="cuda")
    scn.scn_run_montage(job.seq, 0, M, cols, canvas.data_ptr() + 1, pitch, job.stream)
    torch.cuda.synchronize()
    c = canvas.cpu().numpy()[1:1 + rows * pitch].reshape(rows, pitch)
    for k in range(M):
        r, q = divmod(k, cols)
        np.testing.assert_array_equal(c[r * oh:(r + 1) * oh, q * ow3:(q + 1) * ow3], DS[k].reshape(oh, ow3))
    job.close()


@pytest.mark.parametrize("impl", [1, 2])
@pytest.mark.parametrize("bins", [16, 4, 1])
def test_k2a_impls(impl, bins):
    wl = Workload("k2a", 96, 54, 2, 20, ("stride", 1), ("hist", "shotdiff"), spec_kw={"len_min": 3, "len_max": 6})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    for mode in ("shots", "uniform", "constant"):
        spec = wl.spec(mode=mode)
        H, D, _ = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, bins)
        job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, spec=spec, plan_=pl)
        out = job.alloc_outputs(("hist", "shotdiff"), bins)
        scn.scn_set_hist_impl(impl)
        try:
            job.run(out, ("hist", "shotdiff"), bins)
            torch.cuda.synchronize()
        finally:
            scn.scn_set_hist_impl(0)
        np.testing.assert_array_equal(out["hist"].cpu().numpy().view(np.uint32)[:M], H)
        np.testing.assert_array_equal(out["diff"].cpu().numpy().view(np.uint32)[:M], D)
        job.close()


# Every bin count runs the FUSED hist + downsample kernels: B < 16 not dividing 16 with K2b's pair
# keys of B-level bins (aligned, realigning and half-lane kernels), B > 16 with raw byte keys in the
# split table (aligned and realigning)
@pytest.mark.parametrize("bins", [3, 5, 12, 15, 17, 100, 255, 256])
@pytest.mark.parametrize("w,h", [(64, 36), (640, 49), (1366, 24), (854, 33), (67, 41)])
def test_fused_any_bins(w, h, bins):
    wl, job, M, H16, DS = _job(w, h, 7)
    pl = scn_harness.plan(wl)
    H, _, _ = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 0, M, bins, want_ds=False)
    hist = torch.empty((M, 3, bins), dtype=torch.int32, device="cuda")
    ds = torch.empty((M, h // 2, w // 2, 3), dtype=torch.uint8, device="cuda")
    scn.scn_run_hist_downsample(job.seq, 0, M, bins, hist, ds, job.stream)
    assert scn.scn_last_launch_count() == 1  # one fused pass, not histogram + downsample
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hist.cpu().numpy().view(np.uint32), H)
    np.testing.assert_array_equal(ds.cpu().numpy(), DS)
    job.close()
