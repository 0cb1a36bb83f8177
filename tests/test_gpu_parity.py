"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Every stage is integer (u32 counts, u8 pixels), so the bar is exact equality
of every output element. Small cases compare every element;
full-size BASELINE configs (in bench.py's launch configuration) compare
sampled positions one by one against the oracle plus properties that hold at
any size (bin sums = W*H, D = 0 at segment starts, planted cuts)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
import scn_synth
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _oracle_positions(wl):
    vids, rows, seg = [], [], []
    for v in range(wl.n_videos):
        k = wl.sampling[0]
        if k == "stride":
            r = oracle.sample_stride(wl.rows_per_video, wl.sampling[1])
        elif k == "range":
            r = oracle.sample_range(wl.rows_per_video, wl.sampling[1], wl.sampling[2])
        else:
            r = oracle.sample_gather(wl.rows_per_video,
                                     scn_synth.gather_rows(wl.sampling[1], wl.rows_per_video, wl.sampling[2]))
        vids += [v] * len(r)
        rows += r.tolist()
        seg += [1] + [0] * (len(r) - 1) if len(r) else []
    return np.array(vids, np.int32), np.array(rows, np.int64), np.array(seg, np.uint8)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _run(wl, p0, p1, ops, bins, fused=True, spec=None, plan_=None):
    job = scn_harness.DeviceJob(wl, p0, p1, with_halo="shotdiff" in ops, spec=spec, plan_=plan_)
    out = job.alloc_outputs(ops, bins)
    job.run(out, ops, bins, fused=fused)
    torch.cuda.synchronize()
    n = p1 - p0
    res = {}
    if "hist" in ops:
        res["hist"] = _u32(out["hist"])[:n]
    if "shotdiff" in ops:
        res["diff"] = _u32(out["diff"])[:n]
    if "downsample" in ops:
        res["ds"] = out["ds"].cpu().numpy()[:n]
    job.close()
    return res


def test_c1_full_parity_and_planted_cuts():
    wl = scn_synth.WORKLOADS["C1"]
    v, r, s = _oracle_positions(wl)
    pv, pr, ps = scn_harness.plan(wl)
    assert (pr == r).all() and (ps == s).all()
    H, D, _ = oracle.run(wl.spec(), v, r, s, 0, len(r), wl.bins)
    for fused in (True, False):
        got = _run(wl, 0, len(r), ("hist", "shotdiff"), wl.bins, fused=fused)
        np.testing.assert_array_equal(got["hist"], H)
        np.testing.assert_array_equal(got["diff"], D)
    assert set(np.nonzero(got["diff"] > wl.width * wl.height)[0].tolist()) == {57, 131, 198}


SHAPES = [(1, 1), (2, 2), (3, 3), (5, 7), (16, 2), (17, 9), (31, 33), (64, 36), (67, 41), (96, 54), (160, 3),
          (211, 37), (640, 49)]


@pytest.mark.parametrize("w,h", SHAPES)
@pytest.mark.parametrize("bins", [16, 1, 5, 64, 256])
def test_small_shapes_all_ops(w, h, bins):
    wl = Workload("sweep", w, h, 2, 23, ("stride", 2), ("hist", "shotdiff", "downsample"), bins=bins,
                  spec_kw={"len_min": 3, "len_max": 7})
    v, r, s = _oracle_positions(wl)
    H, D, DS = oracle.run(wl.spec(), v, r, s, 0, len(r), bins, want_ds=True)
    got = _run(wl, 0, len(r), ("hist", "shotdiff"), bins)
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["diff"], D)
    got = _run(wl, 0, len(r), ("hist", "downsample"), bins, fused=True)
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["ds"], DS)
    got = _run(wl, 0, len(r), ("downsample",), bins, fused=False)
    np.testing.assert_array_equal(got["ds"], DS)
    got = _run(wl, 0, len(r), ("hist", "downsample", "shotdiff"), bins)  # fused hist+ds, then shot-diff
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["diff"], D)
    np.testing.assert_array_equal(got["ds"], DS)


@pytest.mark.parametrize("mode", ["uniform", "constant", "xgrad", "shots"])
@pytest.mark.parametrize("w,h", [(64, 36), (320, 181), (48, 1)])
def test_content_modes(mode, w, h):
    wl = Workload("modes", w, h, 1, 17, ("stride", 1), ("hist", "shotdiff", "downsample"),
                  spec_kw={"len_min": 4, "len_max": 9})
    spec = wl.spec(mode=mode)
    v, r, s = _oracle_positions(wl)
    H, D, DS = oracle.run(spec, v, r, s, 0, len(r), 16, want_ds=True)
    got = _run(wl, 0, len(r), ("hist", "shotdiff"), 16, spec=spec)
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["diff"], D)
    got = _run(wl, 0, len(r), ("hist", "downsample"), 16, spec=spec)
    np.testing.assert_array_equal(got["ds"], DS)


@pytest.mark.parametrize("sampling", [("range", [(1, 5), (9, 20), (30, 31)], 2), ("gather", 77, 13),
                                      ("stride", 40)])
def test_sampling_kinds_multi_video(sampling):
    wl = Workload("samp", 48, 20, 3, 41, sampling, ("hist", "shotdiff"), spec_kw={"len_min": 2, "len_max": 5})
    v, r, s = _oracle_positions(wl)
    H, D, _ = oracle.run(wl.spec(), v, r, s, 0, len(r), 16)
    got = _run(wl, 0, len(r), ("hist", "shotdiff"), 16)
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["diff"], D)


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_virtual_ranks_sharding_invariance(G):
    # T2: each shard computed alone with its recomputed halo; the concatenation equals the oracle
    wl = Workload("shard", 96, 54, 3, 50, ("stride", 3), ("hist", "shotdiff"), spec_kw={"len_min": 3, "len_max": 8})
    v, r, s = _oracle_positions(wl)
    H, D, _ = oracle.run(wl.spec(), v, r, s, 0, len(r), 16)
    pl = scn_harness.plan(wl)
    hs, ds = [], []
    for rank in range(G):
        b, e = scn.scn_shard_range(len(r), G, rank)
        got = _run(wl, b, e, ("hist", "shotdiff"), 16, plan_=pl)
        hs.append(got["hist"])
        ds.append(got["diff"])
    np.testing.assert_array_equal(np.concatenate(hs), H)
    np.testing.assert_array_equal(np.concatenate(ds), D)


def test_separate_calls_equal_fused_with_halo():
    wl = Workload("halo", 64, 36, 1, 60, ("stride", 1), ("hist", "shotdiff"), spec_kw={"len_min": 5, "len_max": 9})
    pl = scn_harness.plan(wl)
    a = _run(wl, 17, 43, ("hist", "shotdiff"), 16, fused=True, plan_=pl)
    b = _run(wl, 17, 43, ("hist", "shotdiff"), 16, fused=False, plan_=pl)
    np.testing.assert_array_equal(a["hist"], b["hist"])
    np.testing.assert_array_equal(a["diff"], b["diff"])
    v, r, s = _oracle_positions(wl)
    H, D, _ = oracle.run(wl.spec(), v, r, s, 17, 43, 16)
    np.testing.assert_array_equal(a["diff"], D)


def test_absent_row_is_erange():
    wl = Workload("absent", 32, 8, 1, 20, ("stride", 1), ("hist",))
    job = scn_harness.DeviceJob(wl, 5, 10, with_halo=False)
    out = job.alloc_outputs(("hist", "shotdiff"), 16)
    with pytest.raises(scn.ScnError) as e:
        scn.scn_run_histogram(job.seq, 4, 10, 16, out["hist"])
    assert e.value.status == scn.SCN_ERANGE
    with pytest.raises(scn.ScnError) as e:  # the halo (position 4) is absent too
        scn.scn_run_hist_shotdiff(job.seq, 5, 10, 16, out["hist"], out["diff"], out["scratch"])
    assert e.value.status == scn.SCN_ERANGE
    job.close()


def test_empty_and_single():
    wl = Workload("one", 64, 36, 1, 1, ("stride", 5), ("hist", "shotdiff"))
    got = _run(wl, 0, 1, ("hist", "shotdiff"), 16)
    v, r, s = _oracle_positions(wl)
    H, D, _ = oracle.run(wl.spec(), v, r, s, 0, 1, 16)
    np.testing.assert_array_equal(got["hist"], H)
    assert got["diff"].tolist() == [0]
    job = scn_harness.DeviceJob(wl, 0, 1, with_halo=False)
    out = job.alloc_outputs(("hist",), 16)
    scn.scn_run_histogram(job.seq, 0, 0, 16, out["hist"])  # empty range: no-op
    job.close()


def test_host_pipeline_matches_device():
    wl = Workload("e2e", 192, 108, 2, 40, ("stride", 1), ("hist", "shotdiff", "downsample"),
                  spec_kw={"len_min": 5, "len_max": 12})
    pl = scn_harness.plan(wl)
    v, r, s = _oracle_positions(wl)
    for (b, e) in [(0, 80), (13, 61), (41, 42)]:
        H, D, DS = oracle.run(wl.spec(), v, r, s, b, e, 16, want_ds=True)
        hj = scn_harness.HostJob(wl, b, e, with_halo=True, plan_=pl, staging_frames=3)
        dj = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl)
        out = dj.alloc_outputs(("hist", "shotdiff", "downsample"), 16)
        cs = torch.cuda.Stream()
        hj.run(out, ("hist", "shotdiff", "downsample"), 16, stream=torch.cuda.current_stream(), copy_stream=cs)
        torch.cuda.synchronize()
        n = e - b
        np.testing.assert_array_equal(_u32(out["hist"])[:n], H)
        np.testing.assert_array_equal(_u32(out["diff"])[:n], D)
        np.testing.assert_array_equal(out["ds"].cpu().numpy()[:n], DS)
        hj.close()
        dj.close()


def test_plain_c_demo_runs():
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-C", root, "examples/scn_demo"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(root, "examples", "scn_demo")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "scn_demo: ok" in r.stdout


@pytest.mark.parametrize("ops", [("hist",), ("downsample",), ("hist", "downsample"), ("hist", "shotdiff")])
def test_host_pipeline_op_combinations(ops):
    wl = Workload("e2e2", 64, 36, 1, 30, ("stride", 1), ops, spec_kw={"len_min": 4, "len_max": 9})
    pl = scn_harness.plan(wl)
    v, r, s = _oracle_positions(wl)
    H, D, DS = oracle.run(wl.spec(), v, r, s, 7, 30, 16, want_ds=True)
    hj = scn_harness.HostJob(wl, 7, 30, with_halo="shotdiff" in ops, plan_=pl, staging_frames=4)
    dj = scn_harness.DeviceJob(wl, 7, 30, with_halo=False, plan_=pl)
    out = dj.alloc_outputs(("hist", "shotdiff", "downsample"), 16)
    hj.run(out, ops, 16, stream=torch.cuda.current_stream(), copy_stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    n = 23
    if "hist" in ops:
        np.testing.assert_array_equal(_u32(out["hist"])[:n], H)
    if "shotdiff" in ops:
        np.testing.assert_array_equal(_u32(out["diff"])[:n], D)
    if "downsample" in ops:
        np.testing.assert_array_equal(out["ds"].cpu().numpy()[:n], DS)
    hj.close()
    dj.close()


def test_fused_gather_local_destinations():
    # scn_run_hist_shotdiff_to with two local destinations (as ranks' columns): both hold the shard's rows
    wl = Workload("dst", 96, 54, 3, 40, ("stride", 2), ("hist", "shotdiff"), spec_kw={"len_min": 3, "len_max": 9})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    H, D, _ = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 0, M, 16)
    cols = [(torch.full((M, 3, 16), 7, dtype=torch.int32, device="cuda"), torch.full((M,), 7, dtype=torch.int32,
                                                                                      device="cuda"))
            for _ in range(2)]
    scratch = torch.empty(48, dtype=torch.int32, device="cuda")
    for b, e in ((0, M // 2 + 1), (M // 2 + 1, M)):   # two "ranks" in sequence, each writing its rows everywhere
        job = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl)
        scn.scn_run_hist_shotdiff_to(job.seq, b, e, 16, [c[0].data_ptr() for c in cols],
                                     [c[1].data_ptr() for c in cols], 0, scratch)
        torch.cuda.synchronize()
        job.close()
    for h, d in cols:
        np.testing.assert_array_equal(_u32(h), H)
        np.testing.assert_array_equal(_u32(d), D)
    with pytest.raises(scn.ScnError):
        scn.scn_run_hist_shotdiff_to(job.seq, 0, 1, 16, [], [], 0, scratch)


@pytest.mark.parametrize("bins", [2, 3, 5, 7, 8, 12, 15, 17, 100, 128, 255])
@pytest.mark.parametrize("mode", ["uniform", "shots"])
def test_every_bin_kernel_path(bins, mode):
    # bins dividing 16 merge 16-level pair-key bins at the flush; other B < 16 pair SIMD-computed
    # bins (K2b); B > 16 counts raw values and maps them to bins at the flush (K2r) — uniform
    # content reaches every bin edge
    wl = Workload("bins", 211, 37, 2, 12, ("stride", 1), ("hist", "shotdiff"), bins=bins,
                  spec_kw={"len_min": 2, "len_max": 5})
    v, r, s = _oracle_positions(wl)
    spec = wl.spec(mode=mode)
    H, D, _ = oracle.run(spec, v, r, s, 0, len(r), bins)
    got = _run(wl, 0, len(r), ("hist", "shotdiff"), bins, spec=spec)
    np.testing.assert_array_equal(got["hist"], H)
    np.testing.assert_array_equal(got["diff"], D)
    assert scn.scn_hist_variant(bins) == ("tma_pair_lane_private" if 16 % bins == 0 else
                                          "tma_pair_bins_lane_private" if bins < 16 else "tma_raw_lane_private_remap")
