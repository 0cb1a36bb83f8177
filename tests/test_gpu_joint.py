"""NEXT N4 joint-colour histogram on the GPU vs the oracle, bit-exact: frame shapes with
ragged pixel tails (W*H % 16 != 0), several tiles per frame, every J in [1, 8], adversarial
content, multi-table sampling, and BASELINE's C2 frames at sampled positions."""
import numpy as np
import pytest
import torch

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
import scn_synth
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _joint(wl, j, mode="shots", p0=0, p1=None):
    pl = scn_harness.plan(wl)
    M = len(pl[1]) if p1 is None else p1
    spec = wl.spec(mode=mode)
    job = scn_harness.DeviceJob(wl, p0, M, with_halo=False, spec=spec, plan_=pl)
    out = torch.empty((max(M - p0, 1), j ** 3), dtype=torch.int32, device="cuda")
    scn.scn_run_histogram_joint(job.seq, p0, M, j, out, job.stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)[: M - p0]
    job.close()
    return got, oracle.run_joint(spec, pl[0], pl[1], p0, M, j)


@pytest.mark.parametrize("j", [1, 2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("w,h", [(1, 1), (3, 5), (16, 1), (17, 9), (64, 36), (67, 41), (211, 37), (640, 49)])
def test_shapes_and_bins(j, w, h):
    wl = Workload("joint", w, h, 2, 9, ("stride", 2), ("hist",), spec_kw={"len_min": 2, "len_max": 4})
    got, ref = _joint(wl, j)
    np.testing.assert_array_equal(got, ref)
    assert (got.sum(axis=1) == w * h).all()


@pytest.mark.parametrize("mode", ["uniform", "constant", "xgrad"])
@pytest.mark.parametrize("j", [4, 8])
def test_content_modes(mode, j):
    wl = Workload("jmode", 320, 181, 1, 5, ("stride", 1), ("hist",), spec_kw={"len_min": 2, "len_max": 3})
    got, ref = _joint(wl, j, mode)
    np.testing.assert_array_equal(got, ref)


def test_c2_frames_sampled_positions():
    wl = scn_synth.WORKLOADS["C2"]
    got, ref = _joint(wl, 8, p0=5000, p1=5012)
    np.testing.assert_array_equal(got, ref)
    # marginals of the joint histogram = the per-channel histograms of the same frames (B = 8)
    pl = scn_harness.plan(wl)
    H, _, _ = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 5000, 5012, 8, want_diff=False)
    cube = got.reshape(-1, 8, 8, 8).astype(np.int64)
    np.testing.assert_array_equal(cube.sum(axis=(2, 3)), H[:, 0])
    np.testing.assert_array_equal(cube.sum(axis=(1, 2)), H[:, 2])


def test_unsupported_bins():
    wl = Workload("jerr", 8, 8, 1, 2, ("stride", 1), ("hist",))
    job = scn_harness.DeviceJob(wl, 0, 2, with_halo=False)
    out = torch.empty((2, 1000), dtype=torch.int32, device="cuda")
    for j in (0, 9):
        with pytest.raises(scn.ScnError) as e:
            scn.scn_run_histogram_joint(job.seq, 0, 2, j, out)
        assert e.value.status == scn.SCN_EUNSUPPORTED
    job.close()


# --- shot-diff over joint-colour histograms (scn_run_hist_shotdiff_joint) ---------------------

def _joint_diff(wl, j, p0, p1, mode="shots", pl=None):
    pl = pl if pl is not None else scn_harness.plan(wl)
    spec = wl.spec(mode=mode)
    job = scn_harness.DeviceJob(wl, p0, p1, with_halo=True, spec=spec, plan_=pl)
    n = p1 - p0
    H = torch.full((max(n, 1), j ** 3), -1, dtype=torch.int32, device="cuda")
    D = torch.full((max(n, 1),), -1, dtype=torch.int32, device="cuda")
    scratch = torch.full((j ** 3,), -1, dtype=torch.int32, device="cuda")
    scn.scn_run_hist_shotdiff_joint(job.seq, p0, p1, j, H, D, scratch, job.stream)
    nl = scn.scn_last_launch_count()
    torch.cuda.synchronize()
    got_h = H.cpu().numpy().view(np.uint32)[:n]
    got_d = D.cpu().numpy().view(np.uint32)[:n]
    job.close()
    ref_h, ref_d = oracle.run_joint_diff(spec, pl[0], pl[1], pl[2], p0, p1, j)
    return got_h, got_d, ref_h, ref_d, nl


@pytest.mark.parametrize("j", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("w,h", [(1, 1), (17, 9), (67, 41), (640, 49)])
def test_joint_shotdiff_shapes(j, w, h):
    wl = Workload("jdiff", w, h, 3, 11, ("stride", 1), ("hist", "shotdiff"), spec_kw={"len_min": 2, "len_max": 4})
    M = len(scn_harness.plan(wl)[1])
    gh, gd, rh, rd, nl = _joint_diff(wl, j, 0, M)
    np.testing.assert_array_equal(gh, rh)
    np.testing.assert_array_equal(gd, rd)
    assert nl == 2  # one histogram launch (memset is not a kernel of ours) + one shot-diff launch


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("j", [3, 4, 8])
def test_joint_shotdiff_virtual_shards(world, j):
    # every shard recomputes its [-1,0] halo; the concatenation equals the single run and the oracle
    wl = Workload("jshard", 96, 54, 2, 13, ("stride", 2), ("hist", "shotdiff"), spec_kw={"len_min": 2, "len_max": 5})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    hs, ds = [], []
    for r in range(world):
        b, e = scn.scn_shard_range(M, world, r)
        gh, gd, rh, rd, _ = _joint_diff(wl, j, b, e, pl=pl)
        np.testing.assert_array_equal(gh, rh)
        np.testing.assert_array_equal(gd, rd)
        hs.append(gh)
        ds.append(gd)
    full_h, full_d, _, _, _ = _joint_diff(wl, j, 0, M, pl=pl)
    np.testing.assert_array_equal(np.concatenate(hs), full_h)
    np.testing.assert_array_equal(np.concatenate(ds), full_d)


def test_joint_shotdiff_c1_planted_cuts():
    wl = scn_synth.WORKLOADS["C1"]
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    gh, gd, rh, rd, _ = _joint_diff(wl, 4, 0, M, pl=pl)
    np.testing.assert_array_equal(gd, rd)
    np.testing.assert_array_equal(gh, rh)
    # the planted cuts move nearly every pixel to another joint bin; inside shots D stays below W*H
    assert set(np.flatnonzero(gd > wl.width * wl.height).tolist()) == {57, 131, 198}


@pytest.mark.parametrize("mode", ["uniform", "constant"])
def test_joint_shotdiff_content_and_c2(mode):
    wl = scn_synth.WORKLOADS["C2"]
    pl = scn_harness.plan(wl)
    gh, gd, rh, rd, _ = _joint_diff(wl, 8, 7001, 7009, mode=mode, pl=pl)
    np.testing.assert_array_equal(gh, rh)
    np.testing.assert_array_equal(gd, rd)


def test_joint_shotdiff_errors():
    wl = Workload("jderr", 8, 8, 1, 4, ("stride", 1), ("hist",))
    job = scn_harness.DeviceJob(wl, 1, 4, with_halo=True)
    H = torch.empty((3, 512), dtype=torch.int32, device="cuda")
    D = torch.empty(3, dtype=torch.int32, device="cuda")
    for j in (0, 9):
        with pytest.raises(scn.ScnError) as e:
            scn.scn_run_hist_shotdiff_joint(job.seq, 1, 4, j, H, D, H)
        assert e.value.status == scn.SCN_EUNSUPPORTED
    with pytest.raises(scn.ScnError) as e:  # position 1 needs its halo: no scratch given
        scn.scn_run_hist_shotdiff_joint(job.seq, 1, 4, 4, H, D, None)
    assert e.value.status == scn.SCN_EINVAL
    scn.scn_run_hist_shotdiff_joint(job.seq, 2, 2, 4, H, D, None)  # empty range: no-op
    job.close()
