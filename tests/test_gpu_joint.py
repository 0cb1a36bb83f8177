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
