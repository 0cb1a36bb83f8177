"""Pins of the oracle's joint-colour histogram (NEXT N4 joint variant; P:L331
"pixel color histogram", reading Q3's alternative; bins per reading Q2): hand-worked golden
values, closed forms for constant frames, a second formulation (numpy.histogramdd with the
bin edges ceil(256 b / J)), the pixel-count invariant, and its marginals equal to the (itself
pinned) per-channel oracle histogram."""
import json
import os

import numpy as np
import pytest

import oracle
import scn_synth
from scn_synth import Workload

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "joint_A.json")


def test_golden_frame_a():
    g = json.load(open(GOLDEN))
    A = np.array(g["A"], dtype=np.uint8)
    for j, nz in g["joint_nonzero"].items():
        h = oracle.hist_joint(A, int(j))
        assert h.shape == (int(j) ** 3,)
        assert {str(k): int(v) for k, v in enumerate(h) if v} == nz


@pytest.mark.parametrize("j", [1, 2, 3, 4, 5, 7, 8, 16])
@pytest.mark.parametrize("rgb", [(0, 0, 0), (255, 255, 255), (17, 128, 200), (64, 63, 192)])
def test_constant_frame_closed_form(j, rgb):
    w, h = 13, 7
    f = np.empty((h, w, 3), np.uint8)
    f[:] = rgb
    out = oracle.hist_joint(f, j)
    k = ((rgb[0] * j // 256) * j + rgb[1] * j // 256) * j + rgb[2] * j // 256
    expect = np.zeros(j ** 3, np.uint32)
    expect[k] = w * h
    np.testing.assert_array_equal(out, expect)


@pytest.mark.parametrize("j", [2, 3, 4, 6, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_histogramdd_and_marginals(j, seed):
    rng = np.random.default_rng(seed)
    f = rng.integers(0, 256, size=(11, 19, 3), dtype=np.uint8)
    out = oracle.hist_joint(f, j)
    # second formulation: bin b of a channel covers v in [ceil(256 b / J), ceil(256 (b+1) / J))
    edges = [-(-256 * b // j) for b in range(j + 1)]
    ref, _ = np.histogramdd(f.reshape(-1, 3).astype(np.float64), bins=[np.array(edges, np.float64)] * 3)
    np.testing.assert_array_equal(out.reshape(j, j, j), ref.astype(np.uint32))
    assert int(out.sum()) == 11 * 19
    # the marginals are the per-channel histograms
    cube = out.reshape(j, j, j).astype(np.int64)
    per = oracle.hist(f, j)
    np.testing.assert_array_equal(cube.sum(axis=(1, 2)), per[0])
    np.testing.assert_array_equal(cube.sum(axis=(0, 2)), per[1])
    np.testing.assert_array_equal(cube.sum(axis=(0, 1)), per[2])


def test_run_joint_matches_per_frame():
    wl = Workload("jr", 33, 9, 2, 6, ("stride", 2), ("hist",), spec_kw={"len_min": 2, "len_max": 3})
    spec = wl.spec()
    import scn_harness  # noqa: F401  (plan through the product's host sampling, as the GPU tests do)
    part, row, seg = scn_harness.plan(wl)
    out = oracle.run_joint(spec, part, row, 0, len(row), 4)
    for p in range(len(row)):
        np.testing.assert_array_equal(out[p], oracle.hist_joint(spec.frame(int(part[p]), int(row[p])), 4))


def test_rejects_bad_bins():
    f = np.zeros((2, 2, 3), np.uint8)
    for j in (0, 17):
        with pytest.raises(oracle.OracleError):
            oracle.hist_joint(f, j)


def _const(rgb, w=5, h=4):
    f = np.empty((h, w, 3), np.uint8)
    f[:] = rgb
    return f


@pytest.mark.parametrize("j", [2, 3, 4, 8])
def test_joint_shotdiff_closed_forms(j):
    # identical frames -> 0; constant frames A -> B -> 2*W*H if their joint bins differ, else 0
    A, B, C = (10, 200, 30), (250, 40, 128), (12, 201, 31)
    hs = np.stack([oracle.hist_joint(_const(x), j) for x in (A, A, B, C, C)])
    d = oracle.shotdiff_joint(hs)
    kk = lambda x: ((x[0] * j // 256) * j + x[1] * j // 256) * j + x[2] * j // 256  # noqa: E731
    expect = [0, 0, 2 * 20 * (kk(A) != kk(B)), 2 * 20 * (kk(B) != kk(C)), 0]
    np.testing.assert_array_equal(d, expect)
    # segment starts clamp to 0
    np.testing.assert_array_equal(oracle.shotdiff_joint(hs, [1, 0, 1, 0, 0]), [0, 0, 0, expect[3], 0])


def test_joint_shotdiff_planted_cuts_c1():
    # C1's three planted cuts move every channel's base colour >= 65 levels, so at J = 4 (64-level
    # bins) nearly every pixel changes joint bin there (D close to its 2*W*H maximum); inside
    # shots D stays far below W*H
    wl = scn_synth.WORKLOADS["C1"]
    import scn_harness
    part, row, seg = scn_harness.plan(wl)
    H, D = oracle.run_joint_diff(wl.spec(), part, row, seg, 0, len(row), 4)
    wh = wl.width * wl.height
    assert set(np.nonzero(D > wh)[0].tolist()) == {57, 131, 198}
    assert (D[[57, 131, 198]] > 1.9 * wh).all() and (D <= 2 * wh).all()
    # the halo: a shard starting inside the film reproduces the full run's values
    H2, D2 = oracle.run_joint_diff(wl.spec(), part, row, seg, 100, len(row), 4)
    np.testing.assert_array_equal(D2, D[100:])
    np.testing.assert_array_equal(H2, H[100:])


@pytest.mark.parametrize("seed", [0, 1])
def test_joint_shotdiff_metric_properties(seed):
    rng = np.random.default_rng(seed)
    fr = [rng.integers(0, 256, size=(6, 7, 3), dtype=np.uint8) for _ in range(3)]
    h = [oracle.hist_joint(f, 4).astype(np.int64) for f in fr]
    l1 = lambda a, b: int(oracle.shotdiff_joint(np.stack([a, b]))[1])  # noqa: E731
    assert l1(h[0], h[1]) == l1(h[1], h[0]) == int(np.abs(h[0] - h[1]).sum())
    assert l1(h[0], h[2]) <= l1(h[0], h[1]) + l1(h[1], h[2])
    assert l1(h[0], h[1]) <= 2 * 6 * 7 and l1(h[0], h[1]) % 2 == 0
