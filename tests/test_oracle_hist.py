"""Pins for the oracle's HIST (readings Q1-Q3, Q13).

Closed forms (constant, x-gradient), the bin-sum invariant, a second
formulation by bin-edge range predicates via numpy.histogram, and the
hand-worked golden fixture."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "frame_A.json")))
CH = "RGB"


def _expect_from_nonzero(nz, bins):
    out = np.zeros((3, bins), dtype=np.uint32)
    for ci, c in enumerate(CH):
        for b, v in nz[c].items():
            out[ci, int(b)] = v
    return out


def test_golden_frame_A():
    A = np.array(GOLD["A"], dtype=np.uint8)
    Z = np.array(GOLD["Z"], dtype=np.uint8)
    np.testing.assert_array_equal(oracle.hist(A, 16), _expect_from_nonzero(GOLD["hist_A_nonzero"], 16))
    np.testing.assert_array_equal(oracle.hist(Z, 16), _expect_from_nonzero(GOLD["hist_Z_nonzero"], 16))
    f3 = np.array(GOLD["frame_3x3"]["pixels"], dtype=np.uint8)
    assert oracle.hist(f3, 16).sum(axis=1).tolist() == GOLD["frame_3x3"]["hist_channel_sums"]


@pytest.mark.parametrize("bins", [1, 2, 3, 7, 16, 17, 64, 100, 255, 256])
def test_constant_frame_closed_form(bins):
    w, h = 13, 7
    for rgb in [(0, 0, 0), (255, 255, 255), (15, 16, 17), (127, 128, 239), (64, 200, 1)]:
        f = np.empty((h, w, 3), dtype=np.uint8)
        f[:] = rgb
        H = oracle.hist(f, bins)
        for c in range(3):
            b = math.floor(rgb[c] * bins / 256)
            expect = np.zeros(bins, dtype=np.uint32)
            expect[b] = w * h
            np.testing.assert_array_equal(H[c], expect)


def _xgrad(w, h):
    f = np.empty((h, w, 3), dtype=np.uint8)
    f[:] = (np.arange(w) % 256).astype(np.uint8)[None, :, None]
    return f


def test_xgradient_closed_form_1080p():
    # v = x mod 256 over 1920x1080 at B=16: bins 0-7 = 128*1080, bins 8-15 = 112*1080
    H = oracle.hist(_xgrad(1920, 1080), 16)
    for c in range(3):
        assert H[c, :8].tolist() == [138240] * 8
        assert H[c, 8:].tolist() == [120960] * 8


@pytest.mark.parametrize("w,h,bins", [(1, 1, 16), (300, 3, 16), (511, 2, 7), (700, 5, 256), (257, 4, 3)])
def test_xgradient_closed_form_general(w, h, bins):
    # count(v) = floor((W-1-v)/256)+1 for v < W, else 0; H[c][b] = h * sum_{bin(v)=b} count(v)
    H = oracle.hist(_xgrad(w, h), bins)
    expect = np.zeros(bins, dtype=np.int64)
    for v in range(256):
        cnt = (w - 1 - v) // 256 + 1 if v < w else 0
        expect[(v * bins) // 256] += cnt * h
    for c in range(3):
        np.testing.assert_array_equal(H[c].astype(np.int64), expect)


@pytest.mark.parametrize("bins", [1, 2, 3, 5, 16, 17, 64, 100, 255, 256])
def test_range_predicate_formulation(bins):
    # bin b covers v in [ceil(256 b / B), ceil(256 (b+1) / B)) -- numpy.histogram with those edges
    rng = np.random.default_rng(bins)
    edges = np.array([-(-256 * b // bins) for b in range(bins + 1)], dtype=np.float64)
    for _ in range(5):
        h, w = rng.integers(1, 40, size=2)
        f = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        H = oracle.hist(f, bins)
        for c in range(3):
            ref, _ = np.histogram(f[..., c].astype(np.float64), bins=edges)
            np.testing.assert_array_equal(H[c], ref.astype(np.uint32))
            assert int(H[c].sum()) == h * w  # bin-sum invariant


def test_bins_out_of_range():
    f = np.zeros((2, 2, 3), dtype=np.uint8)
    for bad in (0, 257):
        with pytest.raises(oracle.OracleError) as e:
            oracle.hist(f, bad)
        assert e.value.code == oracle.EUNSUPPORTED
