"""Pins for the oracle's [-1,0] shot-diff (readings Q4-Q7)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "frame_A.json")))


def test_golden_sequence():
    A = np.array(GOLD["A"], dtype=np.uint8)
    Z = np.array(GOLD["Z"], dtype=np.uint8)
    hs = np.stack([oracle.hist(f, 16) for f in (Z, A, A, Z)])
    assert oracle.shotdiff(hs).tolist() == GOLD["diff_sequence_ZAAZ"]
    assert oracle.shotdiff(hs[:2])[1] == GOLD["diff_Z_to_A"]


@pytest.mark.parametrize("bins", [1, 4, 16, 256])
def test_constant_cut_closed_form(bins):
    # constant A then constant B: D = 2*W*H*#{c : bin(A_c) != bin(B_c)}
    rng = np.random.default_rng(bins)
    w, h = 9, 5
    for _ in range(50):
        a, b = rng.integers(0, 256, 3), rng.integers(0, 256, 3)
        fa = np.empty((h, w, 3), np.uint8); fa[:] = a
        fb = np.empty((h, w, 3), np.uint8); fb[:] = b
        d = oracle.shotdiff(np.stack([oracle.hist(fa, bins), oracle.hist(fb, bins)]))
        moved = sum((int(a[c]) * bins) // 256 != (int(b[c]) * bins) // 256 for c in range(3))
        assert d.tolist() == [0, 2 * w * h * moved]


def test_metric_properties():
    # identity, symmetry, triangle inequality of the L1 difference on random triples
    rng = np.random.default_rng(3)
    for _ in range(100):
        fs = [rng.integers(0, 256, size=(4, 6, 3), dtype=np.uint8) for _ in range(3)]
        hs = [oracle.hist(f, 16) for f in fs]
        d = lambda x, y: int(oracle.shotdiff(np.stack([x, y]))[1])
        assert d(hs[0], hs[0]) == 0
        assert d(hs[0], hs[1]) == d(hs[1], hs[0])
        assert d(hs[0], hs[2]) <= d(hs[0], hs[1]) + d(hs[1], hs[2])
        assert d(hs[0], hs[1]) % 2 == 0  # equal pixel counts: moved mass counted twice


def test_segment_start_clamps_to_zero():
    rng = np.random.default_rng(5)
    hs = np.stack([oracle.hist(rng.integers(0, 256, size=(3, 3, 3), dtype=np.uint8), 16) for _ in range(6)])
    seg = [1, 0, 0, 1, 0, 0]
    d = oracle.shotdiff(hs, seg)
    assert d[0] == 0 and d[3] == 0
    assert d[1] > 0 and d[4] > 0
    whole = oracle.shotdiff(hs)
    assert whole[3] > 0  # without the segment boundary the stencil crosses tables
