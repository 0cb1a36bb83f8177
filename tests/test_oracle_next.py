"""Pins for the oracle's NEXT rows.

N2 — stencil before sampling (fig:sampling-e; required set P:L255):
closure fixtures from SPEC S:L131 and SURVEY §8(c), brute-force set
enumeration, the identity with the sample-then-stencil D at stride 1, and
planted cuts that (e) and (f) detect differently."""
import json
import os
import random

import numpy as np
import pytest

import oracle
import scn_synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "next_n2.json")))["closures"],
                         ids=lambda c: c["cite"])
def test_n2_closure_fixtures(case):
    got = oracle.required_rows(case["sampled_rows"], case["offset"], case["n_rows"])
    assert got.tolist() == case["required"]


def test_n2_closure_bruteforce():
    rng = random.Random(55)
    for _ in range(500):
        n = rng.randint(1, 60)
        s = sorted(rng.sample(range(n), rng.randint(0, n)))
        o = rng.randint(-5, 5)
        expect = sorted(set(s) | {min(max(r + o, 0), n - 1) for r in s})
        assert oracle.required_rows(s, o, n).tolist() == expect


def test_n2_equals_sample_then_stencil_at_stride_1():
    sp = scn_synth.Spec(40, 22, seed=12, len_min=4, len_max=9)
    n = 60
    rows = oracle.sample_stride(n, 1)
    d_e = oracle.stencil_then_sample(sp, np.zeros(len(rows), np.int32), rows, -1, n, 16)
    seg = np.zeros(len(rows), np.uint8)
    seg[0] = 1
    _, d_f, _ = oracle.run(sp, np.zeros(len(rows), np.int32), rows, seg, 0, len(rows), 16)
    np.testing.assert_array_equal(d_e, d_f)


def test_n2_planted_cuts_distinguish_e_from_f():
    # C1 content (cuts at rows 57, 131, 198), stride 3: (e) compares S_j with the ORIGINAL
    # previous row, so only sampled rows that are cut rows (57, 198) exceed tau; (f) compares
    # neighbouring SAMPLED rows, so it also fires at 132 (the sample after cut 131).
    wl = scn_synth.WORKLOADS["C1"]
    sp = wl.spec()
    rows = oracle.sample_stride(wl.rows_per_video, 3)
    vids = np.zeros(len(rows), np.int32)
    tau = wl.width * wl.height
    d_e = oracle.stencil_then_sample(sp, vids, rows, -1, wl.rows_per_video, 16)
    assert rows[np.nonzero(d_e > tau)[0]].tolist() == [57, 198]
    seg = np.zeros(len(rows), np.uint8)
    seg[0] = 1
    _, d_f, _ = oracle.run(sp, vids, rows, seg, 0, len(rows), 16)
    assert rows[np.nonzero(d_f > tau)[0]].tolist() == [57, 132, 198]
    assert d_e[0] == 0  # row 0 clamps to itself


# ---------------------------------------------------------------------------
# N3 — bounded-state adaptive cut detector with warmup W
# ---------------------------------------------------------------------------
def test_n3_constant_stream_never_cuts():
    # D[p] > k*mean + c is false for a constant stream when k >= 1, c >= 0
    for w in (1, 4, 16):
        d = np.full(50, 777, np.uint32)
        seg = np.zeros(50, np.uint8)
        seg[0] = 1
        assert oracle.adaptive_cuts(d, seg, w, 3, 2, 0).sum() == 0


def test_n3_spike_closed_form():
    # zeros with one spike X at p: cut exactly at p iff X > floor (mean of zeros is 0);
    # the element after the spike sees the spike in its window and does not fire
    for w in (1, 2, 8):
        for x, floor in ((100, 99), (100, 100), (5, 0)):
            d = np.zeros(40, np.uint32)
            d[20] = x
            seg = np.zeros(40, np.uint8)
            seg[0] = 1
            c = oracle.adaptive_cuts(d, seg, w, 4, 1, floor)
            assert np.nonzero(c)[0].tolist() == ([20] if x > floor else [])


def test_n3_step_and_warmup_window():
    # a step from a to b (b > 4a) fires once; W_eff = min(W, p - s0) and the table start resets state
    d = np.array([10] * 10 + [100] * 10, np.uint32)
    seg = np.zeros(20, np.uint8)
    seg[0] = 1
    c = oracle.adaptive_cuts(d, seg, 3, 4, 1, 0)
    assert np.nonzero(c)[0].tolist() == [10]   # at p=11 the window mean is 40: 100 < 4*40
    seg[10] = 1                               # a new table at 10: no window there -> no cut at 10
    assert oracle.adaptive_cuts(d, seg, 3, 4, 1, 0).sum() == 0
    assert oracle.adaptive_cuts(d[:1], seg[:1], 3, 1, 1, 0).tolist() == [0]  # first element: W_eff = 0


def test_n3_planted_cuts_c1():
    wl = scn_synth.WORKLOADS["C1"]
    v = np.zeros(240, np.int32)
    r = np.arange(240)
    seg = np.zeros(240, np.uint8)
    seg[0] = 1
    _, D, _ = oracle.run(wl.spec(), v, r, seg, 0, 240, 16)
    c = oracle.adaptive_cuts(D, seg, 8, 4, 1, 64 * 36 // 8)
    assert np.nonzero(c)[0].tolist() == [57, 131, 198]


# ---------------------------------------------------------------------------
# N1 — two-job shot montage
# ---------------------------------------------------------------------------
def test_n1_shot_starts_planted():
    wl = scn_synth.WORKLOADS["C1"]
    v, r = np.zeros(240, np.int32), np.arange(240)
    seg = np.zeros(240, np.uint8)
    seg[0] = 1
    _, D, _ = oracle.run(wl.spec(), v, r, seg, 0, 240, 16)
    assert oracle.shot_starts(D, seg, 64 * 36).tolist() == [0, 57, 131, 198]
    seg2 = seg.copy()
    seg2[100] = 1  # a second table starting at 100 starts a shot too
    assert oracle.shot_starts(D, seg2, 64 * 36).tolist() == [0, 57, 100, 131, 198]


@pytest.mark.parametrize("cols", [1, 3, 4, 7])
def test_n1_montage_constant_shots_closed_form(cols):
    # constant-colour shots: each tile is the shot's base colour (downsample of a constant is the
    # constant, reading Q11); cells past the last keyframe stay zero; canvas size is closed-form
    sp = scn_synth.Spec(32, 18, mode="constant", cuts=[5, 9, 14, 20], seed=4)
    rows = np.array([0, 5, 9, 14, 20])
    vids = np.zeros(5, np.int32)
    can = oracle.montage(sp, vids, rows, cols)
    oh, ow = 9, 16
    assert can.shape == (-(-5 // cols) * oh, cols * ow, 3)
    for k, row in enumerate(rows):
        tile = can[(k // cols) * oh:(k // cols + 1) * oh, (k % cols) * ow:(k % cols + 1) * ow]
        base = sp.frame(0, int(row))[0, 0]
        assert (tile == base).all()
    for k in range(5, -(-5 // cols) * cols):
        assert (can[(k // cols) * oh:(k // cols + 1) * oh, (k % cols) * ow:(k % cols + 1) * ow] == 0).all()


def test_n1_montage_tile_is_downsampled_keyframe():
    sp = scn_synth.Spec(48, 20, seed=9, len_min=3, len_max=5)
    rows = np.array([0, 4, 9, 17])
    vids = np.array([0, 0, 1, 1], np.int32)
    can = oracle.montage(sp, vids, rows, 3)
    for k in range(4):
        tile = can[(k // 3) * 10:(k // 3 + 1) * 10, (k % 3) * 24:(k % 3 + 1) * 24]
        np.testing.assert_array_equal(tile, oracle.downsample(sp.frame(int(vids[k]), int(rows[k]))))
