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
