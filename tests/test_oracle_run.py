"""Pins for the oracle's whole-job driver (planted cuts, halo/sharding identity).

Planted cuts (reading Q5): the generator guarantees every channel's
base colour moves >= 65 levels (>= 4 bins at B=16) at a cut and only noise
changes within a shot, so the cut set must be exactly {p : D[p] > tau} with
tau = W*H, and also the top-k of D. Sharding (S:L316 determinism; P:L214 halo
as redundant warmup): any split [p0,p1) with its halo equals the full run."""
import numpy as np
import pytest

import oracle
import scn_synth


def _seq(n_videos, rows_per_video, stride=1):
    vids, rows, seg = [], [], []
    for v in range(n_videos):
        r = oracle.sample_stride(rows_per_video, stride)
        vids += [v] * len(r)
        rows += r.tolist()
        seg += [1] + [0] * (len(r) - 1)
    return np.array(vids, np.int32), np.array(rows, np.int64), np.array(seg, np.uint8)


def test_c1_planted_cuts():
    w = scn_synth.WORKLOADS["C1"]
    sp = w.spec()
    v, r, s = _seq(1, w.rows_per_video)
    H, D, _ = oracle.run(sp, v, r, s, 0, len(r), w.bins)
    tau = w.width * w.height
    assert set(np.nonzero(D > tau)[0].tolist()) == {57, 131, 198}
    assert sorted(np.argsort(D)[-3:].tolist()) == [57, 131, 198]
    assert (H.sum(axis=2) == w.width * w.height).all()
    assert D[0] == 0


@pytest.mark.parametrize("w,h", [(96, 54), (64, 36)])
def test_random_shots_detected(w, h):
    sp = scn_synth.Spec(w, h, len_min=48, len_max=240, seed=99)
    v, r, s = _seq(1, 700)
    _, D, _ = oracle.run(sp, v, r, s, 0, len(r), 16)
    cuts = sp.cut_rows(0, 700).tolist()
    assert len(cuts) >= 2
    assert np.nonzero(D > w * h)[0].tolist() == cuts


@pytest.mark.parametrize("bins", [16, 5])
def test_split_with_halo_equals_full(bins):
    sp = scn_synth.Spec(20, 12, len_min=3, len_max=9, seed=5)
    v, r, s = _seq(3, 40, stride=3)
    m = len(r)
    H, D, DS = oracle.run(sp, v, r, s, 0, m, bins, want_ds=True)
    for G in (2, 3, 4, 8):
        parts = [oracle.run(sp, v, r, s, (g * m) // G, ((g + 1) * m) // G, bins, want_ds=True) for g in range(G)]
        np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), H)
        np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), D)
        np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), DS)
    assert (D[s.astype(bool)] == 0).all()


def test_frames_entry_matches_run():
    sp = scn_synth.Spec(33, 17, seed=8, len_min=4, len_max=6)
    v, r, s = _seq(1, 25)
    frames = np.stack([sp.frame(0, int(x)) for x in r])
    H1, D1 = oracle.hist_diff_frames(frames, 16)
    H2, D2, _ = oracle.run(sp, v, r, s, 0, len(r), 16)
    np.testing.assert_array_equal(H1, H2)
    np.testing.assert_array_equal(D1, D2)
    np.testing.assert_array_equal(H1[3], oracle.hist(frames[3], 16))
