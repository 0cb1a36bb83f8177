"""Input generator sanity (not the method): determinism, modes, gather lists."""
import numpy as np

import scn_synth


def test_deterministic_and_modes():
    sp = scn_synth.Spec(37, 11, seed=1)
    a, b = sp.frame(0, 5), sp.frame(0, 5)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(sp.frame(0, 5), sp.frame(1, 5))
    xg = scn_synth.Spec(300, 2, mode="xgrad").frame(0, 0)
    assert (xg[..., 0] == (np.arange(300) % 256)).all()
    k = scn_synth.Spec(8, 8, mode="constant").frame(0, 3)
    assert (k == k[0, 0]).all()


def test_gather_rows():
    g = scn_synth.gather_rows(1805, 65536, 4096)
    assert len(g) == 4096 and len(set(g.tolist())) == 4096
    assert (np.diff(g) > 0).all() and g[0] >= 0 and g[-1] < 65536
    assert scn_synth.gather_rows(1, 10, 10).tolist() == list(range(10))


def test_shot_alternation():
    sp = scn_synth.Spec(16, 16, seed=3, cuts=[4, 9])
    assert [sp.describe(0, r)["shot"] for r in (0, 3, 4, 8, 9, 20)] == [0, 0, 1, 1, 2, 2]
    assert sp.describe(0, 6)["t"] == 2


def test_weak_scaling_workloads_shard_to_one_config_each():
    # bench.py --scaling weak: at g GPUs each contiguous shard holds exactly one config's positions
    import scn_harness
    import paper_1805_07339_b200 as scn
    for name in ("C2", "C3", "C4", "C5"):
        wl = scn_synth.WORKLOADS[name]
        m1 = len(scn_harness.plan(wl)[1])
        assert wl.weak(1) is wl
        for g in (2, 8):
            w = wl.weak(g)
            _, row, seg = scn_harness.plan(w)
            assert len(row) == g * m1
            for r in range(g):
                b, e = scn.scn_shard_range(len(row), g, r)
                assert e - b == m1
            if wl.n_videos == 1:  # one long film: shard starts are stencil halos, not segment starts
                assert seg.sum() == 1
