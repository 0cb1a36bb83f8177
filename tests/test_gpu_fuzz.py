"""Seeded random sweep (T1): random frame shapes (odd sizes, W % 16 == 0 and not, widths
whose rows straddle tiles), bin counts, sampling kinds, table counts, content modes,
shard counts and op combinations, each compared bit-exactly with the oracle. Every case
is derived from its index, so a failure names a reproducible case."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
from scn_synth import Workload

pytestmark = pytest.mark.gpu

BINS = [1, 2, 4, 8, 16, 16, 16, 3, 5, 32, 64, 100, 128, 256]
MODES = ["shots", "shots", "uniform", "constant", "xgrad"]
OPS = [("hist", "shotdiff"), ("hist", "downsample"), ("hist", "downsample", "shotdiff"), ("downsample",),
       ("hist",)]


def _case(i):
    rng = np.random.default_rng(1805_07339 + i)
    w = int(rng.choice([int(rng.integers(1, 80)), 16 * int(rng.integers(1, 48)), 48 * int(rng.integers(1, 30))]))
    h = int(rng.integers(1, 41))
    n_videos = int(rng.integers(1, 4))
    rows = int(rng.integers(0, 30))
    k = rng.integers(0, 3)
    if k == 0:
        sampling = ("stride", int(rng.integers(1, 7)))
    elif k == 1:
        edges = sorted(set(rng.integers(0, rows + 1, 4).tolist())) if rows else [0, 0]
        blocks = [(edges[j], edges[j + 1]) for j in range(0, len(edges) - 1, 2)]
        sampling = ("range", blocks or [(0, 0)], int(rng.integers(1, 4)))
    else:
        sampling = ("gather", int(rng.integers(1, 1 << 30)), int(rng.integers(0, rows + 1)))
    bins = int(rng.choice(BINS))
    mode = str(rng.choice(MODES))
    ops = OPS[int(rng.integers(0, len(OPS)))]
    G = int(rng.choice([1, 1, 2, 3, 5]))
    return w, h, n_videos, rows, sampling, bins, mode, ops, G


N_CASES = int(os.environ.get("SCN_FUZZ_CASES", "160"))  # e.g. 2000 for a long sweep


@pytest.mark.parametrize("i", range(N_CASES))
def test_fuzz_case(i):
    w, h, n_videos, rows, sampling, bins, mode, ops, G = _case(i)
    wl = Workload(f"fuzz{i}", w, h, n_videos, rows, sampling, ops, bins=bins, spec_kw={"len_min": 2, "len_max": 6})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    spec = wl.spec(mode=mode)
    H, D, DS = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, bins, want_ds="downsample" in ops)
    hs, ds_, dss = [], [], []
    for r in range(G):  # G virtual ranks, each shard with its recomputed halo
        b, e = scn.scn_shard_range(M, G, r)
        if e == b:
            continue
        job = scn_harness.DeviceJob(wl, b, e, with_halo="shotdiff" in ops, spec=spec, plan_=pl)
        out = job.alloc_outputs(ops, bins)
        if "downsample" in ops and i % 3 == 1:  # an output buffer at an odd byte offset
            nb = out["ds"].numel()
            raw = torch.empty(nb + 8, dtype=torch.uint8, device=out["ds"].device)
            off = 1 + i % 7
            out["ds"] = raw[off:off + nb].view(out["ds"].shape)
        job.run(out, ops, bins)
        torch.cuda.synchronize()
        n = e - b
        if "hist" in ops:
            hs.append(out["hist"].cpu().numpy().view(np.uint32)[:n])
        if "shotdiff" in ops:
            ds_.append(out["diff"].cpu().numpy().view(np.uint32)[:n])
        if "downsample" in ops:
            dss.append(out["ds"].cpu().numpy()[:n])
        job.close()
    if M == 0:
        return
    if "hist" in ops:
        np.testing.assert_array_equal(np.concatenate(hs), H)
    if "shotdiff" in ops:
        np.testing.assert_array_equal(np.concatenate(ds_), D)
    if "downsample" in ops:
        np.testing.assert_array_equal(np.concatenate(dss), DS)
