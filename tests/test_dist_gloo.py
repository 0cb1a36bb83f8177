"""World-size 2 and 3 gloo tests (CPU) of the multi-GPU host logic: contiguous
shards (scn_shard_range), the recomputed [-1,0] halo and the
padded all-gather + trim of the result columns (ColumnGather, used by bench.py
with NCCL). Per-rank compute uses the oracle here (no GPU on this box); the
gathered columns must equal the single-process oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
from scn_synth import Workload

WL = Workload("gloo", 24, 10, 3, 31, ("stride", 2), ("hist", "shotdiff"), spec_kw={"len_min": 3, "len_max": 6})


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _positions():
    vids, rows, seg = [], [], []
    for v in range(WL.n_videos):
        r = oracle.sample_stride(WL.rows_per_video, WL.sampling[1])
        vids += [v] * len(r)
        rows += r.tolist()
        seg += [1] + [0] * (len(r) - 1)
    return np.array(vids, np.int32), np.array(rows, np.int64), np.array(seg, np.uint8)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v, r, s = _positions()
        M = len(r)
        b, e = scn.scn_shard_range(M, world, rank)
        # the product's halo decision on a metadata-only sequence must match the segment flags
        part, row, seg = scn_harness.plan(WL)
        assert (row == r).all() and (seg == s).all()
        seq = scn_harness._build_seq(WL)
        halo = scn.scn_seq_needs_halo(seq, b)
        scn.scn_seq_destroy(seq)
        assert halo == (1 if (b > 0 and not s[b]) else 0)
        H, D, _ = oracle.run(WL.spec(), v, r, s, b, e, WL.bins)
        g = scn_harness.ColumnGather(M, world, WL.bins, "cpu", dist)
        g.gather(torch.from_numpy(H.view(np.int32)), torch.from_numpy(D.view(np.int32)), e - b)
        hh, dd = g.result()
        if rank == 0:
            q.put((hh.numpy().view(np.uint32).copy(), dd.numpy().view(np.uint32).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_equals_full(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    v, r, s = _positions()
    H, D, _ = oracle.run(WL.spec(), v, r, s, 0, len(r), WL.bins)
    np.testing.assert_array_equal(got[0], H)
    np.testing.assert_array_equal(got[1], D)
