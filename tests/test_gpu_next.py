"""GPU parity for the NEXT rows vs the oracle, bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import paper_1805_07339_b200 as scn
import scn_harness
import scn_synth
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("sampling,offset", [(("stride", 3), -1), (("stride", 1), -1), (("stride", 7), -2),
                                             (("gather", 9, 40), -1), (("range", [(0, 10), (30, 50)], 4), 1),
                                             (("stride", 5), 0)])
def test_n2_stencil_then_sample(sampling, offset):
    wl = Workload("n2", 96, 54, 3, 120, sampling, ("hist", "shotdiff"), spec_kw={"len_min": 5, "len_max": 30})
    job = scn_harness.StencilJob(wl, offset)
    out = job.alloc_outputs()
    job.run(out)
    torch.cuda.synchronize()
    got = _u32(out["diff"])[: job.M]
    expect = oracle.stencil_then_sample(wl.spec(), job.part, job.row, offset, wl.rows_per_video, wl.bins)
    np.testing.assert_array_equal(got, expect)
    # the materialised required set is exactly the oracle's dependency closure, per table
    # (scn_seq_stencil_required numbers the tables that hold sampled rows 0, 1, ... in order)
    req_part, req_row = scn.scn_seq_rows(job.req)
    total, k = 0, 0
    for v in range(wl.n_videos):
        rows = job.row[job.part == v]
        if len(rows) == 0:
            continue
        expect = oracle.required_rows(rows, offset, wl.rows_per_video)
        np.testing.assert_array_equal(req_row[req_part == k], expect)
        total += len(expect)
        k += 1
    assert job.R == total == len(req_row)
    job.close()


def test_n2_c1_cuts():
    wl = scn_synth.Workload("C1e", 64, 36, 1, 240, ("stride", 3), ("hist", "shotdiff"),
                            spec_kw={"cuts": [57, 131, 198]})
    job = scn_harness.StencilJob(wl, -1)
    out = job.alloc_outputs()
    job.run(out)
    torch.cuda.synchronize()
    d = _u32(out["diff"])[: job.M]
    assert job.row[np.nonzero(d > 64 * 36)[0]].tolist() == [57, 198]
    assert job.R == len(oracle.required_rows(job.row, -1, 240))
    job.close()


def _n3_ref(wl, W, kn, kd, fl):
    part, row, seg = scn_harness.plan(wl)
    _, D, _ = oracle.run(wl.spec(), part, row, seg, 0, len(row), wl.bins)
    return oracle.adaptive_cuts(D, seg, W, kn, kd, fl), len(row)


@pytest.mark.parametrize("W", [1, 4, 16])
@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
def test_n3_adaptive_cuts_sharded_with_warmup(W, G):
    import paper_1805_07339_b200 as scn
    wl = Workload("n3", 64, 36, 3, 70, ("stride", 1), ("hist", "shotdiff"), spec_kw={"len_min": 6, "len_max": 20})
    kn, kd, fl = 4, 1, 64 * 36 // 8
    ref, M = _n3_ref(wl, W, kn, kd, fl)
    pl = scn_harness.plan(wl)
    cuts = []
    for r in range(G):
        b, e = scn.scn_shard_range(M, G, r)
        meta = scn_harness._build_seq(wl)  # metadata-only sequence: where does this shard's warmup start?
        wb = scn.scn_seq_warmup_begin(meta, b, W)
        scn.scn_seq_destroy(meta)
        job = scn_harness.DeviceJob(wl, wb, e, with_halo=True, plan_=pl)
        out = job.alloc_outputs(("hist", "shotdiff"), wl.bins)
        job.run(out, ("hist", "shotdiff"), wl.bins)
        c = torch.empty(max(e - b, 1), dtype=torch.uint8, device="cuda")
        scn.scn_run_adaptive_cuts(job.seq, b, e, W, out["diff"], kn, kd, fl, c)
        torch.cuda.synchronize()
        cuts.append(c.cpu().numpy()[: e - b])
        job.close()
    np.testing.assert_array_equal(np.concatenate(cuts), ref)
    assert ref.sum() >= 3


@pytest.mark.parametrize("w,h,nv,cols", [(64, 36, 1, 2), (40, 22, 2, 3), (96, 54, 3, 5), (100, 31, 1, 4)])
def test_n1_shot_montage(w, h, nv, cols):
    wl = Workload("n1", w, h, nv, 150, ("stride", 1), ("hist", "shotdiff"), spec_kw={"len_min": 20, "len_max": 60})
    pl = scn_harness.plan(wl)
    part, row, seg = pl
    job = scn_harness.DeviceJob(wl, 0, len(row), with_halo=True, plan_=pl)
    canvas, pos = scn_harness.shot_montage(job, cols, w * h)
    _, D, _ = oracle.run(wl.spec(), part, row, seg, 0, len(row), wl.bins)
    ref_pos = oracle.shot_starts(D, seg, w * h)
    assert pos.tolist() == ref_pos.tolist()
    ref = oracle.montage(wl.spec(), part[ref_pos], row[ref_pos], cols)
    np.testing.assert_array_equal(canvas.cpu().numpy(), ref)
    job.close()


def test_n1_montage_c2_prefix():
    wl = scn_synth.WORKLOADS["C2"]
    pl = scn_harness.plan(wl)
    part, row, seg = (x[:1200] for x in pl)
    job = scn_harness.DeviceJob(wl, 0, 1200, with_halo=True, plan_=(part, row, seg))
    canvas, pos = scn_harness.shot_montage(job, 4, wl.width * wl.height)
    cuts = set(wl.spec().cut_rows(0, 1200).tolist())
    assert pos.tolist() == [0] + sorted(cuts)
    ref = oracle.montage(wl.spec(), part[pos], row[pos], 4)
    np.testing.assert_array_equal(canvas.cpu().numpy(), ref)
    job.close()


def test_shot_montage_example_runs(tmp_path):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "m.ppm"
    r = subprocess.run([sys.executable, os.path.join(root, "examples", "shot_montage.py"), "--frames", "600",
                        "--out", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    data = out.read_bytes()
    assert data.startswith(b"P6 ")
    wl = scn_synth.WORKLOADS["C2"]
    n_shots = 1 + len(wl.spec().cut_rows(0, 600))
    assert f"{n_shots} shots" in r.stdout
