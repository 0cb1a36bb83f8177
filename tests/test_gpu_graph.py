"""The run calls are CUDA-graph capturable (the design uses streams and graphs, not a
tracing compiler): one step captured with torch.cuda.graph and replayed over outputs
poisoned in between must reproduce the oracle bit-exactly, and replaying twice must
give the same result (outputs are zeroed inside the captured step)."""
import numpy as np
import pytest
import torch

import oracle
import scn_harness
from scn_synth import Workload

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("ops", [("hist", "shotdiff"), ("hist", "downsample"), ("hist", "downsample", "shotdiff")])
def test_graph_capture_replay(ops):
    wl = Workload("graph", 640, 360, 2, 40, ("stride", 2), (), spec_kw={"len_min": 3, "len_max": 9})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    H, D, DS = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 0, M, wl.bins, want_ds=True)
    job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, plan_=pl)
    out = job.alloc_outputs(ops, wl.bins)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        job.run(out, ops, wl.bins, stream=s)  # warm-up outside capture (one-time smem opt-in)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        n_launch = job.run(out, ops, wl.bins, stream=s)
    assert n_launch >= 1
    for _ in range(2):
        for v in out.values():
            v.fill_(-1 if v.dtype == torch.int32 else 255)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert (_u32(out["hist"])[:M] == H).all()
        if "shotdiff" in ops:
            assert (_u32(out["diff"])[:M] == D).all()
        if "downsample" in ops:
            assert (out["ds"].cpu().numpy()[:M] == DS).all()
    del g
    job.close()


def test_concurrent_first_use_from_threads():
    # fresh process: the one-time init (device properties, env tuning, smem opt-in) races
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for _ in range(3):
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "helpers", "threads_check.py")],
                           capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        assert "threads_check ok" in r.stdout
