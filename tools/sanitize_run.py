"""Small workload exercising every kernel once, for compute-sanitizer (T4):
memcheck / racecheck / synccheck must report 0 errors. Also checks parity."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import scn_harness  # noqa: E402
import scn_synth  # noqa: E402
from scn_synth import Workload  # noqa: E402


def check(wl, ops, bins, fused=True, host=False):
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    b, e = M // 3, M
    job = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl)
    out = job.alloc_outputs(ops, bins)
    if host:
        hj = scn_harness.HostJob(wl, b, e, with_halo=True, plan_=pl, staging_frames=2)
        hj.run(out, ops, bins, stream=torch.cuda.current_stream(), copy_stream=torch.cuda.Stream())
    else:
        job.run(out, ops, bins, fused=fused)
    torch.cuda.synchronize()
    H, D, DS = oracle.run(wl.spec(), pl[0], pl[1], pl[2], b, e, bins, want_ds="downsample" in ops)
    n = e - b
    if "hist" in ops:
        assert (out["hist"].cpu().numpy().view(np.uint32)[:n] == H).all()
    if "shotdiff" in ops:
        assert (out["diff"].cpu().numpy().view(np.uint32)[:n] == D).all()
    if "downsample" in ops:
        assert (out["ds"].cpu().numpy()[:n] == DS).all()
    job.close()


def main():
    w1 = Workload("san1", 64, 36, 2, 20, ("stride", 1), (), spec_kw={"len_min": 3, "len_max": 7})
    w2 = Workload("san2", 67, 9, 1, 12, ("stride", 2), (), spec_kw={"len_min": 3, "len_max": 7})
    check(w1, ("hist", "shotdiff"), 16)
    check(w1, ("hist", "shotdiff"), 16, fused=False)
    check(w1, ("hist", "downsample"), 16)
    check(w1, ("downsample",), 16, fused=False)
    check(w2, ("hist", "shotdiff"), 5)
    check(w2, ("hist", "downsample"), 64)
    check(w1, ("hist", "shotdiff", "downsample"), 16, host=True)
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
