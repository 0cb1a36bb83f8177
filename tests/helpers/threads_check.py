"""Concurrent first use of the C ABI from several host threads in a fresh process
(the library's one-time device-property and tuning init races here): each thread
runs its own job on its own stream; every result must equal the oracle."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import scn_harness  # noqa: E402
from scn_synth import Workload  # noqa: E402


def main():
    torch.cuda.set_device(0)
    specs = [(("hist", "shotdiff"), 16), (("hist", "downsample"), 16), (("hist", "shotdiff"), 256),
             (("downsample",), 16), (("hist", "shotdiff"), 5), (("hist", "downsample", "shotdiff"), 16)]
    wl = Workload("thr", 320, 180, 2, 24, ("stride", 1), (), spec_kw={"len_min": 3, "len_max": 7})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    jobs = []
    for ops, bins in specs:  # allocate and fill up front; the library is first called in the threads
        st = torch.cuda.Stream()
        job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, plan_=pl, stream=st)
        jobs.append((job, job.alloc_outputs(ops, bins), ops, bins, st))
    torch.cuda.synchronize()
    go = threading.Barrier(len(jobs))
    errors = []

    def work(i):
        job, out, ops, bins, st = jobs[i]
        try:
            go.wait()
            job.run(out, ops, bins, stream=st)
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for job, out, ops, bins, st in jobs:
        H, D, DS = oracle.run(wl.spec(), pl[0], pl[1], pl[2], 0, M, bins, want_ds="downsample" in ops)
        if "hist" in ops:
            assert (out["hist"].cpu().numpy().view(np.uint32)[:M] == H).all(), (ops, bins)
        if "shotdiff" in ops:
            assert (out["diff"].cpu().numpy().view(np.uint32)[:M] == D).all(), (ops, bins)
        if "downsample" in ops:
            assert (out["ds"].cpu().numpy()[:M] == DS).all(), (ops, bins)
        job.close()
    print("threads_check ok")


if __name__ == "__main__":
    main()
