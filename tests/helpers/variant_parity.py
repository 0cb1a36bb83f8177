"""Parity of the CURRENT kernel variant against the oracle on small multi-table workloads
(aligned and unaligned widths, odd heights), every op combination, bin counts that take
the pair-key kernel (1..16) and the raw-value kernel (3, 5, 64, 100, 256). The variant is
the hist impl in SCN_TEST_HIST_IMPL (scn_set_hist_impl) and, with SCN_LIB=tuning, the
measurement build's SCN_* knobs (read once per process). Exit 0 = pass."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1805_07339_b200 as scn  # noqa: E402
import scn_harness  # noqa: E402
import scn_synth  # noqa: E402
from scn_synth import Workload  # noqa: E402


VERBOSE = os.environ.get("SCN_TEST_VERBOSE") == "1"


def main():
    impl = int(os.environ.get("SCN_TEST_HIST_IMPL", "0"))
    scn.scn_set_hist_impl(impl)
    assert os.path.basename(scn.LIB_PATH) == ("libscn_tuning.so" if os.environ.get("SCN_LIB") == "tuning"
                                              else "libscn.so")
    cases = [scn_synth.WORKLOADS["C1"],
             Workload("v1", 96, 54, 2, 30, ("stride", 3), (), spec_kw={"len_min": 3, "len_max": 9}),
             Workload("v2", 67, 41, 2, 20, ("stride", 1), (), spec_kw={"len_min": 3, "len_max": 9}),
             Workload("v3", 640, 49, 1, 9, ("stride", 1), (), spec_kw={"len_min": 2, "len_max": 4}),
             Workload("v4", 854, 30, 1, 6, ("stride", 1), (), spec_kw={"len_min": 2, "len_max": 4})]
    for wl in cases:
        for mode in ("shots", "uniform"):
            spec = wl.spec(mode=mode)
            pl = scn_harness.plan(wl)
            M = len(pl[1])
            H, D, DS = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, wl.bins, want_ds=True)
            job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, spec=spec, plan_=pl)
            out = job.alloc_outputs(("hist", "shotdiff", "downsample"), wl.bins)
            for ops, fused in ((("hist", "shotdiff"), True), (("hist", "downsample"), True), (("downsample",), False)):
                if VERBOSE:
                    print("case", wl.name, mode, ops, flush=True)
                job.run(out, ops, wl.bins, fused=fused)
                torch.cuda.synchronize()
                if "hist" in ops:
                    assert (out["hist"].cpu().numpy().view(np.uint32)[:M] == H).all(), (wl.name, mode, ops)
                if "shotdiff" in ops:
                    assert (out["diff"].cpu().numpy().view(np.uint32)[:M] == D).all(), (wl.name, mode, ops)
                if "downsample" in ops:
                    assert (out["ds"].cpu().numpy()[:M] == DS).all(), (wl.name, mode, ops)
            job.close()
    for bins in (1, 4, 3, 5, 64, 100, 256):
        for wl in cases[1:]:
            for mode in ("shots", "uniform"):
                spec = wl.spec(mode=mode)
                pl = scn_harness.plan(wl)
                M = len(pl[1])
                H, D, _ = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, bins)
                job = scn_harness.DeviceJob(wl, 0, M, with_halo=True, spec=spec, plan_=pl)
                out = job.alloc_outputs(("hist", "shotdiff"), bins)
                if VERBOSE:
                    print("case", wl.name, mode, bins, flush=True)
                job.run(out, ("hist", "shotdiff"), bins)
                torch.cuda.synchronize()
                assert (out["hist"].cpu().numpy().view(np.uint32)[:M] == H).all(), (wl.name, mode, bins)
                assert (out["diff"].cpu().numpy().view(np.uint32)[:M] == D).all(), (wl.name, mode, bins)
                job.close()
    print("variant_parity ok", {k: v for k, v in os.environ.items() if k.startswith("SCN_")}, scn.scn_version())


if __name__ == "__main__":
    main()
