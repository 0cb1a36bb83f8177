"""Fused result all-gather over peer memory (run under torchrun): every rank maps every
peer's full result columns (CUDA IPC), runs scn_run_hist_shotdiff_to on its shard, and after
a barrier each rank's OWN columns must hold the whole job, bit-identical to a single-process
run and to the oracle at the shard boundaries. Exit 0 = pass."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import paper_1805_07339_b200 as scn  # noqa: E402
import scn_harness  # noqa: E402
from scn_synth import Workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if a.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    wl = Workload("p2p", 320, 180, 9, 90, ("stride", 7), ("hist", "shotdiff"), spec_kw={"len_min": 10, "len_max": 40})
    pl = scn_harness.plan(wl)
    M = len(pl[1])
    cols = scn_harness.PeerColumns(M, wl.bins, dist, dev)
    b, e = scn.scn_shard_range(M, world, rank)
    job = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl, device=dev)
    scratch = torch.empty(3 * wl.bins, dtype=torch.int32, device=dev)
    for _ in range(2):  # twice: the second pass re-zeroes and rewrites the same rows
        scn.scn_run_hist_shotdiff_to(job.seq, b, e, wl.bins, cols.hist_ptrs, cols.diff_ptrs, rank, scratch)
    torch.cuda.synchronize(dev)
    dist.barrier()
    H = cols.hist.cpu().numpy().view(np.uint32)[:M]
    D = cols.diff.cpu().numpy().view(np.uint32)[:M]
    job.close()
    full = scn_harness.DeviceJob(wl, 0, M, with_halo=True, plan_=pl, device=dev)
    fo = full.alloc_outputs(("hist", "shotdiff"), wl.bins)
    full.run(fo, ("hist", "shotdiff"), wl.bins)
    torch.cuda.synchronize(dev)
    ok = bool((fo["hist"].cpu().numpy().view(np.uint32)[:M] == H).all())
    ok &= bool((fo["diff"].cpu().numpy().view(np.uint32)[:M] == D).all())
    for r in range(world):
        pb, _ = scn.scn_shard_range(M, world, r)
        for p in {pb, max(pb - 1, 0)}:
            h, d, _ = oracle.run(wl.spec(), pl[0], pl[1], pl[2], p, p + 1, wl.bins)
            ok &= bool((H[p] == h[0]).all()) and int(D[p]) == int(d[0])
    full.close()
    cols.close()
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32)
    if a.backend == "nccl":
        flag = flag.to(dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    print(f"p2p_check rank={rank} world={world}: {'PASS' if ok else 'FAIL'}", flush=True)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    sys.exit(main())
