"""Multi-rank parity check (run under torchrun): every rank materialises only its
shard (+ the recomputed [-1,0] halo), runs HIST + shot-diff through the C
ABI, and the result columns are all-gathered (ColumnGather, as in bench.py).
Rank 0 then recomputes the whole job in one process and compares bit-exactly,
and checks sampled positions against the oracle. Exit code 0 = pass.
Usage: torchrun --nproc-per-node G tests/helpers/dist_check.py [--backend nccl|gloo] [--config NAME] [--frames N]"""
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
import scn_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--config", default="C3small")
    ap.add_argument("--frames", type=int, default=0)
    a = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if a.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    if a.config == "C3small":  # multi-video, stride 30: shard cuts land inside and between videos
        wl = scn_synth.Workload("C3small", 640, 360, 37, 512, ("stride", 30), ("hist", "shotdiff"),
                                spec_kw={"len_min": 171, "len_max": 512})
    else:
        wl = scn_synth.WORKLOADS[a.config]
    pl = scn_harness.plan(wl)
    M = len(pl[1]) if a.frames <= 0 else min(a.frames, len(pl[1]))
    pl = (pl[0][:M], pl[1][:M], pl[2][:M])
    b, e = scn.scn_shard_range(M, world, rank)
    job = scn_harness.DeviceJob(wl, b, e, with_halo=True, plan_=pl, device=dev)
    out = job.alloc_outputs(("hist", "shotdiff"), wl.bins)
    job.run(out, ("hist", "shotdiff"), wl.bins, fused=False)
    g = scn_harness.ColumnGather(M, world, wl.bins, dev, dist)
    g.gather(out["hist"], out["diff"], e - b)
    torch.cuda.synchronize()
    H, D = g.result()
    H = H.cpu().numpy().view(np.uint32)
    D = D.cpu().numpy().view(np.uint32)
    job.close()
    del job, out
    torch.cuda.empty_cache()
    ok = True
    if rank == 0:
        full = scn_harness.DeviceJob(wl, 0, M, with_halo=True, plan_=pl, device=dev)
        fo = full.alloc_outputs(("hist", "shotdiff"), wl.bins)
        full.run(fo, ("hist", "shotdiff"), wl.bins)
        torch.cuda.synchronize()
        ok &= bool((fo["hist"].cpu().numpy().view(np.uint32)[:M] == H).all())
        ok &= bool((fo["diff"].cpu().numpy().view(np.uint32)[:M] == D).all())
        part, row, seg = pl
        for r in range(world):
            pb, _ = scn.scn_shard_range(M, world, r)
            for p in {pb, max(pb - 1, 0)}:
                h, d, _ = oracle.run(wl.spec(), part, row, seg, p, p + 1, wl.bins)
                ok &= bool((H[p] == h[0]).all()) and int(D[p]) == int(d[0])
        print(f"dist_check world={world} backend={a.backend} M={M}: {'PASS' if ok else 'FAIL'}", flush=True)
        full.close()
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    sys.exit(main())
