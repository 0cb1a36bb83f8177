import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import oracle, paper_1805_07339_b200 as scn, scn_harness
from scn_synth import Workload
w, h, frames, op = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
wl = Workload(f"gen{w}x{h}", w, h, 2, frames, ("stride", 1), ("hist", "downsample"), spec_kw={"len_min": 2, "len_max": 5})
pl = scn_harness.plan(wl); M = len(pl[1])
spec = wl.spec(mode="uniform")
t = time.time(); H, _, DS = oracle.run(spec, pl[0], pl[1], pl[2], 0, M, 16, want_ds=True); print("oracle", time.time() - t, flush=True)
job = scn_harness.DeviceJob(wl, 0, M, with_halo=False, spec=spec, plan_=pl); print("job", flush=True)
out = job.alloc_outputs(("hist", "downsample"), 16)
if op == "fused":
    job.run(out, ("hist", "downsample"), 16)
elif op == "ds":
    job.run(out, ("downsample",), 16, fused=False)
else:
    job.run(out, ("hist",), 16, fused=False)
print("launched", flush=True)
torch.cuda.synchronize(); print("synced", flush=True)
if op != "ds": print("hist ok", (out["hist"].cpu().numpy().view(np.uint32)[:M] == H).all())
if op != "hist": print("ds ok", (out["ds"].cpu().numpy()[:M] == DS).all())
