"""Raw pinned host -> device copy bandwidth (the e2e path's ceiling); not part of the product."""
import json
import torch

n = 3 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}
for chunk in (64 << 20, 256 << 20, 1 << 30, n):
    for _ in range(2):
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    res[f"h2d_GBps_chunk_{chunk >> 20}MiB"] = 3 * n / (a.elapsed_time(b) / 1e3) / 1e9
print(json.dumps(res))
