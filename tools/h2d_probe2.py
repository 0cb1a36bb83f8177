"""Raw pinned host -> device bandwidth with 1, 2 and 4 concurrent copy streams (is the
e2e path's PCIe ceiling per copy engine or per link?). Not part of the product."""
import json

import torch

n = 3 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i, st in enumerate(streams):
            st.wait_event(a)
            with torch.cuda.stream(st):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        b.record()
        torch.cuda.synchronize()
        res[f"h2d_GBps_{ns}_streams"] = max(res.get(f"h2d_GBps_{ns}_streams", 0), n / (a.elapsed_time(b) / 1e3) / 1e9)
print(json.dumps(res))
