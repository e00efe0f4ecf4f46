"""Host->device bandwidth from pinned memory on this box (the e2e path's bound)."""
import json

import torch

n = 1 << 29  # 4 GiB of int64
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.int64, device="cuda:0")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 0.0
for _ in range(5):
    e0.record()
    d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 8 * n / e0.elapsed_time(e1) / 1e6)
print(json.dumps({"h2d_pinned_GB_s": round(best, 2), "bytes": 8 * n}))
