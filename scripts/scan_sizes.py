"""Scan launch time vs record count (fixed overhead + per-record cost)."""
import json, sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb
import tracegen
dev = torch.device("cuda:0")
p = tracegen.build_plan("llama")
N = 1 << 30
rec = torch.empty(N, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec, 0, N)
A = len(p.allocs)
tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A)
for b, s in p.allocs:
    tr.register_alloc(b, s)
res = {}
for rows in (False, True):
    for n in [1 << 16, 1 << 20, 1 << 23, 1 << 25, 1 << 27, 1 << 30]:
        ko = torch.tensor([0, n], dtype=torch.int64, device=dev)
        h = tr.histograms(p.page_shift, n_kernels=1, kernel_rows=rows)
        for _ in range(3):
            tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=ko, finalize=False)
        torch.cuda.synchronize()
        tr.reset_timing(); tr.set_timing(True)
        reps = 10
        for _ in range(reps):
            tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=ko, finalize=False)
        ph, _ = tr.timing(); tr.set_timing(False)
        res[f"rows={int(rows)} n={n}"] = round(ph["scan"] / reps * 1e3, 1)
print(json.dumps(res))
