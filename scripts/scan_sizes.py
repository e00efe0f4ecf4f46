"""Scan launch time vs record count (fixed overhead + per-record cost).
python scripts/scan_sizes.py [config] [n ...]  (prefixes of the config's trace; one kernel
segment, with and without per-kernel rows; plus the config's own kernel offsets for its full n)"""
import json, sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb
import tracegen
dev = torch.device("cuda:0")
cfg = sys.argv[1] if len(sys.argv) > 1 else "llama"
p = tracegen.build_plan(cfg)
ns = [int(x) for x in sys.argv[2:]] or [1 << 16, 1 << 20, 1 << 23, 1 << 25, 1 << 27, 1 << 30]
N = max(ns)
rec = torch.empty(N, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec, 0, N)
A = len(p.allocs)
tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A)
for b, s in p.allocs:
    tr.register_alloc(b, s)
res = {}
def timeit(n, ko, nk, rows, tag):
    h = tr.histograms(p.page_shift, n_kernels=nk, kernel_rows=rows)
    for _ in range(3):
        tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=ko, finalize=False)
    torch.cuda.synchronize()
    tr.reset_timing(); tr.set_timing(True)
    reps = 10
    for _ in range(reps):
        tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=ko, finalize=False)
    ph, _ = tr.timing(); tr.set_timing(False)
    res[tag] = round(ph["scan"] / reps * 1e3, 1)
    del h
for rows in (False, True):
    for n in ns:
        ko = torch.tensor([0, n], dtype=torch.int64, device=dev)
        timeit(n, ko, 1, rows, f"rows={int(rows)} n={n}")
if N == p.n:
    ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.int64)).to(dev)
    timeit(N, ko, len(p.kernel_offsets) - 1, True, f"kernels={len(p.kernel_offsets) - 1} n={N}")
print(json.dumps(res))
