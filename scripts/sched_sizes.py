"""Scan time of a config's prefixes (their own kernel offsets, kernel rows) under the
contiguous and the interleaved schedule: where does interleaving start to pay?
python scripts/sched_sizes.py [config] [n ...]   (config default llama; n default: 5 sizes,
or the config's full n when a config is named without sizes)"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402

dev = torch.device("cuda:0")
args = sys.argv[1:]
cfg = args.pop(0) if args and not args[0].isdigit() else None
p = tracegen.build_plan(cfg or "llama")
ns = [int(x) for x in args] or ([p.n] if cfg else [1 << 19, 1 << 22, 1 << 25, 1 << 27, 1 << 29])
N = max(ns)
rec = torch.empty(N, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec, 0, N)
ko_all = np.asarray(p.kernel_offsets, dtype=np.int64)
A = len(p.allocs)
for n in ns:
    k1 = int(np.searchsorted(ko_all, n, side="left"))
    ko = np.concatenate([ko_all[:k1][ko_all[:k1] < n], [n]])
    kod = torch.from_numpy(ko).to(dev)
    out = {"n": n, "kernels": len(ko) - 1}
    for sched in ("contiguous", "interleaved"):
        tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A, schedule=sched)
        for b, s in p.allocs:
            tr.register_alloc(b, s)
        h = tr.histograms(p.page_shift, n_kernels=len(ko) - 1, kernel_rows=True)
        for _ in range(3):
            tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=kod, finalize=False)
        tr.sync()
        reps = 20
        tr.reset_timing()
        tr.set_timing(True)
        for _ in range(reps):
            tr.analyze(rec[:n], p.page_shift, h, kernel_offsets=kod, finalize=False)
        tr.sync()
        ph, _ = tr.timing()
        ms = ph["scan"] / reps
        out[sched + "_us"] = round(ms * 1e3, 2)
        out[sched + "_frac"] = round(8 * n / ms / 1e6 / 6540.2, 3)
        tr.close()
    print(json.dumps(out), flush=True)
