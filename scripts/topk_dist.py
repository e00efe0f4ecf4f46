"""Diagnostic: the page-count distribution around the K-th largest count per config
(what the top-K selection has to resolve): nnz, T = K-th largest count, pages in T's
pass-1 float bin (bit length + 5 bits), pages equal to T, pages above T.
    python scripts/topk_dist.py [configs...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402

dev = torch.device("cuda:0")
for name in sys.argv[1:] or ["rn50", "gpt2m", "uvm", "llama", "s_perm", "s_hot", "s_manyranges"]:
    p = tracegen.build_plan(name)
    dp = tracegen.DevicePlan(p, dev)
    rec = torch.empty(p.n, dtype=torch.int64, device=dev)
    tracegen.device_records(dp, rec)
    tr = pb.Trace(dev, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        tr.register_alloc(b, s)
    h = tr.histograms(p.page_shift)
    tr.analyze(rec, p.page_shift, h)
    tr.sync()
    del rec
    c = h.page_counts
    nz = c[c > 0]
    srt = torch.sort(nz, descending=True).values
    for K in p.topk:
        kp = min(K, nz.numel())
        T = int(srt[kp - 1])
        L = T.bit_length()
        if L <= 6:
            lo, hi = T, T
        else:
            sh = L - 6
            lo = (T >> sh) << sh
            hi = lo + (1 << sh) - 1
        inbin = int(((nz >= lo) & (nz <= hi)).sum())
        eq = int((nz == T).sum())
        above = int((nz > hi).sum())
        d = {"config": name, "P": p.n_pages, "nnz": int(nz.numel()), "K": K, "T": T, "bin": [lo, hi],
             "pages_in_bin": inbin, "pages_eq_T": eq, "pages_above_bin": above,
             "distinct_in_bin": int(torch.unique(nz[(nz >= lo) & (nz <= hi)]).numel()),
             "max": int(srt[0])}
        print(json.dumps(d), flush=True)
    tr.close()
    del h, nz, srt
    torch.cuda.empty_cache()
