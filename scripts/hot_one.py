"""uvm scan with and without the hotness matrix, one launch each (for ncu)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402

dev = torch.device("cuda:0")
p = tracegen.build_plan("uvm")
rec = torch.empty(p.n, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec)
ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.uint64).view(np.int64).copy()).to(dev)
for wk in (0, 20):
    tr = pb.Trace(dev, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        tr.register_alloc(b, s)
    h = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True, kernel_pages=True, window_kernels=wk)
    tr.analyze(rec, p.page_shift, h, kernel_offsets=ko, finalize=False)
    tr.sync()
    tr.close()
