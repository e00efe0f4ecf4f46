"""Per-warp timeline of one scan launch (build with -DPASTA_TRACE_TIMING=1: start, first
slice ready, a quarter of the warp's slices, end; globaltimer ns). usage:
PASTA_LIB=build/variants/libpasta_tt.so python scripts/warp_times.py <config> [warps]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402
dev = torch.device("cuda:0")
cfg = sys.argv[1] if len(sys.argv) > 1 else "rn50"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 24
p = tracegen.build_plan(cfg)
rec = torch.empty(p.n, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec)
A = len(p.allocs)
tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A)
for b, s in p.allocs:
    tr.register_alloc(b, s)
ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.int64)).to(dev)
h = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True)
for _ in range(4):
    h.zero_()
    tr.analyze(rec, p.page_shift, h, kernel_offsets=ko, finalize=False)
torch.cuda.synchronize()
buf = np.zeros(148 * 64 * 4, dtype=np.uint64)
pb._lib.pasta_debug_warp_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
pb._lib.pasta_debug_warp_times(buf.ctypes.data, buf.size)
t = buf[:148 * W * 4].reshape(-1, 4).astype(np.int64)
rel = (t - t[:, 0].min()) / 1000.0
q = [0, 10, 50, 90, 99, 100]
for i, name in enumerate(["start", "first data", "quarter", "end"]):
    print(f"{cfg} {name:10s} us pct{q}: {np.percentile(rel[:, i], q).round(1)}")
# per-SM view: the last warp of each CTA (one CTA per SM) and the spread inside CTAs
endc = rel[:, 3].reshape(-1, W)
print(f"{cfg} per-CTA last end us pct{q}: {np.percentile(endc.max(1), q).round(1)}")
print(f"{cfg} per-CTA (last - first end) us pct{q}: {np.percentile(endc.max(1) - endc.min(1), q).round(1)}")
work = rel[:, 3] - rel[:, 1]
print(f"{cfg} per-warp busy (end - first data) us pct{q}: {np.percentile(work, q).round(1)}")
