"""Which records do the slowest warps hold? (contiguous schedule, PASTA_TRACE_TIMING build)
python scripts/warp_slow.py N [offset] [config]"""
import sys, ctypes, os, numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("PASTA_LIB", "build/variants/libpasta_ic0tt.so")
import paper_2602_22103_b200 as pb
import tracegen
import tracegen.plan as tp
names = {getattr(tp, k): k for k in dir(tp) if k.isupper() and isinstance(getattr(tp, k), int) and getattr(tp, k) < 16}
n = int(sys.argv[1]); j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0; cfg = sys.argv[3] if len(sys.argv) > 3 else "llama"
dev = torch.device("cuda:0")
p = tracegen.build_plan(cfg)
rec = torch.empty(n, dtype=torch.int64, device=dev)
tracegen.device_records(tracegen.DevicePlan(p, dev), rec, j0, j0 + n)
A = len(p.allocs)
tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A)
for b, s in p.allocs:
    tr.register_alloc(b, s)
ko = torch.tensor([0, n], dtype=torch.int64, device=dev)
h = tr.histograms(p.page_shift, n_kernels=1, kernel_rows=True)
for _ in range(3):
    tr.analyze(rec, p.page_shift, h, kernel_offsets=ko, finalize=False)
torch.cuda.synchronize()
buf = np.zeros(148 * 64 * 4, dtype=np.uint64)
pb._lib.pasta_debug_warp_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
pb._lib.pasta_debug_warp_times(buf.ctypes.data, buf.size)
t = buf[:148 * 24 * 4].reshape(-1, 4).astype(np.int64)
dur = (t[:, 3] - t[:, 0]) / 1000.0
W = t.shape[0]
nsl = (n + 255) // 256
starts = np.array([int(r[0]) for r in p.streams] + [p.n])
print(f"n={n} off={j0}: dur us min/med/max {dur.min():.1f} {np.median(dur):.1f} {dur.max():.1f}")
for g in np.argsort(-dur)[:10]:
    s0, s1 = g * nsl // W, (g + 1) * nsl // W
    a, b = j0 + s0 * 256, j0 + s1 * 256
    i0 = np.searchsorted(starts, a, side="right") - 1
    i1 = np.searchsorted(starts, b, side="left")
    kinds = [(names.get(int(p.streams[i][1])), int(min(b, starts[i + 1]) - max(a, starts[i]))) for i in range(i0, i1)]
    print(f"  warp {g}: {dur[g]:.1f} us recs [{a},{b}) streams {kinds[:8]}{' ...' if len(kinds) > 8 else ''}")
    if g == np.argsort(-dur)[0]:
        for i in range(i0, min(i1, i0 + 6)):
            print("     ", int(starts[i]), names.get(int(p.streams[i][1])), [hex(int(x)) for x in p.streams[i][2:]])
