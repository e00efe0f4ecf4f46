import sys, ctypes, numpy as np, torch, os
sys.path.insert(0, ".")
os.environ.setdefault("PASTA_LIB", "build/variants/libpasta_tt.so")
import paper_2602_22103_b200 as pb
import tracegen
dev = torch.device("cuda:0")
p = tracegen.build_plan("llama")
for n in [int(x) for x in sys.argv[1:]]:
    rec = torch.empty(n, dtype=torch.int64, device=dev)
    tracegen.device_records(tracegen.DevicePlan(p, dev), rec, 0, n)
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
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"n={n}: start {np.percentile(rel[:,0],[0,50,100]).round(1)} first-data {np.percentile(rel[:,1],[0,50,100]).round(1)} quarter {np.percentile(rel[:,2],[0,50,100]).round(1)} end {np.percentile(rel[:,3],[0,50,100]).round(1)} us")
    del rec
    torch.cuda.empty_cache()
    tr.close()
