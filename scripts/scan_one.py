"""One analyze over the first N records of a config (for ncu): python scripts/scan_one.py N [config] [offset]"""
import sys, torch
sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb
import tracegen
n = int(sys.argv[1]); cfg = sys.argv[2] if len(sys.argv) > 2 else "llama"; j0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
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
tr.set_timing(True)
tr.analyze(rec, p.page_shift, h, kernel_offsets=ko, finalize=False)
print(tr.timing())
