"""Rich-record scan throughput (NEXT f4): python scripts/rich_bench.py [config] [n] [mix] [block_log2]"""
import json, sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2602_22103_b200 as pb
import tracegen
from tracegen.rich import rich_device
dev = torch.device("cuda:0")
cfg = sys.argv[1] if len(sys.argv) > 1 else "gpt2m"
p = tracegen.build_plan(cfg)
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else p.n
mix = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
blk = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.int64)).to(dev)
rec = torch.empty((n, 2), dtype=torch.int64, device=dev)
dp = tracegen.DevicePlan(p, dev)
step = 1 << 27
tmp = torch.empty(step, dtype=torch.int64, device=dev)
for j0 in range(0, n, step):
    j1 = min(n, j0 + step)
    tracegen.device_records(dp, tmp[:j1 - j0], j0, j1)
    rec[j0:j1] = rich_device(tmp[:j1 - j0], ko, seed=11, j0=j0, mix=mix, block_log2=blk)
del tmp
torch.cuda.synchronize()
kmax = int(np.searchsorted(np.asarray(p.kernel_offsets, dtype=np.int64), n, side="left"))
A = len(p.allocs)
tr = pb.Trace(dev, p.va_lo, p.va_hi, A, A)
for b, s in p.allocs:
    tr.register_alloc(b, s)
h = tr.histograms(p.page_shift, n_kernels=kmax + 1, kernel_rows=True)
rx = tr.rich_outputs(p.page_shift)
for _ in range(3):
    tr.analyze_rich(rec, 0, kmax, p.page_shift, h, rx, finalize=False)
torch.cuda.synchronize()
tr.reset_timing(); tr.set_timing(True)
reps = 5
for _ in range(reps):
    tr.analyze_rich(rec, 0, kmax, p.page_shift, h, rx, finalize=False)
ph, _ = tr.timing()
ms = ph["scan"] / reps
print(json.dumps({"config": cfg, "n": n, "mix": mix, "block_log2": blk, "scan_ms": round(ms, 3), "G_rec_s": round(n / ms / 1e6, 1),
                  "GB_s": round(16 * n / ms / 1e6, 1), "frac_of_6540.8": round(16 * n / ms / 1e6 / 6540.8, 3)}))
