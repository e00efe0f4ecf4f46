"""Read-bandwidth ceiling probe: stream-read a large int64 buffer (same size as the bench
trace) with (a) torch.sum and (b) a trivial TMA-ring read kernel from the scan's own
infrastructure is not available, so (a) and a torch copy are reported."""
import torch, json, sys
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10 * (1 << 30)
x = torch.ones(n, dtype=torch.int64, device="cuda")
res = {}
for name, fn in [("sum_int64", lambda: x.sum()), ("sum_as_fp64", lambda: x.view(torch.float64).sum()),
                 ("amax_int64", lambda: x.amax())]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[name] = {"ms": ms, "GB/s": 8 * n / ms / 1e6}
y = torch.empty(n // 4, dtype=torch.int64, device="cuda")
xs = x[: n // 4]
for _ in range(2):
    y.copy_(xs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    y.copy_(xs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
res["copy_rw"] = {"ms": ms, "GB/s": 2 * 8 * (n // 4) / ms / 1e6}
print(json.dumps(res))
