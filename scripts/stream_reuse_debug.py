"""Debug: the producer-buffer reuse scenario of tests/test_gpu_parity.py with progress prints."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402

DEV = torch.device("cuda:0")
p = tracegen.build_plan("tiny", seed=23)
host = tracegen.host_records(p)
batch, R = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, int(sys.argv[2]) if len(sys.argv) > 2 else 3
bufs = [torch.empty(batch, dtype=torch.int64, device=DEV) for _ in range(R)]
st = torch.cuda.Stream(DEV)
tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs), stream=st)
for b, sz in p.allocs:
    tr.register_alloc(b, sz)
hist = tr.histograms(p.page_shift)
torch.cuda.synchronize()
s = pb.pasta_stream_open(tr.h, p.page_shift, R, batch, hist.struct())
side = torch.cuda.Stream(DEV)
nb = p.n // batch
t00 = time.time()
try:
    for i in range(nb):
        t0 = time.time()
        while pb.pasta_stream_consumed(s) < i - R + 1:
            if time.time() - t0 > 10:
                print(f"stuck at batch {i}: consumed {pb.pasta_stream_consumed(s)}", flush=True)
                raise SystemExit(3)
        buf = bufs[i % R]
        with torch.cuda.stream(side):
            buf.copy_(torch.from_numpy(host[i * batch:(i + 1) * batch].view(np.int64)), non_blocking=False)
        side.synchronize()
        pb.pasta_stream_push(s, [pb.pasta_stream_batch(buf.data_ptr(), batch, None, 1, 0)])
        print(f"pushed {i}, consumed {pb.pasta_stream_consumed(s)}, {time.time() - t00:.3f}s", flush=True)
finally:
    pb.pasta_stream_close(s)
    print("closed", flush=True)
    pb.pasta_stream_destroy(s)
    print("destroyed", flush=True)
tr.sync()
print("totals", hist.totals[:3].tolist(), "expect", nb * batch)
