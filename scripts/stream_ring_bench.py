"""Streaming ring consumer (NEXT f2) throughput for several (batch, slots) settings on one
resident trace (llama prefix): events around open .. close on the trace's stream.
    python scripts/stream_ring_bench.py [records] [batch:slots ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402
from paper_2602_22103_b200.stream import StreamRing  # noqa: E402

DEV = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 31
settings = [tuple(int(x) for x in a.split(":")) for a in sys.argv[2:]] or [(524288, 256)]
p = tracegen.build_plan("llama", 42, n)
rec = torch.empty(p.n, dtype=torch.int64, device=DEV)
tracegen.device_records(tracegen.DevicePlan(p, DEV), rec)
st = torch.cuda.Stream(DEV)
tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs), stream=st)
for b, sz in p.allocs:
    tr.register_alloc(b, sz)
rows = os.environ.get("RING_ROWS", "1") == "1"
h = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=rows)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for batch, slots in settings:
    ring = StreamRing(tr, h, rec, p.kernel_offsets, p.n, batch, p.page_shift, slots=slots)
    ts = []
    import time
    host = []
    for rep in range(4):
        h.zero_()
        torch.cuda.synchronize()
        e0.record(st)
        t0 = time.perf_counter()
        ring.start()
        t1 = time.perf_counter()
        ring.push_all()
        t2 = time.perf_counter()
        e1.record(st)
        ring.destroy()
        st.synchronize()
        t3 = time.perf_counter()
        if rep:
            ts.append(e0.elapsed_time(e1))
            host.append((t1 - t0, t2 - t1, t3 - t2))
    assert int(h.totals[0].item()) == p.n
    t = sum(ts) / len(ts)
    print(json.dumps({"lib": os.environ.get("PASTA_LIB", "default"), "rows": rows, "batch": batch, "slots": slots, "batches": len(ring.batches), "ms": round(t, 3),
                      "us_per_batch": round(t * 1e3 / len(ring.batches), 3), "G_rec_s": round(p.n / t / 1e6, 1),
                      "host_open_push_drain_ms": [round(1e3 * sum(x[i] for x in host) / len(host), 3) for i in range(3)]}),
          flush=True)
