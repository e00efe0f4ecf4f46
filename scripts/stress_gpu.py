"""Randomized GPU-vs-oracle stress beyond the pytest suite (same helpers, other seeds):
scan adversarial cases under both schedules, rich traces, top-K distributions, and
streaming batches (chained launches, odd batch sizes so misaligned heads and odd tails
put the extras kernel inside chains).
python scripts/stress_gpu.py [n_scan] [n_rich] [n_topk] [seed] [n_stream]"""
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from tests import test_gpu_parity as tp  # noqa: E402
from tests import test_gpu_rich as trr  # noqa: E402
from tests.test_oracle_rich import _pack, _random_rich  # noqa: E402

import oracle  # noqa: E402
import paper_2602_22103_b200 as pb  # noqa: E402

n_scan, n_rich, n_topk, seed, n_stream = ([int(x) for x in sys.argv[1:6]] + [200, 200, 100, 7, 50][len(sys.argv) - 1:])[:5]
t0 = time.time()
rng = random.Random(seed)
for i in range(n_scan):
    s = rng.choice([12, 21])
    n = rng.choice([0, 1, 3, 255, 256, 257, 4097, 60001, 250_000, 700_001])
    nr = rng.choice([0, 1, 5, 40, 300, 2000])
    ranges, rec, va_lo, va_hi = tp._adversarial(rng, n, s, nr, near_top=rng.random() < 0.3)
    nk = rng.choice([1, 2, 7, 50, 400])
    cuts = sorted(rng.randint(0, n) for _ in range(nk - 1))
    ko = [0] + cuts + [n]
    sched = rng.choice(tp.SCHEDULES)
    tp._case(ranges, rec, va_lo, va_hi, s, ko=ko, topk=(1, rng.randint(2, 500)), misalign=rng.random() < 0.4,
             label=f"stress scan {i}", window_kernels=rng.choice([0, 1, 3, 7]), schedule=sched)
print(f"scan: {n_scan} cases ok ({time.time() - t0:.0f} s)", flush=True)
for i in range(n_rich):
    lo, hi, live, recs, g0, g1 = _random_rich(rng)
    rec = _pack(recs)
    if rec.size and rng.random() < 0.7:
        rec = np.tile(rec, rng.randint(2, 3000))
    rows = rng.random() < 0.8
    g, o = trr._run(lo, hi, [(b, sz) for b, sz, _ in live], rec, g0, g1, rows=rows)
    trr._assert(g, o, f"stress rich {i}", rows=rows)
print(f"rich: {n_rich} cases ok ({time.time() - t0:.0f} s)", flush=True)
tr = pb.Trace(tp.DEV, 0, 1 << 32, 1, 1)
for i in range(n_topk):
    P = rng.choice([1, 2, 63, 64, 65, 1000, 65537, 1_000_003, 4_000_000])
    kind = rng.randrange(5)
    nrg = np.random.default_rng(rng.randrange(1 << 30))
    if kind == 0:
        c = nrg.integers(0, rng.choice([2, 5, 64, 1 << 20, 1 << 40]), size=P).astype(np.uint64)
    elif kind == 1:
        c = (nrg.geometric(rng.choice([0.5, 0.01, 0.0001]), size=P) - 1).astype(np.uint64)
    elif kind == 2:
        c = np.full(P, rng.randrange(0, 10), dtype=np.uint64)
    elif kind == 3:
        c = nrg.integers(0, 1 << 63, size=P, dtype=np.uint64) >> nrg.integers(0, 63, size=P).astype(np.uint64)
    else:
        c = np.zeros(P, dtype=np.uint64)
        c[nrg.integers(0, P, max(1, P // 100))] = nrg.integers(1, 1 << 30, max(1, P // 100)).astype(np.uint64)
    K = rng.choice([1, 2, 3, 16, 1000, 1024, 1025, 4096, 68266])
    p, cc, f = tr.topk(tp._t(c), K)
    tr.sync()
    rp, rc, rf = oracle.topk(c, K)
    ok = int(tp.u64(f)[0]) == rf and np.array_equal(tp.u64(cc), rc) and np.array_equal(tp.u64(p), rp)
    if not ok:
        print(f"stress topk {i}: P={P} kind={kind} K={K} counts[:8]={c[:8]} found gpu/oracle {int(tp.u64(f)[0])}/{rf}"
              f" gpu pages {tp.u64(p)[:8]} counts {tp.u64(cc)[:8]} oracle pages {rp[:8]} counts {rc[:8]}", flush=True)
        # the same input again, and once more after a fresh handle
        p2, cc2, f2 = tr.topk(tp._t(c), K)
        tr.sync()
        print("  again:", int(tp.u64(f2)[0]), tp.u64(p2)[:8], tp.u64(cc2)[:8], flush=True)
        t2 = pb.Trace(tp.DEV, 0, 1 << 32, 1, 1)
        p3, cc3, f3 = t2.topk(tp._t(c), K)
        t2.sync()
        print("  fresh handle:", int(tp.u64(f3)[0]), tp.u64(p3)[:8], tp.u64(cc3)[:8], flush=True)
        t2.close()
        raise AssertionError(f"stress topk {i}")
tr.close()
print(f"topk: {n_topk} cases ok ({time.time() - t0:.0f} s)", flush=True)

from paper_2602_22103_b200.stream import BatchRunner  # noqa: E402

for i in range(n_stream):
    s = rng.choice([12, 21])
    n = rng.choice([1, 3, 4097, 60001, 250_000, 700_001])
    ranges, rec, va_lo, va_hi = tp._adversarial(rng, n, s, rng.choice([0, 5, 40, 300]), near_top=rng.random() < 0.3)
    nk = rng.choice([1, 2, 7, 50])
    ko = [0] + sorted(rng.randint(0, n) for _ in range(nk - 1)) + [n]
    batch = rng.choice([1, 2, 255, 256, 257, 4095, 4096, 65537])
    tr = tp.gpu_trace(tp.DEV, va_lo, va_hi, ranges)
    h = tr.histograms(s, n_kernels=nk, kernel_rows=True, kernel_pages=True)
    drec = tp._t(np.asarray(rec, dtype=np.uint64))
    runner = BatchRunner(tr, h, drec, np.asarray(ko, dtype=np.int64), n, batch, s, stable=rng.random() < 0.8)
    for _ in range(rng.choice([1, 2])):  # a second pass accumulates on top
        runner.run()
    reps = _ + 1
    tr.finalize(s, h, n_kernels=nk)
    tr.sync()
    o = tp.oracle_trace(va_lo, va_hi, ranges)
    for _ in range(reps):
        o.analyze(np.asarray(rec, dtype=np.uint64), ko, s, kernel_rows=True, kernel_pages=True)
    assert np.array_equal(tp.u64(h.page_counts), o.page_counts), f"stress stream {i}: pages"
    assert np.array_equal(tp.u64(h.alloc_counts), o.alloc_counts), f"stress stream {i}: allocs"
    assert np.array_equal(tp.u64(h.kernel_alloc_counts).reshape(nk, -1), o.kernel_rows), f"stress stream {i}: rows"
    assert tp.u64(h.totals)[:3].tolist() == o.totals.tolist(), f"stress stream {i}: totals"
    tr.close()
print(f"stream: {n_stream} cases ok ({time.time() - t0:.0f} s)", flush=True)
