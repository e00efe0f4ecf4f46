"""Pins of the oracle's rich-record analysis (NEXT f4; CPU only). DESIGN.md R21-R24.

* brute force: tests/brute.py analyze_rich (linear range scan, page walk) on random
  rich traces with interleaved grid ids, writes, sizes 1-128 and shared-space records;
* SPEC S:366-368 range-filter examples: window [0,0] on a 3-kernel trace keeps only
  kernel 0's accesses; the full window is the identity (equal to the 8-byte analysis
  of the same addresses with the kernels as CSR segments);
* S:372-374 invariants: filter monotonicity and tool-report composability (a filtered
  run equals the full run restricted to the in-range kernels);
* MAX_MEM_REFERENCED_KERNEL: argmax with ties to the lowest kernel.
"""
import random

import numpy as np
import pytest

import oracle
from oracle import OracleTrace
from tests import brute
from tracegen.rich import RICH_DTYPE, rich_host

U64MAX = (1 << 64) - 1


@pytest.fixture(autouse=True)
def _lib(built):
    return built


def _pack(recs):
    out = np.zeros(len(recs), dtype=RICH_DTYPE)
    for i, (a, g, size, w, sh) in enumerate(recs):
        out[i] = (a, g, size, (1 if w else 0) | (2 if sh else 0), 0)
    return out


def _random_rich(rng):
    lo = rng.choice([0, 1 << 40, (1 << 64) - (1 << 17)])
    hi = lo + (1 << 16)
    live = []
    cur = lo + rng.randrange(0, 64)
    for i in range(rng.randint(0, 6)):
        b = cur + (0 if rng.random() < 0.3 else rng.randrange(0, 4096))
        sz = rng.randrange(1, 8192)
        if b + sz >= hi:
            break
        live.append((b, sz, len(live)))
        cur = b + sz
    pts = [lo, hi - 1]
    for b, sz, _ in live:
        pts += [b, b + sz - 1, b + sz, max(lo, b - 1)]
    nk = rng.randint(1, 5)
    recs = []
    for _ in range(rng.randint(0, 150)):
        a = rng.choice(pts) if rng.random() < 0.5 else rng.randrange(lo, hi)
        recs.append((a, rng.randrange(0, nk + 2), 1 << rng.randrange(8), int(rng.random() < 0.3),
                     int(rng.random() < 0.1)))
    g0 = rng.randrange(0, nk)
    g1 = rng.randrange(g0, nk + 1)
    return lo, hi, live, recs, g0, g1


def test_rich_brute_force():
    rng = random.Random(4242)
    for case in range(500):
        lo, hi, live, recs, g0, g1 = _random_rich(rng)
        o = OracleTrace(lo, hi, 8, 8)
        for b, sz, i in live:
            assert o.register_alloc(b, sz) == (oracle.OK, i)
        o.analyze_rich(_pack(recs), g0, g1, 12, kernel_rows=True)
        bf = brute.analyze_rich(live, recs, g0, g1, lo, hi, 12, 8)
        assert o.page_counts.tolist() == bf["page"], case
        assert o.page_writes.tolist() == bf["pw"], case
        assert o.alloc_counts.tolist() == bf["alloc"], case
        assert o.alloc_writes.tolist() == bf["aw"], case
        assert o.alloc_bytes.tolist() == bf["ab"], case
        assert o.kernel_rows.tolist() == bf["kac"] and o.kun.tolist() == bf["kun"], case
        assert o.totals.tolist() == [bf["records"], bf["unattr"], bf["oow"]], case
        assert o.rich_totals.tolist() == [bf["filtered"], bf["shared"], bf["writes"], bf["bytes"]], case
        assert bf["records"] + bf["filtered"] + bf["shared"] == len(recs), case


def _three_kernel_trace():
    base = 1 << 32
    live = [(base, 8192, 0), (base + 16384, 4096, 1)]
    addrs = [base + 8 * i for i in range(100)] + [base + 16384 + 4 * i for i in range(60)] + [base + 12000] * 7
    ko = [0, 100, 160, 167]
    rich = rich_host(np.array(addrs, dtype=np.uint64), ko, seed=9, mix=0.0)
    rich["flags"] &= 1  # no shared-space records here
    return base, live, addrs, ko, rich


def test_spec_window_zero_keeps_only_kernel_zero():
    """window [0,0] on a 3-kernel trace -> only kernel 0's accesses pass."""
    base, live, addrs, ko, rich = _three_kernel_trace()
    o = OracleTrace(base, base + (1 << 20), 4, 4)
    for b, sz, _ in live:
        o.register_alloc(b, sz)
    o.analyze_rich(rich, 0, 0, 12, kernel_rows=True)
    assert int(o.totals[0]) == 100 and int(o.rich_totals[0]) == 67
    assert o.kernel_rows.shape == (1, 4) and o.kernel_rows[0].tolist() == [100, 0, 0, 0]
    assert o.alloc_counts.tolist() == [100, 0, 0, 0]


def test_spec_full_window_is_identity():
    """the full window (and no writes / shared records, size 1) equals the 8-byte
    analysis of the same addresses with the kernels as CSR segments."""
    base, live, addrs, ko, rich = _three_kernel_trace()
    rich["flags"] = 0
    rich["size"] = 1
    a = OracleTrace(base, base + (1 << 20), 4, 4)
    b = OracleTrace(base, base + (1 << 20), 4, 4)
    for bb, sz, _ in live:
        a.register_alloc(bb, sz)
        b.register_alloc(bb, sz)
    a.analyze_rich(rich, 0, 2, 12, kernel_rows=True)
    b.analyze(np.array(addrs, dtype=np.uint64), ko, 12, kernel_rows=True)
    assert np.array_equal(a.page_counts, b.page_counts) and np.array_equal(a.alloc_counts, b.alloc_counts)
    assert np.array_equal(a.kernel_rows, b.kernel_rows) and np.array_equal(a.kun, b.kun)
    assert np.array_equal(a.totals, b.totals)
    assert int(a.rich_totals[3]) == len(addrs) and int(a.rich_totals[2]) == 0


def test_filter_composability_and_monotonicity():
    """a run over grid window [g0, g1] equals the full run restricted to
    kernels g0..g1; narrowing the window never admits more records."""
    rng = random.Random(99)
    for case in range(60):
        lo, hi, live, recs, _, _ = _random_rich(rng)
        gmax = max([g for _, g, _, _, _ in recs] + [0])
        full = OracleTrace(lo, hi, 8, 8)
        for b, sz, _ in live:
            full.register_alloc(b, sz)
        full.analyze_rich(_pack(recs), 0, gmax, 12, kernel_rows=True)
        g0 = rng.randint(0, gmax)
        g1 = rng.randint(g0, gmax)
        part = OracleTrace(lo, hi, 8, 8)
        for b, sz, _ in live:
            part.register_alloc(b, sz)
        part.analyze_rich(_pack(recs), g0, g1, 12, kernel_rows=True)
        assert np.array_equal(part.kernel_rows, full.kernel_rows[g0:g1 + 1]), case
        assert np.array_equal(part.kun, full.kun[g0:g1 + 1]), case
        assert np.array_equal(part.alloc_counts, full.kernel_rows[g0:g1 + 1].sum(axis=0, dtype=np.uint64)), case
        assert int(part.totals[0]) <= int(full.totals[0]), case


def test_max_referenced_kernel():
    """P:443 MAX_MEM_REFERENCED_KERNEL: most analyzed records, ties to the lowest kernel."""
    o = OracleTrace(0, 1 << 20, 2, 2)
    o.register_alloc(0x1000, 0x1000)
    recs = [(0x1000, 0, 4, 0, 0)] * 3 + [(0x5000, 1, 4, 0, 0)] * 5 + [(0x1008, 2, 4, 1, 0)] * 5
    o.analyze_rich(_pack(recs), 0, 2, 12, kernel_rows=True)
    assert o.max_kernel() == 1
    o2 = OracleTrace(0, 1 << 20, 2, 2)
    o2.analyze_rich(_pack([(0x1000, 1, 4, 0, 0)]), 0, 2, 12, kernel_rows=True)
    assert o2.max_kernel() == 1
    o3 = OracleTrace(0, 1 << 20, 2, 2)
    o3.analyze_rich(_pack([]), 0, 2, 12, kernel_rows=True)
    assert o3.max_kernel() == 0


def test_generator_fields():
    """tracegen.rich: sizes in 1..128, grid ids of kernel k or k-1."""
    addr = np.arange(10000, dtype=np.uint64) * 8
    ko = [0, 2500, 5000, 10000]
    r = rich_host(addr, ko, seed=5)
    assert set(np.unique(r["size"]).tolist()) <= {1, 2, 4, 8, 16, 32, 64, 128}
    k = np.searchsorted(np.array(ko), np.arange(10000), side="right") - 1
    d = k - r["grid"].astype(np.int64)
    assert set(np.unique(d).tolist()) <= {0, 1} and np.all(d[k == 0] == 0)
    assert 0.2 < r["flags"].astype(bool).mean() < 0.3
