"""Pins of the CPU oracle (oracle/) to things other than itself (CPU only).

* golden hand-worked traces (tests/golden/, each citing the passages it follows);
* SPEC's worked examples;
* closed forms for sweep / permutation / strided traces;
* invariants (conservation, bitmap <=> count > 0, ws <= footprint, top-K order);
* brute force: tests/brute.py (linear scan, dense lists, repeated-max top-K) on
  >= 1000 random tiny traces including adjacent ranges and 2^64 edges;
* special cases that reduce to a library routine (numpy lexsort for top-K with
  K >= nnz; one all-covering range => alloc count = n).
"""
import json
import os
import random

import numpy as np
import pytest

import oracle
from oracle import OracleTrace
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U64MAX = (1 << 64) - 1


@pytest.fixture(autouse=True)
def _lib(built):
    return built


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_hand_worked_trace():
    g = _load("hand_worked.json")
    e = g["expect"]
    o = OracleTrace(g["window"][0], g["window"][1], max_live=8, max_ids=2)
    for base, size in g["ranges"]:
        assert o.register_alloc(base, size)[0] == oracle.OK
    o.analyze(np.array(g["records"], dtype=np.uint64), g["kernel_offsets"], g["page_shift"], kernel_rows=True,
              kernel_pages=True)
    assert o.page_counts.tolist() == e["page_counts"]
    assert int(o.totals[2]) == e["out_of_window"]
    assert o.alloc_counts.tolist() == e["alloc_counts"]
    assert int(o.totals[1]) == e["unattributed"]
    assert int(o.totals[0]) == len(g["records"])
    assert o.kernel_rows.tolist() == e["kernel_alloc_counts"]
    assert o.kun.tolist() == e["kernel_unattributed"]
    bm, u = o.bitmap()
    assert int(bm[0]) == e["bitmap_word0"] and u == e["unique_pages"]
    fp, ws = o.footprints()
    assert fp.tolist() == e["footprint"] and ws == e["ws_obj"]
    assert o.kernel_unique_pages().tolist() == e["kernel_unique_pages"]
    for K, key in ((2, "top2"), (3, "top3")):
        pages, counts, found = o.topk(K)
        assert found == K
        assert [[int(p), int(c)] for p, c in zip(pages, counts)] == e[key]
    pages, counts, found = o.topk(10)
    assert found == e["top10_found"]
    assert [int(pages[found - 1]), int(counts[found - 1])] == e["top10_last_found"]
    assert all(int(p) == U64MAX and int(c) == 0 for p, c in zip(pages[found:], counts[found:]))

    h = g["at_2MiB"]
    o2 = OracleTrace(h["window"][0], h["window"][1], max_live=8, max_ids=2)
    o2.analyze(np.array(g["records"], dtype=np.uint64), None, h["page_shift"])
    assert o2.page_counts.tolist() == h["page_counts"]
    assert int(o2.totals[2]) == h["out_of_window"]
    pages, counts, found = o2.topk(1)
    assert [[int(pages[0]), int(counts[0])]] == h["top1"]


def test_snapshot_sequence():
    g = _load("snapshot_sequence.json")
    o = OracleTrace(g["window"][0], g["window"][1], max_live=8, max_ids=8)
    for step in g["steps"]:
        if step[0] == "register":
            st, i = o.register_alloc(step[1], step[2])
            assert st == step[3]["status"]
            if "id" in step[3]:
                assert i == step[3]["id"]
        elif step[0] == "free":
            assert o.register_free(step[1]) == step[2]["status"]
        else:
            o.analyze(np.array(step[1], dtype=np.uint64), None, g["page_shift"])
    assert o.alloc_counts[:3].tolist() == g["expect"]["alloc_counts"]
    assert int(o.totals[1]) == g["expect"]["unattributed"]
    assert int(o.totals[0]) == g["expect"]["records"]


# ---------------- SPEC worked examples ----------------
def test_spec_granule_example():
    """a 1024 B tensor at rate 1.0 -> 32 accesses of 32 B tiling it; all in one 4 KB page."""
    base = 0x200000
    o = OracleTrace(0, 1 << 30, 4, 4)
    o.register_alloc(base, 1024)
    o.analyze(np.arange(base, base + 1024, 32, dtype=np.uint64), None, 12)
    assert int(o.alloc_counts[0]) == 32
    assert int(o.page_counts[base >> 12]) == 32 and int(o.page_counts.sum()) == 32


def test_spec_merge_identity_and_sum():
    """merge(m, empty) = m; {o1:2} + {o1:3, o2:1} = {o1:5, o2:1} (accumulate = merge)."""
    o = OracleTrace(0, 1 << 24, 4, 4)
    o.register_alloc(0x1000, 0x1000)  # o1
    o.register_alloc(0x4000, 0x1000)  # o2
    o.analyze(np.array([0x1000, 0x1010], dtype=np.uint64), None, 12)
    o.analyze(np.array([], dtype=np.uint64), None, 12)  # merge with the empty map
    assert o.alloc_counts[:2].tolist() == [2, 0]
    o.analyze(np.array([0x1000, 0x1800, 0x1FFF, 0x4000], dtype=np.uint64), None, 12)
    assert o.alloc_counts[:2].tolist() == [5, 1]


def test_spec_partition_fold():
    """a fold over a random partition of the accesses equals the unpartitioned count."""
    from tracegen import build_plan, host_records

    p = build_plan("tiny", seed=7, n=1 << 16)
    rec = host_records(p)
    ko = [int(x) for x in p.kernel_offsets]

    def fresh():
        o = OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
        for b, s in p.allocs:
            o.register_alloc(b, s)
        return o

    whole = fresh()
    whole.analyze(rec, ko, p.page_shift, kernel_rows=True)
    rng = random.Random(3)
    cuts = sorted(rng.sample(range(1, p.n), 5))
    parts = fresh()
    for a, b in zip([0] + cuts, cuts + [p.n]):
        sub = [0] + [min(max(o - a, 0), b - a) for o in ko[1:-1]] + [b - a]
        parts.analyze(rec[a:b], sub, p.page_shift, kernel_rows=True)
    assert np.array_equal(parts.page_counts, whole.page_counts)
    assert np.array_equal(parts.alloc_counts, whole.alloc_counts)
    assert np.array_equal(parts.totals, whole.totals)
    assert np.array_equal(parts.kernel_rows, whole.kernel_rows)


def test_spec_working_set_examples():
    """one kernel touches one 2 MiB object while another is live -> WS = 2 MiB;
    a kernel whose argument objects are {A, B} but which accesses only A -> footprint = size(A)."""
    MiB = 1 << 20
    o = OracleTrace(0, 1 << 30, 4, 4)
    o.register_alloc(2 * MiB, 2 * MiB)  # A
    o.register_alloc(4 * MiB, 2 * MiB)  # B (live, untouched)
    o.analyze(np.array([2 * MiB, 3 * MiB, 4 * MiB - 8], dtype=np.uint64), [0, 3], 21, kernel_rows=True)
    fp, ws = o.footprints()
    assert fp.tolist() == [2 * MiB] and ws == 2 * MiB
    assert sum(o.sizes) == 4 * MiB  # footprint of the live set is 4 MiB


def test_spec_hotness_examples():
    """one access in 2 MiB block 3 -> a single 1; the histogram sums to the access count."""
    MiB = 1 << 20
    o = OracleTrace(0, 64 * MiB, 4, 4)
    o.analyze(np.array([3 * 2 * MiB + 12345], dtype=np.uint64), None, 21)
    assert o.page_counts.tolist() == [0, 0, 0, 1] + [0] * 28
    rng = np.random.default_rng(0)
    a = rng.integers(0, 64 * MiB, size=5000, dtype=np.uint64)
    o2 = OracleTrace(0, 64 * MiB, 4, 4)
    o2.analyze(a, None, 21)
    assert int(o2.page_counts.sum()) == 5000


# ---------------- closed forms ----------------
@pytest.mark.parametrize("passes", [1, 3])
def test_closed_form_sweep(passes):
    """a_j = base + 8*(j mod S/8): every 4 KB page gets 512*R, every 2 MB page 262144*R;
    alloc = R*S/8; unique pages = S/4096; top-K = the K lowest pages (all tie)."""
    MiB = 1 << 20
    base, S = 64 * MiB, 8 * MiB
    n = passes * S // 8
    a = (base + 8 * (np.arange(n, dtype=np.uint64) % np.uint64(S // 8))).astype(np.uint64)
    for s, per in ((12, 512), (21, 262144)):
        o = OracleTrace(0, 256 * MiB, 2, 2)
        o.register_alloc(base, S)
        o.analyze(a, None, s)
        nz = o.page_counts[o.page_counts > 0]
        assert nz.size == S >> s and np.all(nz == per * passes)
        assert int(o.alloc_counts[0]) == passes * S // 8
        bm, u = o.bitmap()
        assert u == S >> s
        K = min(5, S >> s)
        pages, counts, found = o.topk(K)
        first = base >> s
        assert found == K and pages.tolist() == [first + i for i in range(K)]


def test_closed_form_permutation():
    """base + 8*((alpha*j + c) mod M), M a power of two, alpha odd: bijective per pass,
    so counts equal the sweep's."""
    MiB = 1 << 20
    base, S = 64 * MiB, 4 * MiB
    M = S // 8
    j = np.arange(2 * M, dtype=np.uint64)
    a = base + np.uint64(8) * ((np.uint64(0x9E3779B1) * j + np.uint64(12345)) & np.uint64(M - 1))
    o = OracleTrace(0, 256 * MiB, 2, 2)
    o.register_alloc(base, S)
    o.analyze(a.astype(np.uint64), None, 12)
    nz = o.page_counts[o.page_counts > 0]
    assert nz.size == S // 4096 and np.all(nz == 2 * 512)


def test_closed_form_strided():
    """base + (j*2^t mod S), t >= 12, R passes: every 2^(t-12)-th 4 KB page gets exactly R;
    unique pages = S/2^t; all other pages 0."""
    MiB = 1 << 20
    base, S, t, R = 64 * MiB, 8 * MiB, 14, 5
    n = R * S // (1 << t)
    a = base + ((np.arange(n, dtype=np.uint64) << np.uint64(t)) % np.uint64(S))
    o = OracleTrace(0, 256 * MiB, 2, 2)
    o.register_alloc(base, S)
    o.analyze(a.astype(np.uint64), None, 12)
    first = base >> 12
    stride = 1 << (t - 12)
    expect = np.zeros_like(o.page_counts)
    expect[first:first + S // 4096:stride] = R
    assert np.array_equal(o.page_counts, expect)
    assert o.bitmap()[1] == S >> t


def test_one_covering_range_counts_everything():
    rng = np.random.default_rng(1)
    a = rng.integers(0, U64MAX, size=4000, dtype=np.uint64, endpoint=False)
    o = OracleTrace(0, 1 << 21, 2, 2)
    o.register_alloc(0, U64MAX)  # [0, 2^64 - 1)
    o.analyze(a, None, 12)
    assert int(o.alloc_counts[0]) == int(np.sum(a != np.uint64(U64MAX)))


def test_topk_equals_full_stable_sort():
    rng = np.random.default_rng(2)
    pc = rng.integers(0, 6, size=3000).astype(np.uint64)
    order = np.lexsort((np.arange(pc.size), -pc.astype(np.int64)))  # count desc, page asc
    order = [int(i) for i in order if pc[i] > 0]
    pages, counts, found = oracle.topk(pc, 5000)
    assert found == len(order)
    assert pages[:found].tolist() == order
    assert counts[:found].tolist() == pc[order].tolist()


# ---------------- invariants on generated traces ----------------
@pytest.mark.parametrize("seed", [42, 7, 0, 1])
def test_invariants_tiny(seed):
    from tracegen import build_plan, host_records

    p = build_plan("tiny", seed=seed)
    rec = host_records(p)
    o = OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        o.register_alloc(b, s)
    o.analyze(rec, p.kernel_offsets, p.page_shift, kernel_rows=True, kernel_pages=True)
    n = p.n
    assert int(o.totals[0]) == n
    assert int(o.page_counts.sum()) + int(o.totals[2]) == n
    assert int(o.alloc_counts.sum()) + int(o.totals[1]) == n
    assert np.array_equal(o.kernel_rows.sum(axis=0), o.alloc_counts)
    assert int(o.kun.sum()) == int(o.totals[1])
    bm, u = o.bitmap()
    bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[: o.page_counts.size]
    assert np.array_equal(bits.astype(bool), o.page_counts > 0)
    assert u <= o.page_counts.size
    fp, ws = o.footprints()
    assert ws == int(fp.max()) and int(fp.max()) <= sum(s for _, s in p.allocs)
    kup = o.kernel_unique_pages()
    assert int(kup.max()) <= u
    pages, counts, found = o.topk(16)
    assert found == 16
    c = counts.astype(np.int64)
    assert np.all(c[:-1] >= c[1:])
    for i in range(found - 1):
        if counts[i] == counts[i + 1]:
            assert pages[i] < pages[i + 1]
    # generator: strays are the only unattributed records and the only out-of-window ones
    assert int(o.totals[1]) > 0 and int(o.totals[2]) > 0


# ---------------- brute force ----------------
def _random_case(rng: random.Random):
    edge = rng.random() < 0.25
    s = rng.choice([12, 21])
    npg = rng.randint(1, 40)
    if edge:
        va_hi = (U64MAX >> 21 << 21)  # highest 2 MiB-aligned end representable
        va_lo = va_hi - (npg << s)
    else:
        va_lo = rng.randrange(0, 1 << 30) << 21
        va_hi = va_lo + (npg << s)
    span_lo = max(0, va_lo - (2 << s))
    span_hi = min(U64MAX, va_hi + (2 << s))
    live = []
    nr = rng.randint(0, 8)
    cursor = span_lo + rng.randrange(0, 1 << s)
    for i in range(nr):
        if rng.random() < 0.5 and live:
            base = live[-1][0] + live[-1][1]  # adjacent to the previous range
        else:
            base = cursor + rng.randrange(0, 3 << (s - 2))
        size = rng.randrange(1, 3 << (s - 1))
        if base + size > U64MAX:
            break
        live.append((base, size, len(live)))
        cursor = base + size
    pts = [span_lo, span_hi, 0, U64MAX, va_lo, va_hi, va_lo - 1 if va_lo else 0, va_hi - 1]
    for b, sz, _ in live:
        pts += [b - 1 if b else 0, b, b + sz - 1, b + sz]
    n = rng.randint(0, 64)
    recs = []
    for _ in range(n):
        if rng.random() < 0.5:
            recs.append(min(U64MAX, max(0, rng.choice(pts))))
        else:
            recs.append(rng.randrange(span_lo, span_hi + 1))
    nk = rng.randint(1, 3)
    cuts = sorted(rng.randint(0, n) for _ in range(nk - 1))
    ko = [0] + cuts + [n]
    return live, recs, ko, va_lo, va_hi, s


def test_brute_force_agreement():
    rng = random.Random(2024)
    for case in range(1200):
        live, recs, ko, va_lo, va_hi, s = _random_case(rng)
        max_ids = max(1, len(live))
        o = OracleTrace(va_lo, va_hi, 16, max_ids)
        for b, sz, i in live:
            st, got = o.register_alloc(b, sz)
            assert st == oracle.OK and got == i, (case, b, sz)
        wk = rng.randint(1, 3)
        o.analyze(np.array(recs, dtype=np.uint64), ko, s, kernel_rows=True, kernel_pages=True, window_kernels=wk)
        bf = brute.analyze(live, recs, ko, va_lo, va_hi, s, max_ids, window_kernels=wk)
        assert o.hotness.tolist() == bf["hot"], case
        assert o.page_counts.tolist() == bf["page"], case
        assert o.alloc_counts.tolist() == bf["alloc"], case
        assert o.kernel_rows.tolist() == bf["kac"], case
        assert o.kun.tolist() == bf["kun"], case
        assert int(o.totals[1]) == bf["unattr"] and int(o.totals[2]) == bf["oow"], case
        bm, u = o.bitmap()
        assert bm.tolist() == brute.bitmap_words(bf["page"]), case
        assert u == sum(1 for c in bf["page"] if c), case
        sizes = [sz for _, sz, _ in live] or [0]
        fp, ws = o.footprints()
        bfp = brute.footprints(bf["kac"], sizes)
        assert fp.tolist() == bfp and ws == max(bfp), case
        assert o.kernel_unique_pages().tolist() == [sum(r) for r in bf["kpages"]], case
        K = rng.randint(1, 12)
        pages, counts, found = o.topk(K)
        bt, bfound = brute.topk(bf["page"], K)
        assert found == bfound, case
        assert [(int(p), int(c)) for p, c in zip(pages, counts)] == bt, case


def test_registration_errors():
    o = OracleTrace(0, 1 << 30, max_live=2, max_ids=3)
    assert o.register_alloc(0x1000, 0)[0] == oracle.EINVAL
    assert o.register_alloc(U64MAX - 4, 8)[0] == oracle.EINVAL
    assert o.register_alloc(0x1000, 0x1000) == (oracle.OK, 0)
    assert o.register_alloc(0x1FFF, 1)[0] == oracle.EOVERLAP
    assert o.register_alloc(0x0800, 0x801)[0] == oracle.EOVERLAP
    assert o.register_alloc(0x2000, 0x10) == (oracle.OK, 1)  # adjacent is legal
    assert o.register_alloc(0x3000, 0x10)[0] == oracle.ECAPACITY  # max_live = 2
    assert o.register_free(0x2008) == oracle.ENOENT
    assert o.register_free(0x2000) == oracle.OK
    assert o.register_alloc(0x3000, 0x10) == (oracle.OK, 2)
    assert o.register_free(0x3000) == oracle.OK
    assert o.register_alloc(0x3000, 0x10)[0] == oracle.ECAPACITY  # max_ids = 3, ids never reused


# ---------------- time-windowed hotness (NEXT f1) ----------------
def test_spec_hotness_matrix_examples():
    """one access at block 3 in window 0 -> a matrix with a single 1; the matrix
    sums to the in-window access count; a persistent tensor's block row has no zero window
    while a transient burst's row is zero outside its burst."""
    MiB = 1 << 20
    o = OracleTrace(0, 64 * MiB, 4, 4)
    o.analyze(np.array([3 * 2 * MiB + 5], dtype=np.uint64), [0, 1, 1], 21, kernel_rows=True, window_kernels=1)
    assert o.hotness.shape == (2, 32)
    assert int(o.hotness.sum()) == 1 and int(o.hotness[0, 3]) == 1
    # 10 kernels: block 1 (weights) read in every kernel, block 7 (a transient buffer) in kernels 3-4
    rec, ko = [], [0]
    for k in range(10):
        rec += [1 * 2 * MiB + 64 * i for i in range(50)]
        if k in (3, 4):
            rec += [7 * 2 * MiB + 8 * i for i in range(200)]
        rec += [100 * MiB + 8]  # out of window: not in the matrix
        ko.append(len(rec))
    o2 = OracleTrace(0, 64 * MiB, 4, 4)
    o2.analyze(np.array(rec, dtype=np.uint64), ko, 21, kernel_rows=True, window_kernels=1)
    h = o2.hotness
    assert np.all(h[:, 1] == 50)
    assert h[3, 7] == 200 and h[4, 7] == 200 and int(h[:, 7].sum()) == 400
    assert int(h.sum()) == len(rec) - 10
    # windows of 3 kernels sum rows of the per-kernel matrix
    o3 = OracleTrace(0, 64 * MiB, 4, 4)
    o3.analyze(np.array(rec, dtype=np.uint64), ko, 21, kernel_rows=True, window_kernels=3)
    assert o3.hotness.shape == (4, 32)
    for w in range(4):
        assert np.array_equal(o3.hotness[w], h[3 * w:3 * w + 3].sum(axis=0))


# ---------------- chunk-parallel oracle (full-size parity, all-core cpu_baseline) ----------------
def test_parallel_oracle_brute_force():
    """analyze_parallel (kernel-aligned slabs on worker threads, per-thread arrays summed:
    the S:291-299 partition fold) against the dumb brute force, slab = 1 record so every
    kernel is its own slab and several threads share each trace."""
    rng = random.Random(77)
    for case in range(300):
        live, recs, ko, va_lo, va_hi, s = _random_case(rng)
        nk = rng.randint(1, 9)
        n = len(recs)
        ko = [0] + sorted(rng.randint(0, n) for _ in range(nk - 1)) + [n]
        max_ids = max(1, len(live))
        o = OracleTrace(va_lo, va_hi, 16, max_ids)
        for b, sz, _ in live:
            o.register_alloc(b, sz)
        o.analyze_parallel(np.array(recs, dtype=np.uint64), ko, s, kernel_rows=True, kernel_pages=True,
                           threads=rng.randint(1, 4), slab=1)
        bf = brute.analyze(live, recs, ko, va_lo, va_hi, s, max_ids)
        assert o.page_counts.tolist() == bf["page"], case
        assert o.alloc_counts.tolist() == bf["alloc"], case
        assert o.kernel_rows.tolist() == bf["kac"], case
        assert o.kun.tolist() == bf["kun"], case
        assert int(o.totals[0]) == n and int(o.totals[1]) == bf["unattr"] and int(o.totals[2]) == bf["oow"], case
        assert o.kernel_unique_pages().tolist() == [sum(r) for r in bf["kpages"]], case


@pytest.mark.parametrize("threads,slab", [(1, 1 << 24), (3, 50_000), (8, 1)])
def test_parallel_oracle_equals_serial_tiny(threads, slab):
    """The tiny BASELINE config: analyze_parallel with records given by a generator
    callback equals the single-thread analyze on the whole array, every output; and two
    calls accumulate like the serial oracle."""
    import tracegen

    p = tracegen.build_plan("tiny", seed=5)
    rec = tracegen.host_records(p)
    ser = OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    par = OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, sz in p.allocs:
        ser.register_alloc(b, sz)
        par.register_alloc(b, sz)
    for _ in range(2):
        ser.analyze(rec, p.kernel_offsets, p.page_shift, kernel_rows=True, kernel_pages=True)
        par.analyze_parallel(lambda j0, j1: tracegen.host_records(p, j0, j1), p.kernel_offsets, p.page_shift,
                             kernel_rows=True, kernel_pages=True, threads=threads, slab=slab)
    for a in ("page_counts", "alloc_counts", "totals", "kernel_rows", "kun", "kernel_pages"):
        assert np.array_equal(getattr(par, a), getattr(ser, a)), a
