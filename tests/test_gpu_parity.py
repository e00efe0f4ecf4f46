"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, on the same seeded inputs. Bit-exact on every output (integer path).

Small cases run the whole oracle; full BASELINE sizes (test_full_configs) run in the
bench launch configuration and are checked on sampled kernel segments the oracle
computes one by one, plus invariants that hold at any size.
"""
import json
import os
import random
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2602_22103_b200 as pb  # noqa: E402
import oracle  # noqa: E402
import tracegen  # noqa: E402
from tests.harness import (assert_parity, gpu_trace, oracle_results, oracle_trace, run_gpu, run_oracle,  # noqa: E402
                           u64)  # noqa: E402

DEV = torch.device("cuda:0")
GOLD = os.path.join(os.path.dirname(__file__), "golden")
U64MAX = (1 << 64) - 1


def _t(np_u64):
    return torch.from_numpy(np.ascontiguousarray(np_u64, dtype=np.uint64).view(np.int64)).to(DEV)


def _case(ranges, records, va_lo, va_hi, s, ko=None, rows=True, pages=True, topk=(1, 5, 64), max_ids=None,
          label="", misalign=False, window_kernels=0, schedule="auto"):
    rec = np.asarray(records, dtype=np.uint64)
    tr = gpu_trace(DEV, va_lo, va_hi, ranges, max_ids=max_ids, schedule=schedule)
    o = oracle_trace(va_lo, va_hi, ranges, max_ids=max_ids)
    if ko is None and (rows or pages):
        ko = [0, rec.size]
    if misalign:
        buf = torch.zeros(rec.size + 1, dtype=torch.int64, device=DEV)
        buf[1:] = _t(rec) if rec.size else buf[1:]
        dev_rec = buf[1:]
        assert rec.size == 0 or dev_rec.data_ptr() % 16 == 8
    else:
        dev_rec = _t(rec) if rec.size else torch.zeros(0, dtype=torch.int64, device=DEV)
    wk = window_kernels if rows else 0
    g = run_gpu(tr, dev_rec, s, ko, kernel_rows=rows, kernel_pages=pages and rows, topk=topk, window_kernels=wk)
    r = run_oracle(o, rec, s, ko, kernel_rows=rows, kernel_pages=pages and rows, topk=topk, window_kernels=wk)
    assert_parity(g, r, kernel_rows=rows, kernel_pages=pages and rows, label=label)
    tr.close()
    return g, r


# ------------------------------------------------------------------ generator
def test_device_generator_matches_host():
    for name in ["tiny", "rn50", "llama"]:
        p = tracegen.build_plan(name)
        dp = tracegen.DevicePlan(p, DEV)
        rng = random.Random(11)
        windows = [(0, min(p.n, 1 << 20)), (p.n - 4097, p.n)]
        windows += [(j, j + 100003) for j in (rng.randrange(0, p.n - 100003) for _ in range(3))]
        for j0, j1 in windows:
            out = torch.empty(j1 - j0, dtype=torch.int64, device=DEV)
            tracegen.device_records(dp, out, j0, j1)
            torch.cuda.synchronize()
            assert np.array_equal(u64(out), tracegen.host_records(p, j0, j1)), (name, j0, j1)


# ------------------------------------------------------------------ goldens
def test_hand_worked_golden_on_gpu():
    with open(os.path.join(GOLD, "hand_worked.json")) as f:
        gd = json.load(f)
    e = gd["expect"]
    g, _ = _case(gd["ranges"], gd["records"], gd["window"][0], gd["window"][1], gd["page_shift"],
                 ko=gd["kernel_offsets"], topk=(2, 3, 10), label="hand_worked")
    assert g["page_counts"].tolist() == e["page_counts"]
    assert g["kac"].tolist() == e["kernel_alloc_counts"]
    assert int(g["bitmap"][0]) == e["bitmap_word0"]
    assert g["kstats"][:, 2].tolist() == e["footprint"] and int(g["totals"][4]) == e["ws_obj"]
    assert g["kstats"][:, 3].tolist() == e["kernel_unique_pages"]
    p, c, f = g["topk"][3]
    assert [[int(a), int(b)] for a, b in zip(p, c)] == e["top3"]
    h = gd["at_2MiB"]
    g2, _ = _case(gd["ranges"], gd["records"], h["window"][0], h["window"][1], h["page_shift"], topk=(1,),
                  label="hand_worked_2MiB")
    assert g2["page_counts"].tolist() == h["page_counts"]


def test_snapshot_sequence_on_gpu():
    with open(os.path.join(GOLD, "snapshot_sequence.json")) as f:
        gd = json.load(f)
    tr = pb.Trace(DEV, gd["window"][0], gd["window"][1], 8, 8)
    hist = tr.histograms(gd["page_shift"])
    for step in gd["steps"]:
        if step[0] == "register":
            if step[3]["status"] == 0:
                assert tr.register_alloc(step[1], step[2]) == step[3]["id"]
            else:
                with pytest.raises(pb.PastaError) as ei:
                    tr.register_alloc(step[1], step[2])
                assert ei.value.status == step[3]["status"]
        elif step[0] == "free":
            if step[2]["status"] == 0:
                tr.register_free(step[1])
            else:
                with pytest.raises(pb.PastaError) as ei:
                    tr.register_free(step[1])
                assert ei.value.status == step[2]["status"]
        else:
            tr.analyze(_t(np.array(step[1], dtype=np.uint64)), gd["page_shift"], hist)
    tr.sync()
    assert u64(hist.alloc_counts)[:3].tolist() == gd["expect"]["alloc_counts"]
    assert int(u64(hist.totals)[1]) == gd["expect"]["unattributed"]
    assert int(u64(hist.totals)[0]) == gd["expect"]["records"]


# ------------------------------------------------------------------ tiny config (whole oracle)
# Both scan schedules (contiguous per-warp ranges, interleaved chunks) must give
# identical results; "auto" picks contiguous at these sizes.
SCHEDULES = ["contiguous", "interleaved"]


@pytest.mark.parametrize("seed", [42, 7])
@pytest.mark.parametrize("schedule", SCHEDULES)
def test_tiny_config_parity(seed, schedule):
    p = tracegen.build_plan("tiny", seed=seed)
    rec = tracegen.host_records(p)
    dp = tracegen.DevicePlan(p, DEV)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(dp, drec)
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs, schedule=schedule)
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    ko = [int(x) for x in p.kernel_offsets]
    g = run_gpu(tr, drec, p.page_shift, ko, kernel_rows=True, kernel_pages=True, topk=(16, 1, 1000),
                window_kernels=3)
    r = run_oracle(o, rec, p.page_shift, ko, kernel_rows=True, kernel_pages=True, topk=(16, 1, 1000),
                   window_kernels=3)
    assert_parity(g, r, kernel_rows=True, kernel_pages=True, label=f"tiny/{seed}/{schedule}")
    assert g["hot"].shape == (3, p.n_pages) and int(g["hot"].sum()) == int(g["page_counts"].sum())
    tr.close()


def test_tiny_at_2mib_and_accumulate():
    """page_shift 21, and a trace analyzed in two calls (cut inside kernel 3) accumulates
    exactly like one call: counts are pointwise sums."""
    p = tracegen.build_plan("tiny", seed=3)
    rec = tracegen.host_records(p)
    ko = [int(x) for x in p.kernel_offsets]
    cut = ko[3] + 12345
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
    h1 = tr.histograms(21, n_kernels=4, kernel_rows=True, kernel_pages=True)
    run_gpu(tr, _t(rec[:cut]), 21, ko[:4] + [cut], kernel_rows=True, kernel_pages=True, hist=h1, finalize=False)
    h2 = tr.histograms(21, n_kernels=5, kernel_rows=True, kernel_pages=True)
    ko2 = [0, ko[4] - cut] + [x - cut for x in ko[5:]]
    run_gpu(tr, _t(rec[cut:]), 21, ko2, kernel_rows=True, kernel_pages=True, hist=h2, finalize=False)
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    r = run_oracle(o, rec, 21, ko, kernel_rows=True, kernel_pages=True)
    k1 = u64(h1.kernel_alloc_counts).reshape(4, -1)
    k2 = u64(h2.kernel_alloc_counts).reshape(5, -1)
    kac = np.concatenate([k1[:3], k1[3:4] + k2[:1], k2[1:]])
    assert np.array_equal(kac, r["kac"])
    assert np.array_equal(u64(h1.page_counts) + u64(h2.page_counts), r["page_counts"])
    assert np.array_equal(u64(h1.alloc_counts) + u64(h2.alloc_counts), r["alloc_counts"])
    b1 = u64(h1.kernel_page_bitmap).reshape(4, -1)
    b2 = u64(h2.kernel_page_bitmap).reshape(5, -1)
    assert np.array_equal(np.concatenate([b1[:3], b1[3:4] | b2[:1], b2[1:]]), r["kpb"])
    tr.close()


# ------------------------------------------------------------------ adversarial small traces
def _adversarial(rng, n, s, nr, near_top=False, adjacent=0.5):
    npg = rng.randint(1, 300)
    if near_top:
        va_hi = (U64MAX >> 21) << 21
        va_lo = va_hi - (npg << s)
    else:
        va_lo = rng.randrange(0, 1 << 24) << 21
        va_hi = va_lo + (npg << s)
    lo = max(0, va_lo - (4 << s))
    hi = min(U64MAX, va_hi + (4 << s))
    ranges = []
    cur = lo + rng.randrange(0, 1 << s)
    for _ in range(nr):
        if ranges and rng.random() < adjacent:
            b = ranges[-1][0] + ranges[-1][1]
        else:
            b = cur + rng.randrange(0, 2 << s)
        sz = rng.randrange(1, 2 << s)
        if b + sz > min(hi, U64MAX - 1):
            break
        ranges.append((b, sz))
        cur = b + sz
    pts = [lo, hi, 0, U64MAX, va_lo, va_hi, max(0, va_lo - 1), va_hi - 1]
    for b, sz in ranges:
        pts += [max(0, b - 1), b, b + sz - 1, b + sz]
    rec = []
    run = 0
    while len(rec) < n:
        m = rng.random()
        if m < 0.3:
            rec.append(rng.choice(pts))
        elif m < 0.6:  # coalesced run
            a = rng.randrange(lo, hi)
            e = rng.choice([4, 8, 16])
            ln = rng.randint(1, 200)
            rec += [min(U64MAX, a + e * i) for i in range(ln)]
        else:
            rec.append(rng.randrange(lo, hi + 1))
        run += 1
    rec = rec[:n]
    return ranges, rec, va_lo, va_hi


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("schedule", SCHEDULES)
def test_adversarial_random(seed, schedule):
    rng = random.Random(100 + seed)
    for trial in range(6):
        s = rng.choice([12, 21])
        n = rng.choice([0, 1, 2, 3, 31, 4095, 4096, 4097, 8193, 60001, 250_000])
        nr = rng.choice([0, 1, 5, 40, 300])
        ranges, rec, va_lo, va_hi = _adversarial(rng, n, s, nr, near_top=rng.random() < 0.3)
        nk = rng.choice([1, 2, 7, 50])
        cuts = sorted(rng.randint(0, n) for _ in range(nk - 1))
        if nk > 2 and n > 10:
            cuts[0] = cuts[1]  # an empty kernel
        ko = [0] + cuts + [n]
        _case(ranges, rec, va_lo, va_hi, s, ko=ko, topk=(1, 7, 300), misalign=rng.random() < 0.4,
              label=f"adv{seed}/{trial} n={n} A={len(ranges)} s={s} {schedule}", window_kernels=rng.choice([0, 1, 3]),
              schedule=schedule)


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_many_ranges_global_table(schedule):
    """A = 65,536 live ranges: the boundary array no longer fits shared memory."""
    rng = random.Random(9)
    va_lo = 1 << 40
    ranges = []
    b = va_lo
    for _ in range(65536):
        b += rng.randrange(0, 64) * 64
        sz = rng.randrange(1, 33) * 64
        ranges.append((b, sz))
        b += sz
    va_hi = ((b >> 21) + 1) << 21
    n = 300_000
    rec = [rng.randrange(va_lo - 4096, va_hi + 4096) for _ in range(n // 2)]
    for _ in range(n // 2 // 64):
        a = rng.randrange(va_lo, va_hi)
        rec += [a + 8 * i for i in range(64)]
    ko = [0, n // 3, n // 3, len(rec)]
    _case(ranges, rec, va_lo, va_hi, 12, ko=ko, topk=(10,), label="A=65536", schedule=schedule)


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_contention_and_scatter(schedule):
    MiB = 1 << 20
    va_lo, va_hi = 1 << 41, (1 << 41) + 64 * MiB
    ranges = [(va_lo + i * MiB, MiB) for i in range(64)]
    hot = [va_lo + 5 * MiB + 100] * 1_000_003  # one page, maximal contention
    _case(ranges, hot, va_lo, va_hi, 12, ko=[0, 500_000, len(hot)], topk=(3,), label="hot page", schedule=schedule)
    # every record a distinct page (permutation over the window at 4 KiB stride)
    P = 64 * MiB >> 12
    j = np.arange(P * 3, dtype=np.uint64)
    rec = np.uint64(va_lo) + ((j * np.uint64(2654435761)) % np.uint64(P)) * np.uint64(4096)
    _case(ranges, rec, va_lo, va_hi, 12, ko=[0, P, 2 * P, 3 * P], topk=(1, 100, 5000), label="all distinct",
          schedule=schedule)


def test_host_records_path_equals_device_path():
    p = tracegen.build_plan("tiny", seed=5)
    rec = tracegen.host_records(p)
    ko = [int(x) for x in p.kernel_offsets]
    tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs), host_chunk_bytes=1 << 20)  # 8 chunks
    for b, s in p.allocs:
        tr.register_alloc(b, s)
    host_rec = torch.from_numpy(rec.view(np.int64)).pin_memory()
    g = run_gpu(tr, host_rec, 12, ko, kernel_rows=True, kernel_pages=True, topk=(16,), host=True)
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    r = run_oracle(o, rec, 12, ko, kernel_rows=True, kernel_pages=True, topk=(16,))
    assert_parity(g, r, kernel_rows=True, kernel_pages=True, label="host path")
    tr.close()


# ------------------------------------------------------------------ top-K edge cases
@pytest.mark.parametrize("K", [1, 2, 17, 1024, 2048, 4096, 5000, 68266])
def test_topk_direct(K):
    rng = np.random.default_rng(K)
    P = 300_000
    counts = rng.integers(0, 4, size=P).astype(np.uint64)  # heavy ties, many zeros
    counts[rng.integers(0, P, 50)] = rng.integers(1 << 33, 1 << 34, 50).astype(np.uint64)  # big values
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    pcnt = _t(counts)
    p, c, f = tr.topk(pcnt, K)
    tr.sync()
    rp, rc, rf = oracle.topk(counts, K)
    assert int(u64(f)[0]) == rf
    assert np.array_equal(u64(p), rp) and np.array_equal(u64(c), rc)
    # K > nnz
    small = np.zeros(1000, dtype=np.uint64)
    small[[3, 500, 999]] = [7, 7, 1]
    p, c, f = tr.topk(_t(small), K)
    tr.sync()
    rp, rc, rf = oracle.topk(small, K)
    assert int(u64(f)[0]) == rf == min(K, 3)
    assert np.array_equal(u64(p), rp) and np.array_equal(u64(c), rc)
    # all zero
    p, c, f = tr.topk(_t(np.zeros(77, dtype=np.uint64)), K)
    tr.sync()
    assert int(u64(f)[0]) == 0 and np.all(u64(p) == np.uint64(U64MAX)) and np.all(u64(c) == 0)
    tr.close()


def test_topk_unaligned_tiny_and_k_above_p():
    """The count array may start at an 8-byte (not 16-byte) boundary (a slice of a
    larger buffer), hold 1 or 2 pages, or be shorter than K (scratch sized by min(K, P);
    slots [found, K) are sentinels)."""
    rng = np.random.default_rng(5)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    big = rng.integers(0, 9, size=200_001).astype(np.uint64)
    dbig = _t(big)
    for off, P, K in [(1, 200_000, 1000), (1, 1, 5), (3, 2, 1), (0, 1, 68266), (1, 77, 68266), (0, 2, 2)]:
        sub = big[off:off + P]
        p, c, f = tr.topk(dbig[off:off + P], K)
        tr.sync()
        rp, rc, rf = oracle.topk(sub, K)
        assert int(u64(f)[0]) == rf, (off, P, K)
        assert np.array_equal(u64(p), rp) and np.array_equal(u64(c), rc), (off, P, K)
    tr.close()


@pytest.mark.parametrize("P", [1000, 5000, 70_000, 1 << 20])
def test_topk_small_arrays_few_ctas(P):
    """Small count arrays run on few CTAs, so one CTA can hold every key of the selected
    range: all counts equal (the whole array is the range), two values, sparse. Every K
    against the oracle (a region overflow once sent the fast finish garbage)."""
    rng = np.random.default_rng(P)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    cases = [np.full(P, 8, dtype=np.uint64), np.full(P, 1, dtype=np.uint64),
             rng.integers(7, 9, size=P).astype(np.uint64)]
    sparse = np.zeros(P, dtype=np.uint64)
    sparse[rng.integers(0, P, 3000)] = 5
    cases.append(sparse)
    for i, counts in enumerate(cases):
        for K in (1, 3, 1000, 4096, 5000):
            p, c, f = tr.topk(_t(counts), K)
            tr.sync()
            rp, rc, rf = oracle.topk(counts, K)
            assert int(u64(f)[0]) == rf and np.array_equal(u64(c), rc) and np.array_equal(u64(p), rp), (P, i, K)
    tr.close()


def test_topk_many_and_prefix():
    """pasta_topk_many: each list equals pasta_topk / the oracle for its own k (k above
    nnz and above P included, duplicates, 16 entries); pasta_topk_prefix of a merged list;
    argument errors are status codes."""
    rng = np.random.default_rng(77)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    for P, ks in [(300_001, [16, 1024, 1, 5000, 1024]), (5, [1, 3, 8, 2]),
                  (1_000_000, [1 << i for i in range(16)])]:
        counts = rng.integers(0, 6, size=P).astype(np.uint64)
        counts[rng.integers(0, P, 30)] = rng.integers(1 << 20, 1 << 40, 30).astype(np.uint64)
        outs = [(torch.full((k,), 7, dtype=torch.int64, device=DEV), torch.full((k,), 7, dtype=torch.int64, device=DEV),
                 torch.full((1,), 7, dtype=torch.int64, device=DEV)) for k in ks]
        pb.pasta_topk_many(tr.h, _t(counts), P, ks, outs)
        tr.sync()
        for k, (p, c, f) in zip(ks, outs):
            rp, rc, rf = oracle.topk(counts, k)
            assert int(u64(f)[0]) == rf, (P, k)
            assert np.array_equal(u64(p), rp) and np.array_equal(u64(c), rc), (P, k)
    # prefix of a given list
    counts = rng.integers(0, 1000, size=50_000).astype(np.uint64)
    src = tr.topk(_t(counts), 700)
    outs = {k: (torch.empty(k, dtype=torch.int64, device=DEV), torch.empty(k, dtype=torch.int64, device=DEV),
                torch.empty(1, dtype=torch.int64, device=DEV)) for k in (1, 699, 700)}
    tr.topk_prefix(src, 700, list(outs), list(outs.values()))
    tr.sync()
    for k, (p, c, f) in outs.items():
        rp, rc, rf = oracle.topk(counts, k)
        assert int(u64(f)[0]) == rf and np.array_equal(u64(p), rp) and np.array_equal(u64(c), rc), k
    with pytest.raises(pb.PastaError):
        tr.topk_prefix(src, 700, [701], [outs[700]])
    with pytest.raises(pb.PastaError):
        tr.topk_many(_t(counts), [1] * 17)
    with pytest.raises(pb.PastaError):
        tr.topk_many(_t(counts), [4, 0])
    tr.close()


def _topk_dists():
    rng = np.random.default_rng(2024)
    P = 3_000_017  # several CTAs' ranges, odd length
    yield "all equal", np.full(P, 5, dtype=np.uint64)
    yield "exact small bins", rng.integers(0, 64, size=P).astype(np.uint64)
    geo = (rng.geometric(0.002, size=P) - 1).astype(np.uint64)
    yield "geometric", geo
    wide = (rng.integers(0, 1 << 62, size=P, dtype=np.uint64) >> rng.integers(0, 62, size=P).astype(np.uint64))
    wide[rng.integers(0, P, 40)] = np.uint64(U64MAX)  # bit length 64, tied at the top
    wide[rng.integers(0, P, 40)] = np.uint64(1 << 63)
    yield "64-bit spread", wide
    sparse = np.zeros(P, dtype=np.uint64)
    sparse[rng.integers(0, P, 3000)] = rng.integers(1, 1 << 20, 3000).astype(np.uint64)
    yield "sparse", sparse
    ties = rng.integers(1000, 1010, size=P).astype(np.uint64)  # one 2^k bin, ties cut deep inside
    yield "narrow band", ties


@pytest.mark.parametrize("K", [1, 999, 1024, 4097, 68266])
def test_topk_distributions(K):
    """Threshold bins of every kind: an exact small-value bin (< 64), float-key bins
    of every bit length up to 64, whole-bin takes, and ties spread over every CTA's
    page range (all counts equal), checked against the oracle's full sort."""
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    for name, counts in _topk_dists():
        p, c, f = tr.topk(_t(counts), K)
        tr.sync()
        rp, rc, rf = oracle.topk(counts, K)
        assert int(u64(f)[0]) == rf, name
        assert np.array_equal(u64(c), rc), name
        assert np.array_equal(u64(p), rp), name
    tr.close()


def test_bitmap_or_merge_kernel():
    rng = np.random.default_rng(4)
    g, W = 4, 70001
    bms = rng.integers(0, 1 << 63, size=(g, W), dtype=np.uint64) & rng.integers(0, 1 << 63, size=(g, W), dtype=np.uint64)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    gathered = _t(bms.reshape(-1))
    out = torch.empty(W, dtype=torch.int64, device=DEV)
    pop = torch.zeros(1, dtype=torch.int64, device=DEV)
    tr.bitmap_or(gathered, g, W, out, pop)
    tr.sync()
    ref = np.bitwise_or.reduce(bms, axis=0)
    assert np.array_equal(u64(out), ref)
    assert int(u64(pop)[0]) == int(np.unpackbits(ref.view(np.uint8)).sum())
    tr.close()


def test_errors_are_status_codes():
    with pytest.raises(pb.PastaError) as ei:  # unknown open flags
        pb.pasta_trace_open(0, 0, 1 << 30, 2, 3, 0, 0, flags=3)
    assert ei.value.status == pb.PASTA_EINVAL
    tr = pb.Trace(DEV, 0, 1 << 30, 2, 3)
    with pytest.raises(pb.PastaError) as ei:
        tr.register_alloc(0x1000, 0)
    assert ei.value.status == pb.PASTA_EINVAL
    tr.register_alloc(0x1000, 0x1000)
    with pytest.raises(pb.PastaError) as ei:
        tr.register_alloc(0x1800, 0x10)
    assert ei.value.status == pb.PASTA_EOVERLAP
    with pytest.raises(pb.PastaError) as ei:
        tr.register_free(0x1800)
    assert ei.value.status == pb.PASTA_ENOENT
    hist = tr.histograms(12)
    with pytest.raises(pb.PastaError) as ei:  # page_shift out of range
        tr.analyze(torch.zeros(4, dtype=torch.int64, device=DEV), 11, hist)
    assert ei.value.status == pb.PASTA_EINVAL
    with pytest.raises(pb.PastaError) as ei:  # misaligned window for 2^31 pages
        pb.Trace(DEV, 4096, 1 << 30, 1, 1).analyze(torch.zeros(4, dtype=torch.int64, device=DEV), 21, hist)
    assert ei.value.status == pb.PASTA_EINVAL
    tr.close()


# ------------------------------------------------------------------ full BASELINE sizes
FULL = ["rn50", "gpt2m", "uvm", "llama"]
# SURVEY.md section 8d stress rows at their full sizes: s_perm (gpt2m with every stream a
# permutation), s_hot (2^31 records on one page), s_manyranges (A = 65,536: global table)
STRESS = list(tracegen.plan.STRESS)


@pytest.mark.parametrize("name", FULL + STRESS)
def test_full_config_bit_exact(name):
    """Every output of a full BASELINE config (rn50 5e8, gpt2m 2e9, uvm 4e9 at 2 MiB pages
    with per-kernel page bitmaps and top-68,266, llama 10.7e9) in the bench's launch
    configuration (device-generated records, one analyze + finalize, top-K per plan),
    compared element by element with the WHOLE-trace oracle: page counts (P up to
    16.8 M), alloc counts, totals, bitmap, unique pages, kernel rows and stats,
    footprints, WS_obj, MAX_MEM_REFERENCED_KERNEL, per-kernel page bitmaps, top-K lists.
    The oracle runs chunk-parallel on the host's cores (OracleTrace.analyze_parallel:
    kernel-aligned slabs, host-generated records, per-thread arrays summed)."""
    p = tracegen.build_plan(name)
    free = torch.cuda.mem_get_info(DEV)[0]
    if p.n * 8 + (4 << 30) > free:
        pytest.skip(f"{name} needs {p.n * 8 / 2**30:.1f} GiB")
    dp = tracegen.DevicePlan(p, DEV)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(dp, drec)
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
    ko = [int(x) for x in p.kernel_offsets]
    g = run_gpu(tr, drec, p.page_shift, ko, kernel_rows=True, kernel_pages=p.want_kernel_pages,
                topk=tuple(p.topk))
    tr.close()
    del drec, g["hist"]
    torch.cuda.empty_cache()
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    o.analyze_parallel(lambda j0, j1: tracegen.host_records(p, j0, j1), p.kernel_offsets, p.page_shift,
                       kernel_rows=True, kernel_pages=p.want_kernel_pages)
    r = oracle_results(o, kernel_rows=True, kernel_pages=p.want_kernel_pages, topk=tuple(p.topk))
    assert int(r["totals3"][0]) == p.n
    assert_parity(g, r, kernel_rows=True, kernel_pages=p.want_kernel_pages, label=name)


@pytest.mark.parametrize("name,n", [("gpt2m", 1 << 24), ("llama", 1 << 26), ("uvm", 1 << 25), ("rn50", 3 << 23)])
def test_dynamic_interleaved_schedule_prefixes(name, n):
    """The interleaved schedule with dynamically taken chunks (forced, so the chunk size is
    the largest that gives every warp one: 16-64 slices here, a few hundred chunks taken
    from the counter after the static first round), on plan prefixes cut inside kernels,
    every output against the whole-prefix oracle; 4 KiB paired copies (4-stage rings) and
    single copies (uvm's 3-stage ring)."""
    p = tracegen.build_plan(name)
    ko = [int(x) for x in p.kernel_offsets if int(x) < n] + [n]
    drec = torch.empty(n, dtype=torch.int64, device=DEV)
    tracegen.device_records(tracegen.DevicePlan(p, DEV), drec, 0, n)
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs, schedule="interleaved")
    g = run_gpu(tr, drec, p.page_shift, ko, kernel_rows=True, kernel_pages=p.want_kernel_pages, topk=(1, 1024))
    tr.close()
    del drec
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    o.analyze_parallel(lambda j0, j1: tracegen.host_records(p, j0, j1), ko, p.page_shift, kernel_rows=True,
                       kernel_pages=p.want_kernel_pages)
    r = oracle_results(o, kernel_rows=True, kernel_pages=p.want_kernel_pages, topk=(1, 1024))
    assert int(r["totals3"][0]) == n
    assert_parity(g, r, kernel_rows=True, kernel_pages=p.want_kernel_pages, label=f"{name}/{n}/dynamic")


def _table(rng, A, va_lo, page_shift):
    """A live ranges packed upward from va_lo: sizes 1 B .. 6 pages, half of them adjacent
    to their predecessor, the rest after a gap of up to 2 pages."""
    ranges, b = [], va_lo + rng.randrange(0, 4096)
    for _ in range(A):
        if ranges and rng.random() >= 0.5:
            b += rng.randrange(1, 2 << page_shift)
        sz = rng.randrange(1, 6 << page_shift)
        ranges.append((b, sz))
        b += sz
    return ranges, b


@pytest.mark.parametrize("A", [1544, 1545, 4616, 4617])
@pytest.mark.parametrize("schedule", SCHEDULES)
def test_table_size_transitions(A, schedule):
    """The scan's shared-memory budget changes shape at these table sizes (24 warps: 4 ring
    stages up to 1,544 ranges, 3 up to 4,616, the global-memory table above): the whole
    oracle on 3 M records over each, every output."""
    rng = random.Random(A)
    va_lo = 1 << 40
    ranges, end = _table(rng, A, va_lo, 12)
    va_hi = ((end >> 21) + 1) << 21
    npr = np.random.default_rng(A)
    n = 3_000_001
    starts = npr.integers(va_lo - 8192, va_hi + 8192, size=n // 256 + 1, dtype=np.uint64)
    elem = npr.choice(np.array([4, 8, 64, 4096], dtype=np.uint64), size=starts.size)
    rec = (starts[:, None] + elem[:, None] * np.arange(256, dtype=np.uint64)[None, :]).reshape(-1)[:n]
    scatter = npr.random(n) < 0.05
    rec[scatter] = npr.integers(va_lo - 8192, va_hi + 8192, size=int(scatter.sum()), dtype=np.uint64)
    nk = 37
    ko = [0] + sorted(int(x) for x in npr.integers(0, n, nk - 1)) + [n]
    _case(ranges, rec, va_lo, va_hi, 12, ko=ko, topk=(1, 1024), label=f"A={A} {schedule}", schedule=schedule)


def test_merger_world1_nccl():
    """The NCCL merge path (all_reduce SUM of the packed counts, all_gather + the
    pasta_bitmap_or kernel, all_reduce MAX of WS) at world size 1 leaves a finalized
    result unchanged; its OR output equals the bitmap recomputed from the counts."""
    import socket

    import torch.distributed as dist

    from paper_2602_22103_b200 import dist as pdist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=DEV)
    try:
        p = tracegen.build_plan("tiny", seed=9)
        drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
        tracegen.device_records(tracegen.DevicePlan(p, DEV), drec)
        tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
        ko = torch.from_numpy(p.kernel_offsets.view(np.int64).copy()).to(DEV)
        hist = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True)
        tr.analyze(drec, p.page_shift, hist, kernel_offsets=ko)
        tr.sync()
        before = (u64(hist.packed).copy(), u64(hist.page_bitmap).copy())
        pdist.Merger(tr, hist).merge()
        tr.sync()
        after = u64(hist.packed)
        assert np.array_equal(after, before[0])
        assert np.array_equal(u64(hist.page_bitmap), before[1])
        bm, uq = oracle.bitmap(u64(hist.page_counts))
        assert np.array_equal(u64(hist.page_bitmap), bm) and int(u64(hist.totals)[3]) == uq
        o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
        r = run_oracle(o, tracegen.host_records(p), p.page_shift, [int(x) for x in p.kernel_offsets],
                       kernel_rows=True)
        assert int(after[-pb.TOTALS:][pb.T_MAX_KERNEL]) == r["max_kernel"]  # the ARGMAX merge of the pair
        assert int(after[-pb.TOTALS:][pb.T_MAX_KERNEL_RECORDS]) == r["max_kernel_records"]
        tr.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("g,K", [(1, 16), (3, 100), (8, 1024)])
def test_topk_merge_of_shard_candidates(g, K):
    """pasta_topk_merge over g shard-local top-K lists equals the global top-K."""
    rng = np.random.default_rng(g * 7 + K)
    S = 50_000
    counts = rng.integers(0, 6, size=g * S).astype(np.uint64)
    counts[rng.integers(0, g * S, 300)] = rng.integers(10, 1000, 300).astype(np.uint64)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    cp = torch.empty(g * K, dtype=torch.int64, device=DEV)
    cc = torch.empty(g * K, dtype=torch.int64, device=DEV)
    for r in range(g):
        p, c, _ = tr.topk(_t(counts[r * S:(r + 1) * S]), K)
        cp[r * K:(r + 1) * K] = p
        cc[r * K:(r + 1) * K] = c
    out = (torch.empty(K, dtype=torch.int64, device=DEV), torch.empty(K, dtype=torch.int64, device=DEV),
           torch.empty(1, dtype=torch.int64, device=DEV))
    tr.topk_merge(cp, cc, g, K, S, out)
    tr.sync()
    rp, rc, rf = oracle.topk(counts, K)
    assert int(u64(out[2])[0]) == rf
    assert np.array_equal(u64(out[0]), rp) and np.array_equal(u64(out[1]), rc)
    tr.close()


def test_sharded_merger_world1_nccl():
    """dist.ShardedMerger at world size 1: the shard is the whole page array, and the merged
    top-K / bitmap / totals equal the single-GPU results."""
    import socket

    import torch.distributed as dist

    from paper_2602_22103_b200 import dist as pdist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=DEV)
    try:
        p = tracegen.build_plan("tiny", seed=13)
        drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
        tracegen.device_records(tracegen.DevicePlan(p, DEV), drec)
        tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
        ko = torch.from_numpy(p.kernel_offsets.view(np.int64).copy()).to(DEV)
        hist = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True, pad_pages_to=64)
        tr.analyze(drec, p.page_shift, hist, kernel_offsets=ko)
        ref = tr.topk(hist.page_counts, 16)
        tr.sync()
        ref = tuple(u64(x).copy() for x in ref)
        totals = u64(hist.totals).copy()
        outs = pdist.ShardedMerger(tr, hist, (16, 3), None).merge()
        tr.sync()
        assert np.array_equal(u64(outs[16][0]), ref[0]) and np.array_equal(u64(outs[16][1]), ref[1])
        assert int(u64(outs[16][2])[0]) == int(ref[2][0])
        assert np.array_equal(u64(hist.totals), totals)
        rp, rc, rf = oracle.topk(u64(hist.page_counts), 3)
        assert np.array_equal(u64(outs[3][0]), rp)
        tr.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch,stable", [(4096, True), (4096, False), (10_001 * 2, True)])
def test_streaming_batches_equal_oracle(batch, stable):
    """NEXT f2: the trace analyzed as batches (one NO_FINALIZE call each, kernels cut
    between batches accumulating into the same rows) + one finalize == the oracle."""
    from paper_2602_22103_b200.stream import BatchRunner

    p = tracegen.build_plan("tiny", seed=21)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(tracegen.DevicePlan(p, DEV), drec)
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
    hist = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True, kernel_pages=True)
    runner = BatchRunner(tr, hist, drec, p.kernel_offsets, p.n, batch, p.page_shift, stable=stable)
    runner.run()
    tr.finalize(p.page_shift, hist, n_kernels=p.n_kernels)
    tr.sync()
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    ko = [int(x) for x in p.kernel_offsets]
    r = run_oracle(o, tracegen.host_records(p), p.page_shift, ko, kernel_rows=True, kernel_pages=True)
    g = {"page_counts": u64(hist.page_counts), "alloc_counts": u64(hist.alloc_counts), "totals": u64(hist.totals),
         "bitmap": u64(hist.page_bitmap), "kac": u64(hist.kernel_alloc_counts).reshape(p.n_kernels, -1),
         "kstats": u64(hist.kernel_stats).reshape(p.n_kernels, 4),
         "kpb": u64(hist.kernel_page_bitmap).reshape(p.n_kernels, -1), "topk": {}}
    assert_parity(g, r, kernel_rows=True, kernel_pages=True, label=f"stream/{batch}")
    tr.close()



@pytest.mark.parametrize("batch,slots,rows", [(4096, 2, True), (4096, 64, True), (65_536, 4, True), (10_002, 8, False)])
def test_stream_ring_equals_oracle(batch, slots, rows):
    """NEXT f2 persistent consumer: one launch, batch descriptors published into a ring of
    `slots` while it runs (slots = 2: the host waits for the consumer after every other
    batch), kernels cut between batches accumulating into one row, then one finalize ==
    the oracle on every output."""
    from paper_2602_22103_b200.stream import StreamRing

    p = tracegen.build_plan("tiny", seed=22)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(tracegen.DevicePlan(p, DEV), drec)
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
    hist = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=rows, kernel_pages=rows)
    ring = StreamRing(tr, hist, drec, p.kernel_offsets, p.n, batch, p.page_shift, slots=slots)
    try:
        ring.run()
    finally:
        ring.destroy()  # publishes the end even on failure (the consumer always drains)
    tr.finalize(p.page_shift, hist, n_kernels=p.n_kernels if rows else 0)
    tr.sync()
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    ko = [int(x) for x in p.kernel_offsets]
    r = run_oracle(o, tracegen.host_records(p), p.page_shift, ko, kernel_rows=rows, kernel_pages=rows)
    g = {"page_counts": u64(hist.page_counts), "alloc_counts": u64(hist.alloc_counts), "totals": u64(hist.totals),
         "bitmap": u64(hist.page_bitmap), "topk": {}}
    if rows:
        g.update({"kac": u64(hist.kernel_alloc_counts).reshape(p.n_kernels, -1),
                  "kstats": u64(hist.kernel_stats).reshape(p.n_kernels, 4),
                  "kpb": u64(hist.kernel_page_bitmap).reshape(p.n_kernels, -1)})
    assert_parity(g, r, kernel_rows=rows, kernel_pages=rows, label=f"ring/{batch}/{slots}")
    tr.close()


def test_stream_ring_reuses_producer_buffers():
    """The paper's device buffer: the producer owns R = 3 record buffers of
    one batch each and refills buffer i % R only after pasta_stream_consumed says batch
    i - R has been read; the consumer's result equals the oracle over the whole trace."""
    import paper_2602_22103_b200 as pbm

    p = tracegen.build_plan("tiny", seed=23)
    host = tracegen.host_records(p)
    batch, R = 32_768, 3
    bufs = [torch.empty(batch, dtype=torch.int64, device=DEV) for _ in range(R)]
    # the trace gets its own stream: the producer's copies must not queue behind the
    # persistent consumer (a synchronous copy on torch's default stream would)
    tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs), stream=torch.cuda.Stream(DEV))
    for b, sz in p.allocs:
        tr.register_alloc(b, sz)
    hist = tr.histograms(p.page_shift)
    torch.cuda.synchronize()
    s = pbm.pasta_stream_open(tr.h, p.page_shift, R, batch, hist.struct())
    side = torch.cuda.Stream(DEV)
    nb = p.n // batch
    try:
        for i in range(nb):
            t0 = time.time()
            while pbm.pasta_stream_consumed(s) < i - R + 1:
                assert time.time() - t0 < 30, "consumer made no progress"
            buf = bufs[i % R]
            with torch.cuda.stream(side):
                buf.copy_(torch.from_numpy(host[i * batch:(i + 1) * batch].view(np.int64)), non_blocking=False)
            side.synchronize()
            pbm.pasta_stream_push(s, [pbm.pasta_stream_batch(buf.data_ptr(), batch, None, 1, 0)])
    finally:
        pbm.pasta_stream_close(s)
        pbm.pasta_stream_destroy(s)
    tr.finalize(p.page_shift, hist)
    tr.sync()
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    r = run_oracle(o, host[:nb * batch], p.page_shift, None, kernel_rows=False, kernel_pages=False)
    assert np.array_equal(u64(hist.page_counts), r["page_counts"])
    assert np.array_equal(u64(hist.alloc_counts), r["alloc_counts"])
    assert u64(hist.totals)[:3].tolist() == r["totals3"].tolist()
    tr.close()


def test_stream_ring_errors():
    import paper_2602_22103_b200 as pbm

    tr = pb.Trace(DEV, 0, 1 << 32, 4, 4)
    tr.register_alloc(4096, 4096)
    hist = tr.histograms(12)
    for slots, mb in ((1, 1024), (8, 255), (8, 1025)):
        with pytest.raises(pb.PastaError) as ei:
            pbm.pasta_stream_open(tr.h, 12, slots, mb, hist.struct())
        assert ei.value.status == pb.PASTA_EINVAL
    rec = torch.full((2048,), 4096 + 8, dtype=torch.int64, device=DEV)
    torch.cuda.synchronize()
    # (nothing may be enqueued on the trace's stream -- here torch's default stream --
    # while the consumer runs)
    s = pbm.pasta_stream_open(tr.h, 12, 4, 1024, hist.struct())
    for bad in (pbm.pasta_stream_batch(rec.data_ptr(), 2048, None, 1, 0),  # > max_batch
                pbm.pasta_stream_batch(rec.data_ptr(), 3, None, 1, 0),  # odd
                pbm.pasta_stream_batch(rec.data_ptr() + 8, 2, None, 1, 0)):  # not 16-byte aligned
        with pytest.raises(pb.PastaError) as ei:
            pbm.pasta_stream_push(s, [bad])
        assert ei.value.status == pb.PASTA_EINVAL
    pbm.pasta_stream_push(s, [pbm.pasta_stream_batch(rec.data_ptr(), 1024, None, 1, 0)])
    pbm.pasta_stream_close(s)
    with pytest.raises(pb.PastaError) as ei:
        pbm.pasta_stream_push(s, [pbm.pasta_stream_batch(rec.data_ptr(), 2, None, 1, 0)])
    assert ei.value.status == pb.PASTA_ESTATE
    pbm.pasta_stream_destroy(s)
    tr.sync()
    assert int(u64(hist.totals)[0]) == 1024 and int(u64(hist.alloc_counts)[0]) == 1024
    # a stream left open: pasta_close publishes its end, waits for it and frees it
    s = pbm.pasta_stream_open(tr.h, 12, 4, 1024, hist.struct())
    pbm.pasta_stream_push(s, [pbm.pasta_stream_batch(rec.data_ptr(), 1024, None, 1, 0)])
    tr.close()

def test_pdl_ordering_after_producer_kernels():
    """Programmatic dependent launch must not read stale data: each analyze follows, on
    the same stream, a torch kernel that rewrites the records (and one that zeroes the
    outputs), alternating between two traces; without PASTA_REC_STABLE the scan may only
    touch the records after griddepcontrol.wait. Back-to-back analyze calls into the same
    outputs (the streaming pattern) must also add up exactly."""
    p = tracegen.build_plan("tiny", seed=23)
    r0 = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(tracegen.DevicePlan(p, DEV), r0)
    r1 = torch.flip(r0, [0]).contiguous()
    live = torch.empty_like(r0)
    s = torch.cuda.Stream(DEV)
    tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs), stream=s)
    for b, sz in p.allocs:
        tr.register_alloc(b, sz)
    h = tr.histograms(p.page_shift)
    refs = []
    for rec in (r0, r1):
        o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
        o.analyze(u64(rec), None, p.page_shift)
        refs.append(o.page_counts.copy())
    with torch.cuda.stream(s):
        for it in range(40):
            src = (r0, r1)[it % 2]
            live.copy_(src)  # producer kernel right before the scan
            h.zero_()
            tr.analyze(live, p.page_shift, h)
            got = h.page_counts.clone()  # consumer on the same stream
            s.synchronize()
            assert np.array_equal(u64(got), refs[it % 2]), f"iteration {it}"
        # chained calls into the same outputs: 4 x the same records
        h.zero_()
        for i in range(4):  # the first call waits for the zeroing, the rest are chained
            tr.analyze(live, p.page_shift, h, finalize=False, stable=True, chained=i > 0)
        got = h.page_counts.clone()
        s.synchronize()
    with np.errstate(over="ignore"):
        assert np.array_equal(u64(got), refs[1] * np.uint64(4))
    tr.close()


def test_arbitrary_cut_merge_then_finalize():
    """Shards cut INSIDE kernels (not kernel-aligned): the straddling kernels' rows are
    summed (what dist.merge_kernel_rows does across ranks), and pasta_finalize on the
    merged rows recomputes every per-kernel footprint, WS_obj, the unique pages and the
    MAX_MEM_REFERENCED_KERNEL pair exactly as the whole-trace oracle (WS does not merge
    by MAX for such cuts)."""
    p = tracegen.build_plan("tiny", seed=31)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(tracegen.DevicePlan(p, DEV), drec)
    ko = np.asarray(p.kernel_offsets, dtype=np.int64)
    cuts = [0, int(ko[3]) + 1001, int(ko[6]) - 77, p.n]  # inside kernels 3 and 5
    tr = gpu_trace(DEV, p.va_lo, p.va_hi, p.allocs)
    K = p.n_kernels
    merged = tr.histograms(p.page_shift, n_kernels=K, kernel_rows=True, kernel_pages=True)
    for a, b in zip(cuts[:-1], cuts[1:]):
        k0 = int(np.searchsorted(ko, a, side="right")) - 1
        k1 = int(np.searchsorted(ko, b, side="left"))
        sub = np.concatenate([[0], np.clip(ko[k0 + 1:k1] - a, 0, b - a), [b - a]]).astype(np.int64)
        h = tr.histograms(p.page_shift, n_kernels=len(sub) - 1, kernel_rows=True, kernel_pages=True)
        tr.analyze(drec[a:b], p.page_shift, h, kernel_offsets=torch.from_numpy(sub).to(DEV), n=b - a)
        tr.sync()
        # merge: counts and rows SUM, per-kernel page bits OR (rows of the shard start at k0)
        nk = len(sub) - 1
        merged.page_counts += h.page_counts
        merged.alloc_counts += h.alloc_counts
        merged.totals[:3] += h.totals[:3]
        merged.kernel_alloc_counts.view(K, -1)[k0:k0 + nk] += h.kernel_alloc_counts.view(nk, -1)
        ks = merged.kernel_stats.view(K, 4)
        ks[k0:k0 + nk, :2] += h.kernel_stats.view(nk, 4)[:, :2]
        kp = merged.kernel_page_bitmap.view(K, -1)
        kp[k0:k0 + nk] |= h.kernel_page_bitmap.view(nk, -1)
    tr.finalize(p.page_shift, merged, n_kernels=K)
    tr.sync()
    o = oracle_trace(p.va_lo, p.va_hi, p.allocs)
    r = run_oracle(o, tracegen.host_records(p), p.page_shift, [int(x) for x in ko], kernel_rows=True,
                   kernel_pages=True)
    g = {"page_counts": u64(merged.page_counts), "alloc_counts": u64(merged.alloc_counts),
         "totals": u64(merged.totals), "bitmap": u64(merged.page_bitmap),
         "kac": u64(merged.kernel_alloc_counts).reshape(K, -1), "kstats": u64(merged.kernel_stats).reshape(K, 4),
         "kpb": u64(merged.kernel_page_bitmap).reshape(K, -1), "topk": {}}
    assert_parity(g, r, kernel_rows=True, kernel_pages=True, label="arbitrary cuts + finalize")
    tr.close()
