"""The synthetic trace generator (tracegen/) against its written spec (CPU only).

tracegen is shared input infrastructure, not the method; these tests check the
host implementation against an independent Python transcription of GENERATOR.md
section 3, the patterns' closed forms, and the plans' structural promises.
The device implementation is cross-checked against the host one in
tests/test_gpu_parity.py.
"""
import random

import numpy as np
import pytest

from tracegen import build_plan, host_records, splitmix64
from tracegen.plan import PERM, STRAY, STRIDED, SWEEP, TILED, ZIPF

U64 = (1 << 64) - 1


@pytest.fixture(autouse=True)
def _lib(built):
    return built


def spec_addr(row, cdf, t):
    _, kind, base, S, p0, p1, p2, _ = (int(x) for x in row)
    if kind == SWEEP:
        m = S // p0
        return base + p0 * ((p1 + t % m) % m)
    if kind == STRIDED:
        return base + ((t % (S >> p0)) << p0)
    if kind == PERM:
        return base + p0 * (((p1 * t + p2) & U64) % (S // p0))
    if kind == ZIPF:
        e, re = p0 & 0xFF, (p0 >> 8) & 0xFF
        off, R = p2 >> 32, p2 & 0xFFFFFFFF
        h = splitmix64((p1 + (t >> re)) & U64)
        row_i = min(R - 1, sum(1 for r in range(R) if int(cdf[off + r]) <= h))
        return base + row_i * (e << re) + (t % (1 << re)) * e
    if kind == TILED:
        e, lt, ln = p0 & 0xFF, (p0 >> 8) & 0xFF, (p0 >> 16) & 0xFF
        tile = (p2 + (t >> lt) * p1) % (1 << ln)
        return base + e * (tile * (1 << lt) + t % (1 << lt))
    if kind == STRAY:
        return base + ((splitmix64((p1 + t) & U64) % S) & ~(p0 - 1))
    raise AssertionError(kind)


def test_host_matches_spec_transcription():
    p = build_plan("tiny")
    rec = host_records(p)
    starts = [int(x) for x in p.streams[:, 0]] + [p.n]
    rng = random.Random(5)
    for s in range(len(p.streams)):
        if starts[s + 1] == starts[s]:
            continue
        for _ in range(40):
            j = rng.randrange(starts[s], starts[s + 1])
            assert int(rec[j]) == spec_addr(p.streams[s], p.cdf, j - starts[s]), (s, j)


def test_host_ranges_are_slices():
    p = build_plan("tiny", n=1 << 16)
    full = host_records(p)
    for j0, j1 in [(0, 1), (5, 9), (12345, 40000), (p.n - 3, p.n)]:
        assert np.array_equal(host_records(p, j0, j1), full[j0:j1])


def test_plans_deterministic_and_structured():
    for name in ["tiny", "rn50", "gpt2m", "uvm", "llama"]:
        a, b = build_plan(name), build_plan(name)
        assert np.array_equal(a.streams, b.streams) and np.array_equal(a.kernel_offsets, b.kernel_offsets)
        assert a.allocs == b.allocs
        ko = a.kernel_offsets.astype(np.int64)
        assert ko[0] == 0 and ko[-1] == a.n and np.all(np.diff(ko) >= 0)
        # registrations never overlap and lie in the window
        al = sorted(a.allocs)
        for (b0, s0), (b1, _) in zip(al, al[1:]):
            assert b0 + s0 <= b1
        assert al[0][0] >= a.va_lo and al[-1][0] + al[-1][1] <= a.va_hi
        # no stream straddles a kernel boundary
        st = a.streams[:, 0].astype(np.int64)
        kidx = np.searchsorted(ko, st, side="right") - 1
        ends = np.append(st[1:], a.n)
        assert np.all(ends <= ko[np.minimum(kidx + 1, len(ko) - 1)])
        assert (a.va_hi - a.va_lo) >> a.page_shift < (1 << 32)


def test_non_stray_records_are_attributed():
    """a generated trace attributes every non-stray access (no Unattributed)."""
    p = build_plan("tiny")
    rec = host_records(p)
    al = sorted(p.allocs)
    bases = np.array([b for b, _ in al], dtype=np.uint64)
    ends = np.array([b + s for b, s in al], dtype=np.uint64)
    starts = [int(x) for x in p.streams[:, 0]] + [p.n]
    for s in range(len(p.streams)):
        seg = rec[starts[s]:starts[s + 1]]
        i = np.searchsorted(bases, seg, side="right") - 1
        inside = (i >= 0) & (seg < ends[np.maximum(i, 0)])
        if int(p.streams[s, 1]) == STRAY:
            assert not inside.any()
        else:
            assert inside.all(), s


def test_pattern_closed_forms():
    p = build_plan("tiny")
    rec = host_records(p)
    starts = [int(x) for x in p.streams[:, 0]] + [p.n]
    for s in range(len(p.streams)):
        kind, base, S, p0 = (int(x) for x in p.streams[s, 1:5])
        seg = rec[starts[s]:starts[s + 1]].astype(object)
        if kind == PERM:  # bijective over each aligned block of M records
            M = S // p0
            if len(seg) >= M:
                offs = sorted((int(a) - base) // p0 for a in seg[:M])
                assert offs == list(range(M))
        if kind == SWEEP:
            m = S // p0
            d = [(int(b) - int(a)) for a, b in zip(seg[:-1], seg[1:])]
            assert all(x == p0 or x == p0 - S for x in d)
        if kind == STRIDED:
            assert all((int(a) - base) % (1 << p0) == 0 for a in seg[:1000])


def test_stress_plans_structure():
    """SURVEY.md section 8d stress rows: s_perm keeps gpt2m's kernels / allocations /
    record counts with every non-stray stream a permutation; s_hot puts every record on
    one 4 KiB page; s_manyranges registers 65,536 disjoint ranges inside its window and
    sends ~30 % of its records to the small ones."""
    g, sp = build_plan("gpt2m"), build_plan("s_perm")
    assert sp.n == g.n and sp.allocs == g.allocs and np.array_equal(sp.kernel_offsets, g.kernel_offsets)
    assert np.array_equal(sp.streams[:, 0], g.streams[:, 0])
    kinds = set(int(k) for k in sp.streams[:, 1])
    assert kinds <= {PERM, STRAY} and PERM in kinds
    for row in sp.streams[:50]:
        if int(row[1]) == PERM:
            S, e = int(row[3]), int(row[4])
            assert S & (S - 1) == 0 and S % e == 0 and int(row[5]) & 1
    h = build_plan("s_hot")
    (pb, psz), = h.allocs
    assert psz == 4096 and pb % 4096 == 0 and h.n == 1 << 31
    r = host_records(h, h.n - (1 << 16), h.n)
    assert int(r.min()) >= pb and int(r.max()) < pb + 4096
    m = build_plan("s_manyranges")
    assert len(m.allocs) == 65536
    iv = sorted(m.allocs)
    assert all(b0 + s0 <= b1 for (b0, s0), (b1, _) in zip(iv, iv[1:]))
    assert iv[0][0] >= m.va_lo and iv[-1][0] + iv[-1][1] <= m.va_hi
