"""Pins of the oracle's tensor level and prefetch-plan builder (NEXT f3; CPU only).

Readings: DESIGN.md R18 (two-level attribution: a tensor lies inside one live object,
S:47; live tensors never overlap), R19 (freeing an object ends its tensors), R20 (a
kernel's prefetch plan = the union of the ranges of the objects / tensors it touched,
S:488-514 build_prefetch_plan).

* SPEC's worked examples for build_prefetch_plan;
* brute force (tests/brute.py linear scans over the tensor set) on random tiny
  two-level registrations;
* the plan's interval union against a byte-coverage bitmap (no interval logic);
* invariants: tensor plan inside the object plan, tensor bytes <= object bytes
  (S:514), conservation (tensor counts + untensored = records).
"""
import random

import numpy as np
import pytest

import oracle
from oracle import OracleTrace
from tests import brute

MiB = 1 << 20


@pytest.fixture(autouse=True)
def _lib(built):
    return built


def _bytes(plan_row):
    return sum(b - a for a, b in plan_row)


def test_spec_prefetch_plan_examples():
    """a kernel touching tensor T (512 B) inside a 2 MiB object O stages 2 MiB
    at object level and 512 B at tensor level; a kernel with zero accesses has an empty
    plan entry."""
    O = 0x7F0000200000
    o = OracleTrace(0x7F0000000000, 0x7F0000000000 + 64 * MiB, 4, 4, max_live_tensors=4, max_tensor_ids=4)
    assert o.register_alloc(O, 2 * MiB) == (oracle.OK, 0)
    assert o.register_tensor(O + 4096, 512) == (oracle.OK, 0)
    rec = np.array([O + 4096 + 100], dtype=np.uint64)
    o.analyze(rec, [0, 1, 1], 21, kernel_rows=True)
    assert o.prefetch_plan("object") == [[(O, O + 2 * MiB)], []]
    assert o.prefetch_plan("tensor") == [[(O + 4096, O + 4096 + 512)], []]
    fo, wso = o.footprints()
    ft, wst = o.tensor_footprints()
    assert fo.tolist() == [2 * MiB, 0] and wso == 2 * MiB
    assert ft.tolist() == [512, 0] and wst == 512
    assert o.tensor_counts[:1].tolist() == [1] and o.untensored == 0


def test_tensor_counts_hand_worked():
    """Two objects; tensors at the start, middle and end of the first; accesses inside a
    tensor, in an object outside its tensors, in a gap and outside the window."""
    base = 1 << 30
    o = OracleTrace(base, base + 16 * MiB, 4, 4, max_live_tensors=8, max_tensor_ids=8)
    o.register_alloc(base, 1 * MiB)             # id 0
    o.register_alloc(base + 2 * MiB, 1 * MiB)   # id 1
    assert o.register_tensor(base, 4096) == (oracle.OK, 0)
    assert o.register_tensor(base + 4096, 4096) == (oracle.OK, 1)          # adjacent to tensor 0
    assert o.register_tensor(base + MiB - 256, 256) == (oracle.OK, 2)      # ends at the object end
    rec = [base, base + 4095, base + 4096, base + 8191, base + 8192, base + MiB - 1, base + MiB,
           base + 2 * MiB + 5, base - 1, base + 32 * MiB]
    o.analyze(np.array(rec, dtype=np.uint64), [0, 4, 10], 12, kernel_rows=True)
    assert o.tensor_counts[:3].tolist() == [2, 2, 1]
    # untensored: base+8192 (object 0, no tensor), base+MiB (gap), object 1, base-1, outside
    assert o.untensored == 5
    assert o.alloc_counts[:2].tolist() == [6, 1]
    assert o.tensor_rows.tolist()[0][:3] == [2, 2, 0] and o.tensor_rows.tolist()[1][:3] == [0, 0, 1]
    # adjacent tensors 0 and 1 merge into one staged range
    assert o.prefetch_plan("tensor") == [[(base, base + 8192)], [(base + MiB - 256, base + MiB)]]
    assert o.prefetch_plan("object") == [[(base, base + MiB)], [(base, base + MiB), (base + 2 * MiB, base + 3 * MiB)]]


def test_tensor_registration_rules():
    o = OracleTrace(0, 1 << 30, 4, 4, max_live_tensors=2, max_tensor_ids=3)
    assert o.register_tensor(0x1000, 16)[0] == oracle.EINVAL            # no object
    o.register_alloc(0x1000, 0x1000)
    assert o.register_tensor(0x1F00, 0x200)[0] == oracle.EINVAL         # straddles the object end
    assert o.register_tensor(0x0F00, 0x200)[0] == oracle.EINVAL         # starts before the object
    assert o.register_tensor(0x1000, 0) [0] == oracle.EINVAL
    assert o.register_tensor(0x1100, 0x100) == (oracle.OK, 0)
    assert o.register_tensor(0x11FF, 0x10)[0] == oracle.EOVERLAP
    assert o.register_tensor(0x1200, 0x10) == (oracle.OK, 1)             # adjacent
    assert o.register_tensor(0x1400, 0x10)[0] == oracle.ECAPACITY        # 2 live
    assert o.register_tensor_free(0x1208) == oracle.ENOENT
    assert o.register_tensor_free(0x1200) == oracle.OK
    assert o.register_tensor(0x1400, 0x10) == (oracle.OK, 2)
    # R19: freeing the object ends its tensors
    assert o.register_free(0x1000) == oracle.OK
    assert o.register_tensor_free(0x1100) == oracle.ENOENT
    o.register_alloc(0x1000, 0x1000)
    assert o.register_tensor(0x1100, 0x100)[0] == oracle.ECAPACITY       # 3 tensor ids issued
    # a handle without a tensor level rejects tensors
    assert OracleTrace(0, 1 << 30, 4, 4).register_tensor(0x1000, 16)[0] == oracle.EINVAL


def _two_level_case(rng):
    """Objects in [lo, lo + 2^16), tensors inside them, records around them."""
    lo = rng.choice([0, 1 << 40, (1 << 64) - (1 << 17)])
    objs, tens = [], []
    cur = lo + rng.randrange(0, 64)
    for _ in range(rng.randint(0, 6)):
        b = cur + (0 if rng.random() < 0.3 else rng.randrange(0, 2048))
        sz = rng.randrange(1, 4096)
        if b + sz >= lo + (1 << 16):
            break
        objs.append((b, sz))
        cur = b + sz
    for b, sz in objs:
        t = b + (0 if rng.random() < 0.3 else rng.randrange(0, max(1, sz // 4)))
        while t < b + sz and rng.random() < 0.8:
            tsz = rng.randrange(1, max(2, (b + sz - t) // 2 + 1))
            if t + tsz > b + sz:
                break
            tens.append((t, tsz))
            t = t + tsz + (0 if rng.random() < 0.4 else rng.randrange(0, 256))
    hi = lo + (1 << 16)
    pts = [lo, hi - 1]
    for b, sz in objs + tens:
        pts += [b, b + sz - 1, b + sz, max(lo, b - 1)]
    recs = [rng.choice(pts) if rng.random() < 0.5 else rng.randrange(lo, hi) for _ in range(rng.randint(0, 120))]
    n = len(recs)
    nk = rng.randint(1, 4)
    ko = [0] + sorted(rng.randint(0, n) for _ in range(nk - 1)) + [n]
    return lo, hi, objs, tens, recs, ko


def _coverage_union(intervals, lo, hi):
    """Union by byte coverage over [lo, hi): a boolean array, then its runs."""
    cov = np.zeros(hi - lo, dtype=bool)
    for a, b in intervals:
        cov[a - lo:b - lo] = True
    out = []
    i = 0
    while i < cov.size:
        if cov[i]:
            j = i
            while j < cov.size and cov[j]:
                j += 1
            out.append((lo + i, lo + j))
            i = j
        else:
            i += 1
    return out


def test_tensor_level_brute_force():
    rng = random.Random(77)
    for case in range(400):
        lo, hi, objs, tens, recs, ko = _two_level_case(rng)
        o = OracleTrace(lo, hi, 8, 8, max_live_tensors=64, max_tensor_ids=64)
        for b, sz in objs:
            assert o.register_alloc(b, sz)[0] == oracle.OK, case
        for b, sz in tens:
            assert o.register_tensor(b, sz)[0] == oracle.OK, (case, b, sz)
        o.analyze(np.array(recs, dtype=np.uint64), ko, 12, kernel_rows=True)
        tlive = [(b, sz, t) for t, (b, sz) in enumerate(tens)]
        olive = [(b, sz, i) for i, (b, sz) in enumerate(objs)]
        bt = brute.analyze(tlive, recs, ko, lo, hi, 12, 64)
        bo = brute.analyze(olive, recs, ko, lo, hi, 12, 8)
        assert o.tensor_counts.tolist() == bt["alloc"], case
        assert o.untensored == bt["unattr"], case
        assert o.tensor_rows.tolist() == bt["kac"], case
        assert o.alloc_counts.tolist() == bo["alloc"], case
        assert int(o.tensor_counts.sum()) + o.untensored == len(recs), case
        ft, wst = o.tensor_footprints()
        bft = brute.footprints(bt["kac"], [sz for _, sz in tens] + [0] * (64 - len(tens)))
        assert ft.tolist() == bft and wst == max(bft), case
        pt, po = o.prefetch_plan("tensor"), o.prefetch_plan("object")
        for k in range(len(ko) - 1):
            touched_t = [(b, b + sz) for t, (b, sz) in enumerate(tens) if bt["kac"][k][t]]
            touched_o = [(b, b + sz) for i, (b, sz) in enumerate(objs) if bo["kac"][k][i]]
            assert pt[k] == _coverage_union(touched_t, lo, hi), (case, k)
            assert po[k] == _coverage_union(touched_o, lo, hi), (case, k)
            # S:514 / S:546: tensor plan inside the object plan, never more bytes
            assert _bytes(pt[k]) <= _bytes(po[k]), (case, k)
            for a, b in pt[k]:
                assert any(x <= a and b <= y for x, y in po[k]), (case, k)


def test_tensor_level_accumulates_and_respects_snapshots():
    """Two analyze calls accumulate; a tensor freed between them stops counting (R13)."""
    base = 1 << 32
    o = OracleTrace(base, base + MiB, 4, 4, max_live_tensors=4, max_tensor_ids=4)
    o.register_alloc(base, 65536)
    o.register_tensor(base, 4096)
    o.register_tensor(base + 4096, 4096)
    rec = np.array([base + 10, base + 5000, base + 9000], dtype=np.uint64)
    o.analyze(rec, None, 12)
    o.register_tensor_free(base + 4096)
    o.analyze(rec, None, 12)
    assert o.tensor_counts[:2].tolist() == [2, 1]
    assert o.untensored == 1 + 2
    assert o.alloc_counts[:1].tolist() == [6]
