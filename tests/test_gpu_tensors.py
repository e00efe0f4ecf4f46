"""GPU parity of the tensor level and the prefetch-plan builder (NEXT f3; DESIGN.md
R18-R20): the CUDA path through the C ABI against the oracle, bit-exact.

* hand-worked two-level trace and SPEC's plan examples;
* random two-level registrations (tests/test_oracle_tensors.py's generator) under both
  scan schedules, every output: object level, tensor counts, untensored, per-kernel
  tensor rows, tensor footprints / WS_tensor, object and tensor plans;
* the tiny config with objects = 4 MiB blocks and tensors = its allocations, whole
  trace; the uvm config at full size (objects = pool chunks, tensors = its ~1,700
  allocations) checked on sampled kernels, conservation, and plans recomputed by the
  oracle from the GPU's rows (the plan kernel at 2,000 rows).
"""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2602_22103_b200 as pb  # noqa: E402
import oracle  # noqa: E402
import tracegen  # noqa: E402
from oracle import OracleTrace  # noqa: E402
from tests.harness import u64  # noqa: E402
from tests.test_oracle_tensors import _two_level_case  # noqa: E402

DEV = torch.device("cuda:0")
MiB = 1 << 20


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(DEV)


def _plan_rows(offsets, ranges):
    off = u64(offsets)
    rg = u64(ranges).reshape(-1, 2)
    return [[(int(a), int(b)) for a, b in rg[off[k]:off[k + 1]]] for k in range(off.size - 1)]


def _run_both(va_lo, va_hi, objs, tens, recs, ko, page_shift=12, schedule="auto", max_ids=None, max_tids=None):
    max_ids = max_ids or max(1, len(objs))
    max_tids = max_tids or max(1, len(tens))
    tr = pb.Trace(DEV, va_lo, va_hi, max(1, len(objs)), max_ids, schedule=schedule,
                  max_live_tensors=max(1, len(tens)), max_tensor_ids=max_tids)
    o = OracleTrace(va_lo, va_hi, max(1, len(objs)), max_ids, max_live_tensors=max(1, len(tens)),
                    max_tensor_ids=max_tids)
    for b, s in objs:
        tr.register_alloc(b, s)
        assert o.register_alloc(b, s)[0] == oracle.OK
    for b, s in tens:
        tr.register_tensor(b, s)
        assert o.register_tensor(b, s)[0] == oracle.OK
    nk = len(ko) - 1
    h = tr.histograms(page_shift, n_kernels=nk, kernel_rows=True)
    rec = np.asarray(recs, dtype=np.uint64)
    drec = _t(rec) if rec.size else torch.zeros(0, dtype=torch.int64, device=DEV)
    tr.analyze(drec, page_shift, h, kernel_offsets=_t(np.asarray(ko, dtype=np.uint64)))
    po_off, po_rg = tr.prefetch_plan(h, "object")
    pt_off, pt_rg = tr.prefetch_plan(h, "tensor")
    tr.sync()
    o.analyze(rec, ko, page_shift, kernel_rows=True)
    g = dict(alloc=u64(h.alloc_counts), tot=u64(h.totals), tc=u64(h.tensor_counts),
             kac=u64(h.kernel_alloc_counts).reshape(nk, -1), ktc=u64(h.kernel_tensor_counts).reshape(nk, -1),
             kst=u64(h.kernel_stats).reshape(nk, 4), ktf=u64(h.kernel_tensor_footprint),
             plan_o=_plan_rows(po_off, po_rg), plan_t=_plan_rows(pt_off, pt_rg))
    tr.close()
    return g, o


def _assert_tensor_parity(g, o, label):
    assert np.array_equal(g["alloc"], o.alloc_counts), f"{label}: alloc_counts"
    assert int(g["tot"][1]) == int(o.totals[1]), f"{label}: unattributed"
    assert np.array_equal(g["tc"], o.tensor_counts), f"{label}: tensor_counts"
    assert int(g["tot"][pb.T_UNTENSORED]) == o.untensored, f"{label}: untensored"
    assert np.array_equal(g["kac"], o.kernel_rows), f"{label}: kernel_alloc_counts"
    assert np.array_equal(g["ktc"], o.tensor_rows), f"{label}: kernel_tensor_counts"
    fo, wso = o.footprints()
    ft, wst = o.tensor_footprints()
    assert np.array_equal(g["kst"][:, 2], fo) and int(g["tot"][pb.T_WS_OBJ]) == wso, f"{label}: object footprints"
    assert np.array_equal(g["ktf"], ft), f"{label}: tensor footprints"
    assert int(g["tot"][pb.T_WS_TENSOR]) == wst, f"{label}: WS_tensor"
    assert g["plan_o"] == o.prefetch_plan("object"), f"{label}: object plan"
    assert g["plan_t"] == o.prefetch_plan("tensor"), f"{label}: tensor plan"


def test_spec_plan_example_on_gpu():
    O = 0x7F0000200000
    g, o = _run_both(0x7F0000000000, 0x7F0000000000 + 64 * MiB, [(O, 2 * MiB)], [(O + 4096, 512)],
                     [O + 4096 + 100], [0, 1, 1], page_shift=21)
    _assert_tensor_parity(g, o, "spec")
    assert g["plan_o"] == [[(O, O + 2 * MiB)], []]
    assert g["plan_t"] == [[(O + 4096, O + 4096 + 512)], []]


def test_hand_worked_two_level_on_gpu():
    base = 1 << 30
    objs = [(base, MiB), (base + 2 * MiB, MiB)]
    tens = [(base, 4096), (base + 4096, 4096), (base + MiB - 256, 256)]
    rec = [base, base + 4095, base + 4096, base + 8191, base + 8192, base + MiB - 1, base + MiB,
           base + 2 * MiB + 5, base - 1, base + 32 * MiB]
    g, o = _run_both(base, base + 16 * MiB, objs, tens, rec, [0, 4, 10])
    _assert_tensor_parity(g, o, "hand")
    assert g["tc"][:3].tolist() == [2, 2, 1] and int(g["tot"][pb.T_UNTENSORED]) == 5


@pytest.mark.parametrize("schedule", ["contiguous", "interleaved"])
def test_random_two_level(schedule):
    rng = random.Random(5150)
    for case in range(60):
        lo, hi, objs, tens, recs, ko = _two_level_case(rng)
        # grow some traces past one slice per warp so several tiers run
        if rng.random() < 0.3 and recs:
            recs = recs * rng.randint(50, 3000)
            n = len(recs)
            ko = [0] + sorted(rng.randint(0, n) for _ in range(len(ko) - 2)) + [n]
        g, o = _run_both(lo, hi, objs, tens, recs, ko, schedule=schedule, max_ids=8, max_tids=64)
        _assert_tensor_parity(g, o, f"case {case} {schedule}")


def test_tiny_config_two_level():
    p = tracegen.build_plan("tiny", seed=11)
    rec = tracegen.host_records(p)
    ko = [int(x) for x in p.kernel_offsets]
    g, o = _run_both(p.va_lo, p.va_hi, p.objects, p.allocs, rec, ko, page_shift=p.page_shift)
    _assert_tensor_parity(g, o, "tiny two-level")
    # tensor plans never stage more than object plans
    for rt, ro in zip(g["plan_t"], g["plan_o"]):
        assert sum(b - a for a, b in rt) <= sum(b - a for a, b in ro)


def test_uvm_two_level_full_size():
    """uvm at full size (4e9 records): objects = pool chunks, tensors = allocations."""
    p = tracegen.build_plan("uvm")
    free = torch.cuda.mem_get_info(DEV)[0]
    if p.n * 8 + (4 << 30) > free:
        pytest.skip("needs device memory for the full trace")
    dp = tracegen.DevicePlan(p, DEV)
    drec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(dp, drec)
    tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.objects), len(p.objects), max_live_tensors=len(p.allocs),
                  max_tensor_ids=len(p.allocs))
    for b, s in p.objects:
        tr.register_alloc(b, s)
    for b, s in p.allocs:
        tr.register_tensor(b, s)
    nk = p.n_kernels
    h = tr.histograms(p.page_shift, n_kernels=nk, kernel_rows=True)
    ko = [int(x) for x in p.kernel_offsets]
    tr.analyze(drec, p.page_shift, h, kernel_offsets=_t(np.asarray(ko, dtype=np.uint64)))
    po = _plan_rows(*tr.prefetch_plan(h, "object"))
    pt = _plan_rows(*tr.prefetch_plan(h, "tensor"))
    tr.sync()
    del drec
    torch.cuda.empty_cache()
    tc, tot = u64(h.tensor_counts), u64(h.totals)
    kac = u64(h.kernel_alloc_counts).reshape(nk, -1)
    ktc = u64(h.kernel_tensor_counts).reshape(nk, -1)
    n = p.n
    assert int(tot[0]) == n
    assert int(tc.sum()) + int(tot[pb.T_UNTENSORED]) == n
    assert int(u64(h.alloc_counts).sum()) + int(tot[1]) == n
    assert np.array_equal(ktc.sum(axis=0), tc)
    # every tensor lies in one object, so per-object tensor sums never exceed the object count
    ob = [b for b, _ in p.objects]
    per_obj = np.zeros(len(p.objects), dtype=np.uint64)
    for t, (b, s) in enumerate(p.allocs):
        per_obj[np.searchsorted(ob, b, side="right") - 1] += tc[t]
    assert np.all(per_obj <= u64(h.alloc_counts))
    # plans = the oracle's union over the GPU's rows
    obase, osz = [b for b, _ in p.objects], [s for _, s in p.objects]
    tbase, tsz = [b for b, _ in p.allocs], [s for _, s in p.allocs]
    for k in range(nk):
        assert po[k] == oracle.interval_union([(obase[i], obase[i] + osz[i]) for i in np.nonzero(kac[k])[0]]), k
        assert pt[k] == oracle.interval_union([(tbase[i], tbase[i] + tsz[i]) for i in np.nonzero(ktc[k])[0]]), k
        assert sum(b - a for a, b in pt[k]) <= sum(b - a for a, b in po[k]), k
    # sampled kernels recomputed by the oracle from host-generated records
    rng = random.Random(3)
    for k in sorted(set([0, nk - 1] + [rng.randrange(nk) for _ in range(4)])):
        j0, j1 = ko[k], ko[k + 1]
        if j1 - j0 > 40_000_000:
            continue
        rec = tracegen.host_records(p, j0, j1)
        o = OracleTrace(p.va_lo, p.va_hi, len(p.objects), len(p.objects), max_live_tensors=len(p.allocs),
                        max_tensor_ids=len(p.allocs))
        for b, s in p.objects:
            o.register_alloc(b, s)
        for b, s in p.allocs:
            o.register_tensor(b, s)
        o.analyze(rec, [0, j1 - j0], p.page_shift, kernel_rows=True)
        assert np.array_equal(kac[k], o.kernel_rows[0]), k
        assert np.array_equal(ktc[k], o.tensor_rows[0]), k
    tr.close()


def test_tensor_errors_are_status_codes():
    tr = pb.Trace(DEV, 0, 1 << 30, 4, 4, max_live_tensors=2, max_tensor_ids=3)
    with pytest.raises(pb.PastaError) as ei:
        tr.register_tensor(0x1000, 16)  # no object
    assert ei.value.status == pb.PASTA_EINVAL
    tr.register_alloc(0x1000, 0x1000)
    for b, s, st in [(0x1F00, 0x200, pb.PASTA_EINVAL), (0x0F00, 0x200, pb.PASTA_EINVAL), (0x1000, 0, pb.PASTA_EINVAL)]:
        with pytest.raises(pb.PastaError) as ei:
            tr.register_tensor(b, s)
        assert ei.value.status == st
    assert tr.register_tensor(0x1100, 0x100) == 0
    with pytest.raises(pb.PastaError) as ei:
        tr.register_tensor(0x11FF, 0x10)
    assert ei.value.status == pb.PASTA_EOVERLAP
    assert tr.register_tensor(0x1200, 0x10) == 1
    with pytest.raises(pb.PastaError) as ei:
        tr.register_tensor(0x1400, 0x10)
    assert ei.value.status == pb.PASTA_ECAPACITY
    tr.register_free(0x1000)  # R19: ends both tensors
    with pytest.raises(pb.PastaError) as ei:
        tr.register_tensor_free(0x1100)
    assert ei.value.status == pb.PASTA_ENOENT
    # tensor outputs on a handle without a tensor level, and plans at a missing level
    tr2 = pb.Trace(DEV, 0, 1 << 30, 4, 4)
    with pytest.raises(pb.PastaError) as ei:
        tr2.register_tensor(0x1000, 16)
    assert ei.value.status == pb.PASTA_EINVAL
    h = tr2.histograms(12, n_kernels=1, kernel_rows=True)
    off = torch.empty(2, dtype=torch.int64, device=DEV)
    with pytest.raises(pb.PastaError) as ei:
        pb.pasta_prefetch_plan(tr2.h, h.kernel_alloc_counts, 1, pb.LEVEL_TENSOR, off, None, 0)
    assert ei.value.status == pb.PASTA_EINVAL
    st, total = pb.pasta_prefetch_plan(tr2.h, h.kernel_alloc_counts, 1, pb.LEVEL_OBJECT, off, None, 0)
    assert st == pb.PASTA_OK and total == 0
    tr.close()
    tr2.close()
