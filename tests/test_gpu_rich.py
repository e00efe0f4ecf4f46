"""GPU parity of the rich-record analysis (NEXT f4; R21-R24): the CUDA path
through pasta_analyze_rich against the oracle (oracle_analyze_rich), bit-exact.

* the rich generator's device version against its host version;
* SPEC's range-filter examples (window [0,0] on a 3-kernel trace; full window = the
  8-byte analysis of the same addresses);
* 40 random rich traces (interleaved grid ids, writes, sizes 1-128, shared records,
  partial windows), replicated to span many slices;
* the tiny config and a 2^24-record llama prefix as rich traces (5 % of records from
  the previous kernel), full and partial windows: every output including write
  counts, byte weights, the dropped counts and MAX_MEM_REFERENCED_KERNEL.
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
from tests.test_oracle_rich import _pack, _random_rich, _three_kernel_trace  # noqa: E402
from tracegen.rich import RICH_DTYPE, rich_device, rich_host  # noqa: E402

DEV = torch.device("cuda:0")


def _dev_rich(rec):
    rec = np.ascontiguousarray(rec, dtype=RICH_DTYPE)
    if rec.size == 0:
        return torch.zeros((0, 2), dtype=torch.int64, device=DEV)
    return torch.from_numpy(rec.view(np.int64).reshape(-1, 2).copy()).to(DEV)


def _run(va_lo, va_hi, live, rec, g0, g1, s=12, misalign=False, rows=True):
    A = max(1, len(live))
    tr = pb.Trace(DEV, va_lo, va_hi, A, A)
    o = OracleTrace(va_lo, va_hi, A, A)
    for b, sz in live:
        tr.register_alloc(b, sz)
        o.register_alloc(b, sz)
    nk = g1 - g0 + 1
    h = tr.histograms(s, n_kernels=nk, kernel_rows=rows)
    rx = tr.rich_outputs(s)
    tr.analyze_rich(_dev_rich(rec), g0, g1, s, h, rx)
    tr.sync()
    o.analyze_rich(rec, g0, g1, s, kernel_rows=rows)
    g = dict(page=u64(h.page_counts), alloc=u64(h.alloc_counts), tot=u64(h.totals),
             kac=u64(h.kernel_alloc_counts).reshape(nk, -1) if rows else None,
             kst=u64(h.kernel_stats).reshape(nk, 4) if rows else None,
             pw=u64(rx.page_write_counts), aw=u64(rx.alloc_write_counts), ab=u64(rx.alloc_bytes),
             rt=u64(rx.rich_totals), bm=u64(h.page_bitmap))
    tr.close()
    return g, o


def _assert(g, o, label, rows=True):
    assert np.array_equal(g["page"], o.page_counts), f"{label}: page_counts"
    assert np.array_equal(g["pw"], o.page_writes), f"{label}: page_write_counts"
    assert np.array_equal(g["alloc"], o.alloc_counts), f"{label}: alloc_counts"
    assert np.array_equal(g["aw"], o.alloc_writes), f"{label}: alloc_write_counts"
    assert np.array_equal(g["ab"], o.alloc_bytes), f"{label}: alloc_bytes"
    assert g["tot"][:3].tolist() == o.totals.tolist(), f"{label}: totals"
    assert np.array_equal(g["rt"], o.rich_totals), f"{label}: rich_totals"
    bm, u = o.bitmap()
    assert np.array_equal(g["bm"], bm) and int(g["tot"][3]) == u, f"{label}: bitmap"
    if not rows:
        return
    assert np.array_equal(g["kac"], o.kernel_rows), f"{label}: kernel rows"
    assert np.array_equal(g["kst"][:, 1], o.kun), f"{label}: kernel unattributed"
    fp, ws = o.footprints()
    assert np.array_equal(g["kst"][:, 2], fp) and int(g["tot"][4]) == ws, f"{label}: footprints"
    assert int(g["tot"][pb.T_MAX_KERNEL]) == o.max_kernel(), f"{label}: max kernel"


def test_rich_generator_device_matches_host():
    p = tracegen.build_plan("llama")
    n = 1 << 20
    addr = tracegen.host_records(p, 5_000_000, 5_000_000 + n)
    ko = np.asarray(p.kernel_offsets, dtype=np.int64)
    hr = rich_host(addr, ko, seed=7, j0=5_000_000)
    dr = rich_device(_dev_rich_addr(addr), torch.from_numpy(ko).to(DEV), seed=7, j0=5_000_000)
    assert np.array_equal(dr.cpu().numpy().reshape(-1).view(np.uint8), hr.view(np.uint8))


def _dev_rich_addr(addr):
    return torch.from_numpy(np.ascontiguousarray(addr, dtype=np.uint64).view(np.int64)).to(DEV)


def test_spec_range_filter_examples_on_gpu():
    base, live, addrs, ko, rich = _three_kernel_trace()
    lv = [(b, sz) for b, sz, _ in live]
    g, o = _run(base, base + (1 << 20), lv, rich, 0, 0)
    _assert(g, o, "window [0,0]")
    assert int(g["tot"][0]) == 100 and int(g["rt"][0]) == 67
    g, o = _run(base, base + (1 << 20), lv, rich, 0, 2)
    _assert(g, o, "full window")


def test_random_rich_traces():
    rng = random.Random(808)
    for case in range(40):
        lo, hi, live, recs, g0, g1 = _random_rich(rng)
        rec = _pack(recs)
        if rng.random() < 0.5 and rec.size:
            rec = np.tile(rec, rng.randint(20, 2000))
        g, o = _run(lo, hi, [(b, sz) for b, sz, _ in live], rec, g0, g1)
        _assert(g, o, f"case {case}")


@pytest.mark.parametrize("window", ["full", "part"])
def test_tiny_rich(window):
    p = tracegen.build_plan("tiny", seed=2)
    addr = tracegen.host_records(p)
    rec = rich_host(addr, p.kernel_offsets, seed=3, grid_base=100)
    g0, g1 = (100, 107) if window == "full" else (102, 105)
    g, o = _run(p.va_lo, p.va_hi, p.allocs, rec, g0, g1, s=p.page_shift)
    _assert(g, o, f"tiny {window}")


def test_llama_prefix_rich():
    p = tracegen.build_plan("llama")
    n = 1 << 24
    addr = tracegen.host_records(p, 0, n)
    rec = rich_host(addr, p.kernel_offsets, seed=11)
    kmax = int(np.searchsorted(np.asarray(p.kernel_offsets, dtype=np.int64), n, side="left"))
    g, o = _run(p.va_lo, p.va_hi, p.allocs, rec, 0, kmax, s=p.page_shift)
    _assert(g, o, "llama prefix")
    assert int(g["rt"][3]) > 0 and int(g["rt"][2]) > 0


def test_rich_errors():
    tr = pb.Trace(DEV, 0, 1 << 30, 2, 2)
    h = tr.histograms(12, n_kernels=2, kernel_rows=True, kernel_pages=True)
    rx = tr.rich_outputs(12)
    rec = torch.zeros((4, 2), dtype=torch.int64, device=DEV)
    with pytest.raises(pb.PastaError) as ei:  # per-kernel page bitmaps are not offered for rich records
        tr.analyze_rich(rec, 0, 1, 12, h, rx)
    assert ei.value.status == pb.PASTA_EINVAL
    h2 = tr.histograms(12, n_kernels=2, kernel_rows=True)
    with pytest.raises(pb.PastaError) as ei:  # grid_lo > grid_hi
        tr.analyze_rich(rec, 3, 1, 12, h2, rx)
    assert ei.value.status == pb.PASTA_EINVAL
    buf = torch.zeros(9, dtype=torch.int64, device=DEV)
    with pytest.raises(pb.PastaError) as ei:  # records not 16-byte aligned
        pb.pasta_analyze_rich(tr.h, buf[1:], 4, 0, 1, 12, h2.struct(), rx.struct())
    assert ei.value.status == pb.PASTA_EINVAL
    tr.close()


@pytest.mark.parametrize("mix,block_log2,rows", [(0.0, 0, True), (0.05, 5, True), (0.05, 5, False), (0.3, 0, True),
                                                 (0.05, 0, False), (0.5, 3, True)])
def test_llama_prefix_rich_mixes(mix, block_log2, rows):
    """Concurrent-kernel mixes that select each scan tier: one kernel per slice (tier RC),
    warp-sized bursts of the previous kernel (tier RC with two kernels), single records
    of it (two-kernel tier, fast path), heavy mixing (leader loop); with and without
    kernel rows. Partial grid window so some slices mix filtered records."""
    p = tracegen.build_plan("llama")
    n = (1 << 22) + 77
    j0 = 3 << 22
    addr = tracegen.host_records(p, j0, j0 + n)
    rec = rich_host(addr, p.kernel_offsets, seed=5, mix=mix, j0=j0, block_log2=block_log2)
    ko = np.asarray(p.kernel_offsets, dtype=np.int64)
    k0 = int(np.searchsorted(ko, j0, side="right")) - 1
    k1 = int(np.searchsorted(ko, j0 + n, side="left"))
    for g0, g1 in ((k0 - 1, k1), (k0 + 2, k1 - 3)):
        g, o = _run(p.va_lo, p.va_hi, p.allocs, rec, g0, g1, s=p.page_shift, rows=rows)
        _assert(g, o, f"mix={mix} blk={block_log2} rows={rows} window=[{g0},{g1}]", rows=rows)
