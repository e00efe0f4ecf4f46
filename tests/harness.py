"""Shared test helpers: run the CUDA path (through the C ABI binding) and the oracle
on the same seeded inputs and return comparable numpy arrays. Test-only."""
from __future__ import annotations

import numpy as np

import oracle

U64MAX = (1 << 64) - 1


def u64(t):
    """int64 CUDA/CPU tensor -> numpy uint64 (bit pattern)."""
    return t.detach().cpu().numpy().view(np.uint64)


def gpu_trace(device, va_lo, va_hi, ranges, max_ids=None, max_live=None, frees=(), schedule="auto"):
    import paper_2602_22103_b200 as pb

    max_ids = max_ids or max(1, len(ranges))
    max_live = max_live or max(1, len(ranges))
    tr = pb.Trace(device, va_lo, va_hi, max_live, max_ids, schedule=schedule)
    for b, s in ranges:
        tr.register_alloc(b, s)
    return tr


def oracle_trace(va_lo, va_hi, ranges, max_ids=None, max_live=None):
    max_ids = max_ids or max(1, len(ranges))
    max_live = max_live or max(1, len(ranges))
    o = oracle.OracleTrace(va_lo, va_hi, max_live, max_ids)
    for b, s in ranges:
        st, _ = o.register_alloc(b, s)
        assert st == oracle.OK
    return o


def run_gpu(tr, records, page_shift, kernel_offsets=None, kernel_rows=False, kernel_pages=False, topk=(),
            hist=None, finalize=True, host=False, n=None, window_kernels=0):
    """records: CUDA int64 tensor (or pinned CPU tensor with host=True)."""
    import torch

    nk = 0 if kernel_offsets is None else len(kernel_offsets) - 1
    if hist is None:
        hist = tr.histograms(page_shift, n_kernels=nk, kernel_rows=kernel_rows, kernel_pages=kernel_pages,
                             window_kernels=window_kernels)
    ko = None
    if kernel_offsets is not None:
        ko = torch.tensor(np.asarray(kernel_offsets, dtype=np.uint64).view(np.int64), dtype=torch.int64)
        ko = ko.pin_memory() if host else ko.to(tr.device)
    tr.analyze(records, page_shift, hist, kernel_offsets=ko, finalize=finalize, host=host, n=n)
    out = {"hist": hist}
    # every requested list from one selection (pasta_topk_many: pasta_topk of the largest
    # k, prefixes for the others); tests/test_gpu_parity.py covers pasta_topk per k
    tops = tr.topk_many(hist.page_counts, list(dict.fromkeys(topk))) if topk else {}
    tr.sync()
    out["page_counts"] = u64(hist.page_counts)
    out["alloc_counts"] = u64(hist.alloc_counts)
    out["totals"] = u64(hist.totals)
    if hist.page_bitmap is not None:
        out["bitmap"] = u64(hist.page_bitmap)
    if hist.kernel_alloc_counts is not None:
        out["kac"] = u64(hist.kernel_alloc_counts).reshape(hist.n_kernels, -1)[:nk]
        out["kstats"] = u64(hist.kernel_stats).reshape(hist.n_kernels, 4)[:nk]
    if hist.kernel_page_bitmap is not None:
        out["kpb"] = u64(hist.kernel_page_bitmap).reshape(hist.n_kernels, -1)[:nk]
    if hist.hotness is not None:
        out["hot"] = u64(hist.hotness).reshape(hist.n_windows, -1)
    out["topk"] = {K: (u64(p), u64(c), int(u64(f)[0])) for K, (p, c, f) in tops.items()}
    return out


def run_oracle(o, records_np, page_shift, kernel_offsets=None, kernel_rows=False, kernel_pages=False, topk=(),
               window_kernels=0):
    o.analyze(records_np, kernel_offsets, page_shift, kernel_rows=kernel_rows, kernel_pages=kernel_pages,
              window_kernels=window_kernels)
    return oracle_results(o, kernel_rows=kernel_rows, kernel_pages=kernel_pages, topk=topk,
                          window_kernels=window_kernels)


def oracle_results(o, kernel_rows=False, kernel_pages=False, topk=(), window_kernels=0):
    """Every output of an OracleTrace after its analyze calls, in assert_parity's form."""
    out = {"page_counts": o.page_counts.copy(), "alloc_counts": o.alloc_counts.copy(), "totals3": o.totals.copy()}
    bm, u = o.bitmap()
    out["bitmap"], out["unique"] = bm, u
    if kernel_rows:
        out["kac"] = o.kernel_rows.copy()
        out["kun"] = o.kun.copy()
        fp, ws = o.footprints()
        out["footprint"], out["ws"] = fp, ws
        out["max_kernel"] = o.max_kernel()
        per = o.kernel_rows.sum(axis=1, dtype=np.uint64) + o.kun
        out["max_kernel_records"] = int(per[out["max_kernel"]]) if per.size else 0
    if kernel_pages:
        out["kpb"] = o.kernel_pages.copy()
        out["kup"] = o.kernel_unique_pages()
    if window_kernels:
        out["hot"] = o.hotness.copy()
    out["topk"] = {K: o.topk(K) for K in topk}
    return out


def assert_parity(g, r, kernel_rows=False, kernel_pages=False, label=""):
    """Bit-exact comparison of every output."""
    assert np.array_equal(g["page_counts"], r["page_counts"]), f"{label}: page_counts"
    assert np.array_equal(g["alloc_counts"], r["alloc_counts"]), f"{label}: alloc_counts"
    assert int(g["totals"][0]) == int(r["totals3"][0]), f"{label}: records"
    assert int(g["totals"][1]) == int(r["totals3"][1]), f"{label}: unattributed"
    assert int(g["totals"][2]) == int(r["totals3"][2]), f"{label}: out_of_window"
    assert int(g["totals"][3]) == r["unique"], f"{label}: unique_pages"
    if "bitmap" in g:
        assert np.array_equal(g["bitmap"], r["bitmap"]), f"{label}: bitmap"
    if kernel_rows:
        assert np.array_equal(g["kac"], r["kac"]), f"{label}: kernel_alloc_counts"
        ks = g["kstats"]
        assert np.array_equal(ks[:, 0], r["kac"].sum(axis=1).astype(np.uint64)), f"{label}: kstats attributed"
        assert np.array_equal(ks[:, 1], r["kun"]), f"{label}: kstats unattributed"
        assert np.array_equal(ks[:, 2], r["footprint"]), f"{label}: footprint"
        assert int(g["totals"][4]) == r["ws"], f"{label}: ws_obj"
        assert int(g["totals"][7]) == r["max_kernel"], f"{label}: max_mem_referenced_kernel"
        assert int(g["totals"][8]) == r["max_kernel_records"], f"{label}: max_mem_referenced_kernel records"
    if kernel_pages:
        assert np.array_equal(g["kpb"], r["kpb"]), f"{label}: kernel_page_bitmap"
        assert np.array_equal(g["kstats"][:, 3], r["kup"]), f"{label}: kernel unique pages"
    if "hot" in g or "hot" in r:
        assert np.array_equal(g["hot"], r["hot"]), f"{label}: hotness"
    for K, (p, c, f) in g["topk"].items():
        rp, rc, rf = r["topk"][K]
        assert f == rf, f"{label}: top{K} found {f} != {rf}"
        assert np.array_equal(p, rp) and np.array_equal(c, rc), f"{label}: top{K} list"
