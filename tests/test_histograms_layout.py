"""Host logic of the binding's Histograms (CPU tensors): every output is a view of one
zero-initialised arena at a 256-byte aligned offset, the packed layout
[page_counts | alloc_counts | totals | tensor_counts] the mergers rely on, and zero_()
resetting every part with one fill."""
import pytest

torch = pytest.importorskip("torch")

import paper_2602_22103_b200 as pb  # noqa: E402


@pytest.mark.parametrize("kw", [dict(), dict(n_kernels=7, kernel_rows=True), dict(n_kernels=5, kernel_rows=True, kernel_pages=True),
                                dict(n_kernels=9, kernel_rows=True, window_kernels=4, max_tensor_ids=3, pad_pages_to=128),
                                dict(bitmap=False)])
def test_arena_views(kw):
    P, max_ids = 1000, 13
    h = pb.Histograms(P, max_ids, torch.device("cpu"), **kw)
    base = h.arena.data_ptr()
    parts = {n: getattr(h, n) for n in ("packed", "page_bitmap", "kernel_alloc_counts", "kernel_stats",
                                         "kernel_page_bitmap", "hotness", "kernel_tensor_counts",
                                         "kernel_tensor_footprint")}
    spans = []
    for name, t in parts.items():
        if t is None:
            continue
        assert t.untyped_storage().data_ptr() == h.arena.untyped_storage().data_ptr(), name
        off = t.data_ptr() - base
        assert off % 256 == 0, name
        spans.append((off, off + 8 * t.numel(), name))
    spans.sort()
    for (a0, a1, n0), (b0, b1, n1) in zip(spans, spans[1:]):
        assert a1 <= b0, (n0, n1)  # disjoint
    assert h.page_counts.numel() == P and h.alloc_counts.numel() == max_ids and h.totals.numel() == pb.TOTALS
    assert h.page_counts.data_ptr() == h.packed.data_ptr()
    assert h.alloc_counts.data_ptr() == h.packed.data_ptr() + 8 * h.P_pad
    assert h.small.data_ptr() == h.alloc_counts.data_ptr() and h.P_pad % kw.get("pad_pages_to", 1) == 0
    if kw.get("kernel_rows"):
        assert h.kernel_alloc_counts.numel() == kw["n_kernels"] * max_ids
        assert h.kernel_stats.numel() == kw["n_kernels"] * pb.KSTATS
    if kw.get("window_kernels"):
        assert h.hotness.numel() == h.n_windows * P
    h.arena.fill_(7)
    h.zero_()
    assert int(h.arena.abs().sum()) == 0
