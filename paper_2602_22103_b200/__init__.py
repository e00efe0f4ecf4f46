"""paper_2602_22103_b200 -- thin Python binding of the PASTA trace-analysis C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
libpasta.so (include/pasta.h). The functions keep the C names; ``PastaError`` is
raised for a non-zero status. PyTorch supplies device memory and streams only.
There is no CPU fallback: importing this package fails loudly if libpasta.so is
missing, and opening a handle fails without a CUDA device.

Convenience layer (still marshalling only):
  * ``Histograms`` allocates the output arrays as views into ONE packed int64
    device buffer ``[page_counts | alloc_counts | totals | ...]`` so the multi-GPU
    merge is a single all_reduce (see .dist);
  * ``Trace`` wraps a handle with register / analyze / topk methods.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PASTA_LIB selects an alternative build of the same C ABI (A/B performance runs).
_LIB_PATH = os.environ.get("PASTA_LIB") or os.path.join(_HERE, "libpasta.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(_LIB_PATH)

PASTA_OK, PASTA_EINVAL, PASTA_EOVERLAP, PASTA_ENOENT, PASTA_ECAPACITY, PASTA_ECUDA, PASTA_ESTATE, PASTA_ENOMEM = (
    0, -1, -2, -3, -4, -5, -6, -7)
T_RECORDS, T_UNATTRIBUTED, T_OUT_OF_WINDOW, T_UNIQUE_PAGES, T_WS_OBJ, TOTALS = 0, 1, 2, 3, 4, 9
T_UNTENSORED, T_WS_TENSOR, T_MAX_KERNEL, T_MAX_KERNEL_RECORDS = 5, 6, 7, 8
RT_FILTERED, RT_SHARED, RT_WRITES, RT_BYTES, RICH_TOTALS = 0, 1, 2, 3, 4
ACC_WRITE, ACC_SHARED = 1, 2
LEVEL_OBJECT, LEVEL_TENSOR = 0, 1
K_ATTRIBUTED, K_UNATTRIBUTED, K_FOOTPRINT, K_UNIQUE_PAGES, KSTATS = 0, 1, 2, 3, 4
PASTA_REC_HOST = 1
PASTA_REC_STABLE = 2
PASTA_REC_CHAINED = 4
PASTA_NO_FINALIZE = 1
PASTA_SCHED_CONTIGUOUS = 1
PASTA_SCHED_INTERLEAVED = 2
_SCHED = {"auto": 0, "contiguous": PASTA_SCHED_CONTIGUOUS, "interleaved": PASTA_SCHED_INTERLEAVED}
PH_SCAN, PH_FINALIZE, PH_TOPK, PH_MERGE, PH_COPY, PH_PLAN, PHASES = 0, 1, 2, 3, 4, 5, 6
PHASE_NAMES = ("scan", "finalize", "topk", "merge", "copy", "plan")


class pasta_open_params(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("max_live", ctypes.c_uint32), ("max_ids", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("va_lo", ctypes.c_uint64), ("va_hi", ctypes.c_uint64),
                ("stream", ctypes.c_void_p), ("host_chunk_bytes", ctypes.c_uint64),
                ("max_live_tensors", ctypes.c_uint32), ("max_tensor_ids", ctypes.c_uint32)]


class pasta_records(ctypes.Structure):
    _fields_ = [("addr", ctypes.c_void_p), ("kernel_offsets", ctypes.c_void_p), ("n_kernels", ctypes.c_uint32),
                ("flags", ctypes.c_uint32)]


class pasta_histograms(ctypes.Structure):
    _fields_ = [("page_counts", ctypes.c_void_p), ("alloc_counts", ctypes.c_void_p), ("totals", ctypes.c_void_p),
                ("page_bitmap", ctypes.c_void_p), ("kernel_alloc_counts", ctypes.c_void_p),
                ("kernel_stats", ctypes.c_void_p), ("kernel_page_bitmap", ctypes.c_void_p),
                ("flags", ctypes.c_uint32), ("window_kernels", ctypes.c_uint32), ("hotness", ctypes.c_void_p),
                ("tensor_counts", ctypes.c_void_p), ("kernel_tensor_counts", ctypes.c_void_p),
                ("kernel_tensor_footprint", ctypes.c_void_p), ("kernel_row0", ctypes.c_uint64)]


class pasta_batch(ctypes.Structure):
    _fields_ = [("trace", pasta_records), ("n", ctypes.c_uint64), ("out", pasta_histograms)]


class pasta_peer_slot(ctypes.Structure):
    _fields_ = [("index", ctypes.c_uint32), ("op", ctypes.c_uint32)]


class pasta_peer_copy(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("n", ctypes.c_uint64), ("op", ctypes.c_uint32),
                ("pad", ctypes.c_uint32)]


class pasta_ipc_handle(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_ubyte * 64), ("offset", ctypes.c_uint64), ("block_bytes", ctypes.c_uint64),
                ("device", ctypes.c_int32), ("pad", ctypes.c_int32)]


class pasta_stream_params(ctypes.Structure):
    _fields_ = [("page_shift", ctypes.c_uint32), ("slots", ctypes.c_uint32), ("max_batch", ctypes.c_uint64)]


class pasta_stream_batch(ctypes.Structure):
    _fields_ = [("addr", ctypes.c_void_p), ("n", ctypes.c_uint64), ("kernel_offsets", ctypes.c_void_p),
                ("n_kernels", ctypes.c_uint32), ("kernel_row0", ctypes.c_uint32)]


class pasta_rich_records(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("grid_lo", ctypes.c_uint32), ("grid_hi", ctypes.c_uint32)]


class pasta_rich_outputs(ctypes.Structure):
    _fields_ = [("rich_totals", ctypes.c_void_p), ("page_write_counts", ctypes.c_void_p),
                ("alloc_write_counts", ctypes.c_void_p), ("alloc_bytes", ctypes.c_void_p)]


_vp, _u64, _u32, _int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
_SIGS = {
    "pasta_trace_open": (_int, [ctypes.POINTER(pasta_open_params), ctypes.POINTER(_vp)]),
    "pasta_register_alloc": (_int, [_vp, _u64, _u64, ctypes.POINTER(_u32)]),
    "pasta_register_free": (_int, [_vp, _u64]),
    "pasta_register_tensor": (_int, [_vp, _u64, _u64, ctypes.POINTER(_u32)]),
    "pasta_register_tensor_free": (_int, [_vp, _u64]),
    "pasta_report_memory_usage": (_int, [_vp, _u64, ctypes.c_int64, ctypes.POINTER(_u32)]),
    "pasta_prefetch_plan": (_int, [_vp, _vp, _u32, _u32, _vp, _vp, _u64, ctypes.POINTER(_u64)]),
    "pasta_analyze": (_int, [_vp, ctypes.POINTER(pasta_records), _u64, _u32, ctypes.POINTER(pasta_histograms)]),
    "pasta_analyze_batches": (_int, [_vp, ctypes.POINTER(pasta_batch), _u32, _u32]),
    "pasta_finalize": (_int, [_vp, _u32, _u32, ctypes.POINTER(pasta_histograms)]),
    "pasta_analyze_rich": (_int, [_vp, ctypes.POINTER(pasta_rich_records), _u64, _u32,
                                  ctypes.POINTER(pasta_histograms), ctypes.POINTER(pasta_rich_outputs)]),
    "pasta_topk": (_int, [_vp, _vp, _u64, _u32, _vp, _vp, _vp]),
    "pasta_topk_many": (_int, [_vp, _vp, _u64, _u32, ctypes.POINTER(_u32), ctypes.POINTER(_vp),
                               ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "pasta_topk_prefix": (_int, [_vp, _vp, _vp, _vp, _u32, _u32, ctypes.POINTER(_u32), ctypes.POINTER(_vp),
                                 ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "pasta_bitmap_or": (_int, [_vp, _vp, _u32, _u64, _vp, _vp]),
    "pasta_topk_merge": (_int, [_vp, _vp, _vp, _u32, _u32, _u64, _vp, _vp, _vp]),
    "pasta_peer_reduce": (_int, [_vp, ctypes.POINTER(_vp), _u32, _u64, _u64, _u32, _vp, _vp, _vp]),
    "pasta_enable_peer": (_int, [_vp, _int]),
    "pasta_peer_reduce_small": (_int, [_vp, ctypes.POINTER(_vp), _u32, _u64, _u64, ctypes.POINTER(pasta_peer_slot),
                                       _u32, _vp]),
    "pasta_peer_gather": (_int, [_vp, ctypes.POINTER(pasta_peer_copy), _u32]),
    "pasta_stream_open": (_int, [_vp, ctypes.POINTER(pasta_stream_params), ctypes.POINTER(pasta_histograms),
                                 ctypes.POINTER(_vp)]),
    "pasta_stream_push": (_int, [_vp, ctypes.POINTER(pasta_stream_batch), _u32]),
    "pasta_stream_consumed": (_int, [_vp, ctypes.POINTER(_u64)]),
    "pasta_stream_close": (_int, [_vp]),
    "pasta_stream_destroy": (_int, [_vp]),
    "pasta_ipc_export": (_int, [_vp, _vp, ctypes.POINTER(pasta_ipc_handle)]),
    "pasta_ipc_open": (_int, [_vp, ctypes.POINTER(pasta_ipc_handle), ctypes.POINTER(_vp)]),
    "pasta_ipc_close": (_int, [_vp, _vp]),
    "pasta_sync": (_int, [_vp]),
    "pasta_close": (_int, [_vp]),
    "pasta_strerror": (ctypes.c_char_p, [_int]),
    "pasta_set_timing": (_int, [_vp, _int]),
    "pasta_get_timing": (_int, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64)]),
    "pasta_reset_timing": (_int, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class PastaError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        super().__init__(f"{what}: {pasta_strerror(status)} ({status})")


def _check(status, what):
    if status != PASTA_OK:
        raise PastaError(status, what)
    return status


def _ptr(t):
    """Device (or host) address of a tensor / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


# ----------------------------- C-name functions -----------------------------
def pasta_strerror(status: int) -> str:
    return _lib.pasta_strerror(status).decode()


def pasta_trace_open(device: int, va_lo: int, va_hi: int, max_live: int, max_ids: int, stream=0,
                     host_chunk_bytes: int = 0, flags: int = 0, max_live_tensors: int = 0, max_tensor_ids: int = 0):
    p = pasta_open_params(device, max_live, max_ids, flags, va_lo, va_hi, ctypes.c_void_p(stream or 0),
                          host_chunk_bytes, max_live_tensors, max_tensor_ids)
    h = ctypes.c_void_p()
    _check(_lib.pasta_trace_open(ctypes.byref(p), ctypes.byref(h)), "pasta_trace_open")
    return h


def pasta_register_alloc(h, base: int, size: int) -> int:
    out = _u32()
    _check(_lib.pasta_register_alloc(h, base, size, ctypes.byref(out)), "pasta_register_alloc")
    return out.value


def pasta_register_free(h, base: int):
    _check(_lib.pasta_register_free(h, base), "pasta_register_free")


def pasta_register_tensor(h, base: int, size: int) -> int:
    out = _u32()
    _check(_lib.pasta_register_tensor(h, base, size, ctypes.byref(out)), "pasta_register_tensor")
    return out.value


def pasta_register_tensor_free(h, base: int):
    _check(_lib.pasta_register_tensor_free(h, base), "pasta_register_tensor_free")


def pasta_report_memory_usage(h, ptr: int, delta: int) -> int:
    out = _u32(0)
    _check(_lib.pasta_report_memory_usage(h, ptr, delta, ctypes.byref(out)), "pasta_report_memory_usage")
    return out.value


def pasta_prefetch_plan(h, rows, n_kernels: int, level: int, plan_offsets, plan_ranges, cap: int) -> tuple:
    """Returns (status, total): ECAPACITY is returned, not raised, so callers can size."""
    total = _u64()
    st = _lib.pasta_prefetch_plan(h, _ptr(rows), n_kernels, level, _ptr(plan_offsets), _ptr(plan_ranges), cap,
                                  ctypes.byref(total))
    if st not in (PASTA_OK, PASTA_ECAPACITY):
        raise PastaError(st, "pasta_prefetch_plan")
    return st, total.value


def pasta_analyze(h, addr, n: int, page_shift: int, hist, kernel_offsets=None, n_kernels: int = 0, flags: int = 0):
    rec = pasta_records(_ptr(addr), _ptr(kernel_offsets), n_kernels, flags)
    _check(_lib.pasta_analyze(h, ctypes.byref(rec), n, page_shift, ctypes.byref(hist)), "pasta_analyze")


def pasta_analyze_batches(h, batches, page_shift: int):
    """batches: a ctypes array of pasta_batch (kept alive by the caller)."""
    _check(_lib.pasta_analyze_batches(h, batches, len(batches), page_shift), "pasta_analyze_batches")


def pasta_analyze_rich(h, records, n: int, grid_lo: int, grid_hi: int, page_shift: int, hist, rich):
    tr = pasta_rich_records(_ptr(records), grid_lo, grid_hi)
    _check(_lib.pasta_analyze_rich(h, ctypes.byref(tr), n, page_shift, ctypes.byref(hist), ctypes.byref(rich)),
           "pasta_analyze_rich")


def pasta_finalize(h, page_shift: int, n_kernels: int, hist):
    _check(_lib.pasta_finalize(h, page_shift, n_kernels, ctypes.byref(hist)), "pasta_finalize")


def pasta_topk(h, page_counts, P: int, k: int, out_page, out_count, out_found):
    _check(_lib.pasta_topk(h, _ptr(page_counts), P, k, _ptr(out_page), _ptr(out_count), _ptr(out_found)),
           "pasta_topk")


def _topk_arrays(ks, outs):
    n = len(ks)
    return ((_u32 * n)(*ks), (_vp * n)(*[_ptr(o[0]) for o in outs]), (_vp * n)(*[_ptr(o[1]) for o in outs]),
            (_vp * n)(*[_ptr(o[2]) for o in outs]))


def pasta_topk_many(h, page_counts, P: int, ks, outs):
    """outs[j] = (out_page, out_count, out_found) for ks[j]."""
    a_k, a_p, a_c, a_f = _topk_arrays(ks, outs)
    _check(_lib.pasta_topk_many(h, _ptr(page_counts), P, len(ks), a_k, a_p, a_c, a_f), "pasta_topk_many")


def pasta_topk_prefix(h, src, k_src: int, ks, outs):
    """src = (page, count, found) of a top-k_src list; outs[j] = (page, count, found) for ks[j]."""
    a_k, a_p, a_c, a_f = _topk_arrays(ks, outs)
    _check(_lib.pasta_topk_prefix(h, _ptr(src[0]), _ptr(src[1]), _ptr(src[2]), k_src, len(ks), a_k, a_p, a_c, a_f),
           "pasta_topk_prefix")


def pasta_bitmap_or(h, gathered, g: int, words: int, out_bitmap, out_popcount=None):
    _check(_lib.pasta_bitmap_or(h, _ptr(gathered), g, words, _ptr(out_bitmap), _ptr(out_popcount)),
           "pasta_bitmap_or")


def pasta_topk_merge(h, cand_page, cand_count, g: int, k: int, shard_pages: int, out_page, out_count, out_found):
    _check(_lib.pasta_topk_merge(h, _ptr(cand_page), _ptr(cand_count), g, k, shard_pages, _ptr(out_page),
                                 _ptr(out_count), _ptr(out_found)), "pasta_topk_merge")


PASTA_PEER_SUM, PASTA_PEER_MAX, PASTA_PEER_ARGMAX = 0, 1, 2


def pasta_peer_reduce(h, srcs, lo: int, n: int, out, out_bitmap=None, out_popcount=None, op: int = PASTA_PEER_SUM):
    """srcs: device addresses (ints) or tensors readable from h's device (local or CUDA-IPC mapped)."""
    arr = (_vp * len(srcs))(*[_ptr(s) for s in srcs])
    _check(_lib.pasta_peer_reduce(h, arr, len(srcs), lo, n, op, _ptr(out), _ptr(out_bitmap), _ptr(out_popcount)),
           "pasta_peer_reduce")


def pasta_enable_peer(h, peer_device: int):
    _check(_lib.pasta_enable_peer(h, peer_device), "pasta_enable_peer")


PASTA_PEER_ZERO = 3
PASTA_COPY, PASTA_COPY_ADD = 0, 1


def pasta_peer_reduce_small(h, srcs, lo: int, n: int, slots, out):
    """slots: [(index, op)] with op PASTA_PEER_MAX / PASTA_PEER_ARGMAX / PASTA_PEER_ZERO."""
    arr = (_vp * len(srcs))(*[_ptr(s) for s in srcs])
    sl = (pasta_peer_slot * max(1, len(slots)))(*[pasta_peer_slot(i, op) for i, op in slots])
    _check(_lib.pasta_peer_reduce_small(h, arr, len(srcs), lo, n, sl, len(slots), _ptr(out)),
           "pasta_peer_reduce_small")


def pasta_peer_gather(h, copies):
    """copies: [(src, dst, n_words, op)] (device addresses or tensors), one launch."""
    tab = (pasta_peer_copy * len(copies))(*[pasta_peer_copy(_ptr(a), _ptr(b), n, op, 0) for a, b, n, op in copies])
    _check(_lib.pasta_peer_gather(h, tab, len(copies)), "pasta_peer_gather")


def pasta_stream_open(h, page_shift: int, slots: int, max_batch: int, hist):
    out = _vp()
    prm = pasta_stream_params(page_shift, slots, max_batch)
    _check(_lib.pasta_stream_open(h, ctypes.byref(prm), ctypes.byref(hist), ctypes.byref(out)), "pasta_stream_open")
    return out


def pasta_stream_push(s, batches, count: int | None = None):
    """batches: a ctypes array of pasta_stream_batch (or a list of them)."""
    if not isinstance(batches, ctypes.Array):
        batches = (pasta_stream_batch * len(batches))(*batches)
    _check(_lib.pasta_stream_push(s, batches, len(batches) if count is None else count), "pasta_stream_push")


def pasta_stream_consumed(s) -> int:
    out = _u64()
    _check(_lib.pasta_stream_consumed(s, ctypes.byref(out)), "pasta_stream_consumed")
    return int(out.value)


def pasta_stream_close(s):
    _check(_lib.pasta_stream_close(s), "pasta_stream_close")


def pasta_stream_destroy(s):
    _check(_lib.pasta_stream_destroy(s), "pasta_stream_destroy")


def pasta_ipc_export(h, ptr) -> bytes:
    """The IPC handle of the device block holding ptr, as plain bytes (for any channel)."""
    out = pasta_ipc_handle()
    _check(_lib.pasta_ipc_export(h, _ptr(ptr), ctypes.byref(out)), "pasta_ipc_export")
    return bytes(out)


def pasta_ipc_open(h, handle: bytes) -> int:
    """Map another process's exported block in h's device context; returns the address."""
    hd = pasta_ipc_handle.from_buffer_copy(handle)
    out = _vp()
    _check(_lib.pasta_ipc_open(h, ctypes.byref(hd), ctypes.byref(out)), "pasta_ipc_open")
    return int(out.value)


def pasta_ipc_close(h, ptr: int):
    _check(_lib.pasta_ipc_close(h, ptr), "pasta_ipc_close")


def pasta_sync(h):
    _check(_lib.pasta_sync(h), "pasta_sync")


def pasta_close(h):
    _check(_lib.pasta_close(h), "pasta_close")


def pasta_set_timing(h, enable: bool):
    _check(_lib.pasta_set_timing(h, 1 if enable else 0), "pasta_set_timing")


def pasta_get_timing(h):
    ms = (ctypes.c_double * PHASES)()
    n = _u64()
    _check(_lib.pasta_get_timing(h, ms, ctypes.byref(n)), "pasta_get_timing")
    return dict(zip(PHASE_NAMES, list(ms))), n.value


def pasta_reset_timing(h):
    _check(_lib.pasta_reset_timing(h), "pasta_reset_timing")


# ----------------------------- convenience layer -----------------------------
class Histograms:
    """Output arrays as int64 CUDA tensors (u64 bit patterns).

    ``packed`` = [page_counts (P) | alloc_counts (max_ids) | totals (9) | tensor_counts
    (max_tensor_ids)] is one contiguous part, so the merge across ranks is one
    all_reduce(SUM); it and every other output are views of one
    zero-initialised arena (zero_() is one fill)."""

    def __init__(self, P: int, max_ids: int, device, n_kernels: int = 0, kernel_rows: bool = False,
                 kernel_pages: bool = False, bitmap: bool = True, pad_pages_to: int = 1, window_kernels: int = 0,
                 max_tensor_ids: int = 0, kernel_row0: int = 0):
        import torch

        self.P, self.max_ids, self.n_kernels, self.max_tensor_ids = P, max_ids, n_kernels, max_tensor_ids
        self.kernel_row0 = kernel_row0  # global index of kernel row 0 (a shard's first kernel)
        self.words = (P + 63) // 64
        # the page part is padded with zero pages to a multiple of `pad_pages_to` so it
        # can be reduce-scattered in equal shards (dist.ShardedMerger)
        self.P_pad = (P + pad_pages_to - 1) // pad_pages_to * pad_pages_to
        # every output lives in ONE zero-initialised arena (256-byte aligned parts), so a
        # step's reset is one fill launch instead of one per array
        sizes = {"packed": self.P_pad + max_ids + TOTALS + max_tensor_ids,
                 "page_bitmap": self.words if bitmap else 0,
                 "kernel_alloc_counts": n_kernels * max_ids if kernel_rows else 0,
                 "kernel_stats": n_kernels * KSTATS if kernel_rows else 0,
                 "kernel_tensor_counts": n_kernels * max_tensor_ids if (kernel_rows and max_tensor_ids) else 0,
                 "kernel_tensor_footprint": n_kernels if (kernel_rows and max_tensor_ids) else 0,
                 "kernel_page_bitmap": n_kernels * self.words if kernel_pages else 0}
        self.window_kernels = window_kernels
        self.n_windows = (n_kernels + window_kernels - 1) // window_kernels if window_kernels else 0
        sizes["hotness"] = self.n_windows * P
        offs, total = {}, 0
        for name, n in sizes.items():
            offs[name] = total
            total += (n + 31) // 32 * 32
        self.arena = torch.zeros(max(total, 1), dtype=torch.int64, device=device)

        def part(name, present=True):
            n = sizes[name]
            return self.arena[offs[name]:offs[name] + n] if present else None

        self.packed = part("packed")
        self.page_counts = self.packed[:P]
        self.pages_padded = self.packed[:self.P_pad]
        self.small = self.packed[self.P_pad:]  # [alloc_counts | totals | tensor_counts]
        self.alloc_counts = self.packed[self.P_pad:self.P_pad + max_ids]
        self.totals = self.packed[self.P_pad + max_ids:self.P_pad + max_ids + TOTALS]
        self.tensor_counts = self.packed[self.P_pad + max_ids + TOTALS:] if max_tensor_ids else None
        self.page_bitmap = part("page_bitmap", bitmap)
        self.kernel_alloc_counts = part("kernel_alloc_counts", kernel_rows)
        self.kernel_stats = part("kernel_stats", kernel_rows)
        self.kernel_tensor_counts = part("kernel_tensor_counts", kernel_rows and bool(max_tensor_ids))
        self.kernel_tensor_footprint = part("kernel_tensor_footprint", kernel_rows and bool(max_tensor_ids))
        self.kernel_page_bitmap = part("kernel_page_bitmap", kernel_pages)
        self.hotness = part("hotness", bool(window_kernels))

    def zero_(self):
        self.arena.zero_()
        return self

    def struct(self, flags: int = 0) -> pasta_histograms:
        return pasta_histograms(_ptr(self.page_counts), _ptr(self.alloc_counts), _ptr(self.totals),
                                _ptr(self.page_bitmap), _ptr(self.kernel_alloc_counts), _ptr(self.kernel_stats),
                                _ptr(self.kernel_page_bitmap), flags, self.window_kernels, _ptr(self.hotness),
                                _ptr(self.tensor_counts), _ptr(self.kernel_tensor_counts),
                                _ptr(self.kernel_tensor_footprint), self.kernel_row0)


class RichOutputs:
    """Extra outputs of the rich analysis (NEXT f4) as int64 CUDA tensors."""

    def __init__(self, P: int, max_ids: int, device, writes: bool = True, bytes_: bool = True):
        import torch

        self.rich_totals = torch.zeros(RICH_TOTALS, dtype=torch.int64, device=device)
        self.page_write_counts = torch.zeros(P, dtype=torch.int64, device=device) if writes else None
        self.alloc_write_counts = torch.zeros(max_ids, dtype=torch.int64, device=device) if writes else None
        self.alloc_bytes = torch.zeros(max_ids, dtype=torch.int64, device=device) if bytes_ else None

    def struct(self) -> pasta_rich_outputs:
        return pasta_rich_outputs(_ptr(self.rich_totals), _ptr(self.page_write_counts),
                                  _ptr(self.alloc_write_counts), _ptr(self.alloc_bytes))


class Trace:
    """A pasta_trace handle bound to one CUDA device and stream."""

    def __init__(self, device, va_lo: int, va_hi: int, max_live: int, max_ids: int, stream=None,
                 host_chunk_bytes: int = 0, schedule: str = "auto", max_live_tensors: int = 0,
                 max_tensor_ids: int = 0):
        import torch

        self.device = torch.device(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        self.va_lo, self.va_hi, self.max_live, self.max_ids = va_lo, va_hi, max_live, max_ids
        self.max_tensor_ids = max_tensor_ids
        self.h = pasta_trace_open(self.device.index or 0, va_lo, va_hi, max_live, max_ids, stream.cuda_stream,
                                  host_chunk_bytes, _SCHED[schedule], max_live_tensors, max_tensor_ids)

    def n_pages(self, page_shift: int) -> int:
        return (self.va_hi - self.va_lo) >> page_shift

    def register_alloc(self, base: int, size: int) -> int:
        return pasta_register_alloc(self.h, base, size)

    def register_free(self, base: int):
        pasta_register_free(self.h, base)

    def register_tensor(self, base: int, size: int) -> int:
        return pasta_register_tensor(self.h, base, size)

    def report_memory_usage(self, ptr: int, delta: int) -> int:
        """c10::reportMemoryUsage convention: delta > 0 allocates, < 0 releases."""
        return pasta_report_memory_usage(self.h, ptr, delta)

    def register_tensor_free(self, base: int):
        pasta_register_tensor_free(self.h, base)

    def prefetch_plan(self, hist: Histograms, level: str = "object"):
        """(offsets[n_kernels + 1], ranges[total, 2]) int64 device tensors: row k's staged
        ranges are ranges[offsets[k]:offsets[k+1]] as (start, end) (R20)."""
        import torch

        lv = LEVEL_TENSOR if level == "tensor" else LEVEL_OBJECT
        rows = hist.kernel_tensor_counts if lv == LEVEL_TENSOR else hist.kernel_alloc_counts
        nk = hist.n_kernels
        offsets = torch.empty(nk + 1, dtype=torch.int64, device=self.device)
        st, total = pasta_prefetch_plan(self.h, rows, nk, lv, offsets, None, 0)
        ranges = torch.empty((max(total, 1), 2), dtype=torch.int64, device=self.device)
        if total:
            st, total = pasta_prefetch_plan(self.h, rows, nk, lv, offsets, ranges, total)
            assert st == PASTA_OK
        return offsets, ranges[:total]

    def histograms(self, page_shift: int, n_kernels: int = 0, kernel_rows=False, kernel_pages=False, bitmap=True,
                   pad_pages_to: int = 1, window_kernels: int = 0, kernel_row0: int = 0):
        return Histograms(self.n_pages(page_shift), self.max_ids, self.device, n_kernels, kernel_rows, kernel_pages,
                          bitmap, pad_pages_to, window_kernels, self.max_tensor_ids, kernel_row0)

    def analyze(self, records, page_shift: int, hist: Histograms, kernel_offsets=None, n: int | None = None,
                finalize: bool = True, host: bool = False, stable: bool = False, chained: bool = False):
        if n is None:
            n = records.numel()
        nk = 0 if kernel_offsets is None else kernel_offsets.numel() - 1
        pasta_analyze(self.h, records, n, page_shift, hist.struct(0 if finalize else PASTA_NO_FINALIZE),
                      kernel_offsets, nk, (PASTA_REC_HOST if host else 0) | (PASTA_REC_STABLE if stable else 0)
                      | (PASTA_REC_CHAINED if chained else 0))

    def rich_outputs(self, page_shift: int, writes: bool = True, bytes_: bool = True) -> RichOutputs:
        return RichOutputs(self.n_pages(page_shift), self.max_ids, self.device, writes, bytes_)

    def analyze_rich(self, records, grid_lo: int, grid_hi: int, page_shift: int, hist: Histograms,
                     rich: RichOutputs, finalize: bool = True):
        """records: int64 CUDA tensor [n, 2] holding pasta_rich_record bytes (tracegen.rich)."""
        n = records.shape[0] if records.dim() == 2 else records.numel() // 2
        pasta_analyze_rich(self.h, records, n, grid_lo, grid_hi, page_shift,
                           hist.struct(0 if finalize else PASTA_NO_FINALIZE), rich.struct())

    def finalize(self, page_shift: int, hist: Histograms, n_kernels: int = 0):
        pasta_finalize(self.h, page_shift, n_kernels, hist.struct())

    def topk(self, page_counts, k: int, out=None):
        import torch

        if out is None:
            out = (torch.empty(k, dtype=torch.int64, device=self.device),
                   torch.empty(k, dtype=torch.int64, device=self.device),
                   torch.empty(1, dtype=torch.int64, device=self.device))
        pasta_topk(self.h, page_counts, page_counts.numel(), k, out[0], out[1], out[2])
        return out

    def topk_many(self, page_counts, ks, outs=None):
        """Every top-k list of ks with one selection (pasta_topk_many); returns {k: (page, count, found)}."""
        import torch

        ks = list(ks)
        if outs is None:
            outs = [(torch.empty(k, dtype=torch.int64, device=self.device),
                     torch.empty(k, dtype=torch.int64, device=self.device),
                     torch.empty(1, dtype=torch.int64, device=self.device)) for k in ks]
        pasta_topk_many(self.h, page_counts, page_counts.numel(), ks, outs)
        return dict(zip(ks, outs))

    def topk_prefix(self, src, k_src: int, ks, outs):
        pasta_topk_prefix(self.h, src, k_src, list(ks), outs)
        return dict(zip(ks, outs))

    def bitmap_or(self, gathered, g: int, words: int, out_bitmap, out_popcount=None):
        pasta_bitmap_or(self.h, gathered, g, words, out_bitmap, out_popcount)

    def topk_merge(self, cand_page, cand_count, g: int, k: int, shard_pages: int, out):
        pasta_topk_merge(self.h, cand_page, cand_count, g, k, shard_pages, out[0], out[1], out[2])
        return out

    def peer_reduce(self, srcs, lo: int, n: int, out, out_bitmap=None, out_popcount=None, op: int = 0):
        pasta_peer_reduce(self.h, srcs, lo, n, out, out_bitmap, out_popcount, op)

    def enable_peer(self, peer_device: int):
        pasta_enable_peer(self.h, peer_device)

    def peer_reduce_small(self, srcs, lo: int, n: int, slots, out):
        pasta_peer_reduce_small(self.h, srcs, lo, n, slots, out)

    def peer_gather(self, copies):
        pasta_peer_gather(self.h, copies)

    def ipc_export(self, t) -> bytes:
        return pasta_ipc_export(self.h, t)

    def ipc_open(self, handle: bytes) -> int:
        return pasta_ipc_open(self.h, handle)

    def ipc_close(self, ptr: int):
        pasta_ipc_close(self.h, ptr)

    def sync(self):
        pasta_sync(self.h)

    def set_timing(self, on: bool):
        pasta_set_timing(self.h, on)

    def timing(self):
        return pasta_get_timing(self.h)

    def reset_timing(self):
        pasta_reset_timing(self.h)

    def close(self):
        if self.h is not None:
            pasta_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
