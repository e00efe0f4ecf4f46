"""oracle -- CPU oracle for the PASTA trace-analysis hot path (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl
reference`` leg may import this package. It shares no code with the CUDA path
(paper_2602_22103_b200/) and never imports it.

``OracleTrace`` mirrors the handle semantics of include/pasta.h with its own plain
Python registration bookkeeping (a dict of live ranges and a bisect-sorted list of
bases for the overlap check), and
delegates the per-record definition to oracle/oracle.cpp (std::map lookup, hash-map
counts, std::sort top-K). Everything is accumulated in
numpy uint64 arrays.

Status codes are the ones include/pasta.h documents (values restated, not imported).
"""
from __future__ import annotations

import bisect
import ctypes
import os

import numpy as np

OK, EINVAL, EOVERLAP, ENOENT, ECAPACITY = 0, -1, -2, -3, -4
U64MAX = (1 << 64) - 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


class _Range(ctypes.Structure):
    _fields_ = [("base", ctypes.c_uint64), ("size", ctypes.c_uint64), ("id", ctypes.c_uint32),
                ("pad", ctypes.c_uint32)]


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.oracle_analyze.restype = ctypes.c_int
        L.oracle_analyze.argtypes = [vp, u64, vp, u64, vp, u64, u64, u64, u32, u64, vp, vp, vp, vp, vp, vp, vp, u64]
        L.oracle_analyze_rich.restype = ctypes.c_int
        L.oracle_analyze_rich.argtypes = [vp, u64, vp, u64, u64, u64, u64, u64, u32, u64, vp, vp, vp, vp, vp, vp, vp,
                                          vp, vp]
        L.oracle_bitmap.restype = u64
        L.oracle_bitmap.argtypes = [vp, u64, vp]
        L.oracle_footprint.restype = u64
        L.oracle_footprint.argtypes = [vp, u64, u64, vp, vp]
        L.oracle_row_popcount.restype = None
        L.oracle_row_popcount.argtypes = [vp, u64, u64, vp]
        L.oracle_topk.restype = u64
        L.oracle_topk.argtypes = [vp, u64, u64, vp, vp]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleTrace:
    """Oracle counterpart of a pasta_trace handle (include/pasta.h)."""

    def __init__(self, va_lo: int, va_hi: int, max_live: int, max_ids: int, max_live_tensors: int = 0,
                 max_tensor_ids: int = 0):
        self.va_lo, self.va_hi = int(va_lo), int(va_hi)
        self.max_live, self.max_ids = int(max_live), int(max_ids)
        self.live = {}  # base -> (size, id)
        self.bases = []  # sorted live bases
        self.sizes = []  # id -> registered size (ids are never reused)
        self.id_base = []  # id -> registered base (kept after free, for prefetch plans)
        # tensor level (NEXT f3, R18-R20): tensors inside live objects
        self.max_live_tensors, self.max_tensor_ids = int(max_live_tensors), int(max_tensor_ids)
        self.tlive = {}  # base -> (size, tid)
        self.tbases = []
        self.tsizes = []
        self.tid_base = []
        self.tensor_counts = np.zeros(self.max_tensor_ids, dtype=np.uint64)
        self.untensored = 0
        self.tensor_rows = None
        self.kernel_rows = None
        self.kun = None
        self.kernel_pages = None
        self.hotness = None
        self.page_counts = None
        self.page_shift = None
        self.alloc_counts = np.zeros(self.max_ids, dtype=np.uint64)
        self.totals = np.zeros(3, dtype=np.uint64)  # records, unattributed, out_of_window

    # ---- registration: snapshot semantics, SPEC S:53 (no live overlap), S:210 ----
    def register_alloc(self, base: int, size: int):
        base, size = int(base), int(size)
        if size <= 0 or base < 0 or base + size > U64MAX:
            return EINVAL, None
        # intersecting live ranges: the nearest live base at or below base+size-1 is
        # the only candidate (live ranges never overlap); a sorted list of bases
        i = bisect.bisect_right(self.bases, base + size - 1) - 1
        if i >= 0:
            b = self.bases[i]
            s = self.live[b][0]
            if base < b + s and b < base + size:  # half-open intervals intersect
                return EOVERLAP, None
        if len(self.live) >= self.max_live or len(self.sizes) >= self.max_ids:
            return ECAPACITY, None
        i = len(self.sizes)
        self.sizes.append(size)
        self.id_base.append(base)
        self.live[base] = (size, i)
        bisect.insort(self.bases, base)
        return OK, i

    def register_free(self, base: int):
        base = int(base)
        if base not in self.live:
            return ENOENT
        size = self.live[base][0]
        del self.live[base]
        self.bases.pop(bisect.bisect_left(self.bases, base))
        # R19: the object's live tensors end with it
        for tb in [b for b in self.tbases if base <= b < base + size]:
            self.register_tensor_free(tb)
        return OK

    # ---- tensor level (R18): a tensor lies inside one live object, live tensors
    # never overlap, tensor ids are their own monotone never-reused space ----
    def register_tensor(self, base: int, size: int):
        base, size = int(base), int(size)
        if self.max_tensor_ids == 0 or size <= 0 or base < 0 or base + size > U64MAX:
            return EINVAL, None
        # containing object: the live object with the largest base <= base
        i = bisect.bisect_right(self.bases, base) - 1
        if i < 0:
            return EINVAL, None
        ob = self.bases[i]
        if not (base + size <= ob + self.live[ob][0]):
            return EINVAL, None
        i = bisect.bisect_right(self.tbases, base + size - 1) - 1
        if i >= 0:
            b = self.tbases[i]
            if base < b + self.tlive[b][0] and b < base + size:
                return EOVERLAP, None
        if len(self.tlive) >= self.max_live_tensors or len(self.tsizes) >= self.max_tensor_ids:
            return ECAPACITY, None
        t = len(self.tsizes)
        self.tsizes.append(size)
        self.tid_base.append(base)
        self.tlive[base] = (size, t)
        bisect.insort(self.tbases, base)
        return OK, t

    def register_tensor_free(self, base: int):
        base = int(base)
        if base not in self.tlive:
            return ENOENT
        del self.tlive[base]
        self.tbases.pop(bisect.bisect_left(self.tbases, base))
        return OK

    def report_memory_usage(self, ptr: int, delta: int):
        """Signed-size event (P:540 c10::reportMemoryUsage; negative size
        = release, normalized to a positive size) -> (status, id): to the tensor
        level if this handle has one, else to the object level. A release must name a
        live range starting at ptr (else ENOENT) of size -delta (else EINVAL)."""
        ptr, delta = int(ptr), int(delta)
        if delta == 0 or not -(1 << 63) < delta < (1 << 63):
            return EINVAL, None
        tensors = self.max_tensor_ids > 0
        if delta > 0:
            return self.register_tensor(ptr, delta) if tensors else self.register_alloc(ptr, delta)
        table = self.tlive if tensors else self.live
        if ptr not in table:
            return ENOENT, None
        size, ident = table[ptr]
        if size != -delta:
            return EINVAL, None
        st = self.register_tensor_free(ptr) if tensors else self.register_free(ptr)
        return st, ident

    # ---- one analyze call, accumulating ----
    def analyze(self, addr: np.ndarray, kernel_offsets=None, page_shift: int = 12, kernel_rows: bool = False,
                kernel_pages: bool = False, window_kernels: int = 0):
        addr = np.ascontiguousarray(addr, dtype=np.uint64)
        n = addr.size
        P = (self.va_hi - self.va_lo) >> page_shift
        W = (P + 63) // 64
        if self.page_counts is None or self.page_shift != page_shift:
            self.page_counts = np.zeros(P, dtype=np.uint64)
            self.page_shift = page_shift
        if kernel_offsets is None:
            ko = np.array([0, n], dtype=np.uint64)
        else:
            ko = np.ascontiguousarray(kernel_offsets, dtype=np.uint64)
        nk = ko.size - 1
        kac = kun = kp = None
        if kernel_rows:
            if self.kernel_rows is None or self.kernel_rows.shape != (nk, self.max_ids):
                self.kernel_rows = np.zeros((nk, self.max_ids), dtype=np.uint64)
                self.kun = np.zeros(nk, dtype=np.uint64)
            kac, kun = self.kernel_rows, self.kun
        if kernel_pages:
            if self.kernel_pages is None or self.kernel_pages.shape != (nk, W):
                self.kernel_pages = np.zeros((nk, W), dtype=np.uint64)
            kp = self.kernel_pages
        hot = None
        if window_kernels:
            nw = (nk + window_kernels - 1) // window_kernels
            if self.hotness is None or self.hotness.shape != (nw, P):
                self.hotness = np.zeros((nw, P), dtype=np.uint64)
            hot = self.hotness
        live = (_Range * max(1, len(self.live)))()
        for i, (b, (s, idx)) in enumerate(sorted(self.live.items())):
            live[i].base, live[i].size, live[i].id = b, s, idx
        rc = lib().oracle_analyze(ctypes.addressof(live), len(self.live), _ptr(addr), n, _ptr(ko), nk,
                                  self.va_lo, self.va_hi, page_shift, self.max_ids, _ptr(self.page_counts),
                                  _ptr(self.alloc_counts), _ptr(self.totals), _ptr(kac), _ptr(kun), _ptr(kp),
                                  _ptr(hot), window_kernels)
        if rc != 0:
            raise ValueError(f"oracle_analyze rejected its input ({rc})")
        if self.max_tensor_ids:
            self._analyze_tensors(addr, ko, nk, page_shift, kernel_rows)

    def _analyze_tensors(self, addr, ko, nk, page_shift, kernel_rows):
        """Tensor level (R18): the same definition over the live tensor set:
        each record counts for the live tensor holding its address, else as untensored.
        The page outputs of this second pass are discarded."""
        P = (self.va_hi - self.va_lo) >> page_shift
        scratch_pages = np.zeros(P, dtype=np.uint64)
        tot = np.zeros(3, dtype=np.uint64)
        ktc = kun = None
        if kernel_rows:
            if self.tensor_rows is None or self.tensor_rows.shape != (nk, self.max_tensor_ids):
                self.tensor_rows = np.zeros((nk, self.max_tensor_ids), dtype=np.uint64)
            ktc = self.tensor_rows
            kun = np.zeros(nk, dtype=np.uint64)
        live = (_Range * max(1, len(self.tlive)))()
        for i, (b, (s, t)) in enumerate(sorted(self.tlive.items())):
            live[i].base, live[i].size, live[i].id = b, s, t
        rc = lib().oracle_analyze(ctypes.addressof(live), len(self.tlive), _ptr(addr), addr.size, _ptr(ko), nk,
                                  self.va_lo, self.va_hi, page_shift, self.max_tensor_ids, _ptr(scratch_pages),
                                  _ptr(self.tensor_counts), _ptr(tot), _ptr(ktc), _ptr(kun), None, None, 0)
        if rc != 0:
            raise ValueError(f"oracle_analyze (tensors) rejected its input ({rc})")
        self.untensored += int(tot[1])

    def analyze_parallel(self, records, kernel_offsets, page_shift: int = 12, kernel_rows: bool = False,
                         kernel_pages: bool = False, threads: int | None = None, slab: int = 1 << 24):
        """The same definition as ``analyze`` over a whole trace, run chunk-parallel on
        the host's cores (the full-size parity tests and the all-core cpu_baseline).

        The trace is cut at kernel boundaries into slabs of about ``slab`` records; each
        worker thread runs the unchanged single-thread oracle_analyze on one slab after
        another into its OWN page / alloc / totals arrays (kernel rows, per-kernel
        unattributed and per-kernel page rows are disjoint between kernel-aligned slabs,
        so they are written in place), and the per-thread arrays are summed at the end.
        That fold is SPEC S:291-299 (every count is a pointwise sum over any partition
        of the records), pinned in tests/test_oracle_pins.py against the serial call.

        records: a numpy uint64 array [n], or a callable (j0, j1) -> numpy records of
        [j0, j1) (e.g. tracegen.host_records, so a 10^10-record trace never has to be
        held in host memory at once). ctypes releases the GIL around every C call, so
        the threads run concurrently. No hotness, no tensor level (use ``analyze``)."""
        import threading

        assert not self.max_tensor_ids, "analyze_parallel: one level only"
        ko = np.ascontiguousarray(kernel_offsets, dtype=np.uint64)
        nk = ko.size - 1
        n = int(ko[-1])
        if callable(records):
            get = records
        else:
            arr = np.ascontiguousarray(records, dtype=np.uint64)
            assert arr.size == n
            get = lambda j0, j1: arr[j0:j1]  # noqa: E731
        P = (self.va_hi - self.va_lo) >> page_shift
        W = (P + 63) // 64
        if self.page_counts is None or self.page_shift != page_shift:
            self.page_counts = np.zeros(P, dtype=np.uint64)
            self.page_shift = page_shift
        kac = kun = kp = None
        if kernel_rows:
            if self.kernel_rows is None or self.kernel_rows.shape != (nk, self.max_ids):
                self.kernel_rows = np.zeros((nk, self.max_ids), dtype=np.uint64)
                self.kun = np.zeros(nk, dtype=np.uint64)
            kac, kun = self.kernel_rows, self.kun
        if kernel_pages:
            if self.kernel_pages is None or self.kernel_pages.shape != (nk, W):
                self.kernel_pages = np.zeros((nk, W), dtype=np.uint64)
            kp = self.kernel_pages
        # kernel-aligned slabs [k_a, k_b) of about `slab` records (a kernel is never cut)
        slabs, k = [], 0
        while k < nk:
            kb = int(np.searchsorted(ko, int(ko[k]) + slab, side="right")) - 1
            kb = min(nk, max(kb, k + 1))
            slabs.append((k, kb))
            k = kb
        live = (_Range * max(1, len(self.live)))()
        for i, (b, (s, idx)) in enumerate(sorted(self.live.items())):
            live[i].base, live[i].size, live[i].id = b, s, idx
        n_live = len(self.live)
        T = max(1, min(threads or os.cpu_count() or 1, len(slabs)))
        acc = [(np.zeros(P, dtype=np.uint64), np.zeros(self.max_ids, dtype=np.uint64), np.zeros(3, dtype=np.uint64))
               for _ in range(T)]
        nxt = [0]
        lock = threading.Lock()
        errors = []

        def row(a, k0, width):
            return None if a is None else a.ctypes.data + 8 * k0 * width

        def worker(t):
            pages, allocs, tot = acc[t]
            while not errors:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(slabs):
                    return
                ka, kb = slabs[i]
                j0, j1 = int(ko[ka]), int(ko[kb])
                rec = np.ascontiguousarray(get(j0, j1), dtype=np.uint64)
                offs = np.ascontiguousarray(ko[ka:kb + 1] - np.uint64(j0))
                rc = lib().oracle_analyze(ctypes.addressof(live), n_live, _ptr(rec), j1 - j0, _ptr(offs), kb - ka,
                                          self.va_lo, self.va_hi, page_shift, self.max_ids, _ptr(pages),
                                          _ptr(allocs), _ptr(tot), row(kac, ka, self.max_ids), row(kun, ka, 1),
                                          row(kp, ka, W), None, 0)
                if rc != 0:
                    errors.append(f"oracle_analyze rejected slab {ka}..{kb} ({rc})")

        ths = [threading.Thread(target=worker, args=(t,)) for t in range(T)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        if errors:
            raise ValueError(errors[0])
        with np.errstate(over="ignore"):
            for pages, allocs, tot in acc:  # the partition fold
                self.page_counts += pages
                self.alloc_counts += allocs
                self.totals += tot
        return T

    # ---- rich 16-byte records (NEXT f4, R21-R23) ----
    def analyze_rich(self, rec16: np.ndarray, grid_lo: int, grid_hi: int, page_shift: int = 12,
                     kernel_rows: bool = False):
        """rec16: uint8 [n, 16] (or any buffer of n * 16 bytes) in the layout of
        oracle_analyze_rich. Accumulates page / alloc counts and totals like analyze, plus
        page_writes, alloc_writes, alloc_bytes, rich_totals [filtered, shared, writes,
        bytes]; kernel rows are indexed by grid_id - grid_lo."""
        rec = np.ascontiguousarray(rec16).view(np.uint8).reshape(-1)
        n = rec.size // 16
        P = (self.va_hi - self.va_lo) >> page_shift
        if self.page_counts is None or self.page_shift != page_shift:
            self.page_counts = np.zeros(P, dtype=np.uint64)
            self.page_shift = page_shift
        if getattr(self, "page_writes", None) is None or self.page_writes.size != P:
            self.page_writes = np.zeros(P, dtype=np.uint64)
            self.alloc_writes = np.zeros(self.max_ids, dtype=np.uint64)
            self.alloc_bytes = np.zeros(self.max_ids, dtype=np.uint64)
            self.rich_totals = np.zeros(4, dtype=np.uint64)
        nk = int(grid_hi) - int(grid_lo) + 1
        kac = kun = None
        if kernel_rows:
            if self.kernel_rows is None or self.kernel_rows.shape != (nk, self.max_ids):
                self.kernel_rows = np.zeros((nk, self.max_ids), dtype=np.uint64)
                self.kun = np.zeros(nk, dtype=np.uint64)
            kac, kun = self.kernel_rows, self.kun
        live = (_Range * max(1, len(self.live)))()
        for i, (b, (s, idx)) in enumerate(sorted(self.live.items())):
            live[i].base, live[i].size, live[i].id = b, s, idx
        rc = lib().oracle_analyze_rich(ctypes.addressof(live), len(self.live), _ptr(rec), n, int(grid_lo),
                                       int(grid_hi), self.va_lo, self.va_hi, page_shift, self.max_ids,
                                       _ptr(self.page_counts), _ptr(self.page_writes), _ptr(self.alloc_counts),
                                       _ptr(self.alloc_writes), _ptr(self.alloc_bytes), _ptr(self.totals),
                                       _ptr(self.rich_totals), _ptr(kac), _ptr(kun))
        if rc != 0:
            raise ValueError(f"oracle_analyze_rich rejected its input ({rc})")

    def max_kernel(self):
        """MAX_MEM_REFERENCED_KERNEL: the kernel with the most analyzed records
        (attributed + unattributed), ties to the lowest index (R24); None without rows."""
        if self.kernel_rows is None or self.kernel_rows.shape[0] == 0:
            return None
        per = self.kernel_rows.sum(axis=1, dtype=np.uint64) + self.kun
        return int(np.argmax(per))

    # ---- derived results ----
    def bitmap(self):
        P = self.page_counts.size
        bm = np.zeros((P + 63) // 64, dtype=np.uint64)
        u = lib().oracle_bitmap(_ptr(self.page_counts), P, _ptr(bm))
        return bm, int(u)

    def footprints(self):
        sizes = np.zeros(self.max_ids, dtype=np.uint64)
        sizes[: len(self.sizes)] = self.sizes
        nk = self.kernel_rows.shape[0]
        fp = np.zeros(nk, dtype=np.uint64)
        ws = lib().oracle_footprint(_ptr(self.kernel_rows), nk, self.max_ids, _ptr(sizes), _ptr(fp))
        return fp, int(ws)

    def tensor_footprints(self):
        """footprint_t[k] = sum of tensor sizes with a count in kernel k; WS_tensor = max."""
        sizes = np.zeros(self.max_tensor_ids, dtype=np.uint64)
        sizes[: len(self.tsizes)] = self.tsizes
        nk = self.tensor_rows.shape[0]
        fp = np.zeros(nk, dtype=np.uint64)
        ws = lib().oracle_footprint(_ptr(self.tensor_rows), nk, self.max_tensor_ids, _ptr(sizes), _ptr(fp))
        return fp, int(ws)

    def prefetch_plan(self, level: str):
        """R20 (S:488-514 build_prefetch_plan): per kernel, the union of [base, base+size)
        of every object (level "object") or tensor ("tensor") with >= 1 access in that
        kernel, as sorted disjoint (start, end) intervals, touching ones merged."""
        if level == "object":
            rows, base, size = self.kernel_rows, self.id_base, self.sizes
        else:
            rows, base, size = self.tensor_rows, self.tid_base, self.tsizes
        return [interval_union([(base[i], base[i] + size[i]) for i in np.nonzero(row)[0]]) for row in rows]

    def kernel_unique_pages(self):
        nk, W = self.kernel_pages.shape
        out = np.zeros(nk, dtype=np.uint64)
        lib().oracle_row_popcount(_ptr(self.kernel_pages), nk, W, _ptr(out))
        return out

    def topk(self, K: int):
        return topk(self.page_counts, K)


def interval_union(iv):
    """Sorted disjoint union of half-open intervals; touching intervals are merged."""
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


def topk(page_counts: np.ndarray, K: int):
    """(pages[K], counts[K], found) ordered by (count desc, page asc) (R10)."""
    pc = np.ascontiguousarray(page_counts, dtype=np.uint64)
    pages = np.empty(K, dtype=np.uint64)
    counts = np.empty(K, dtype=np.uint64)
    found = lib().oracle_topk(_ptr(pc), pc.size, K, _ptr(pages), _ptr(counts))
    return pages, counts, int(found)


def bitmap(page_counts: np.ndarray):
    pc = np.ascontiguousarray(page_counts, dtype=np.uint64)
    bm = np.zeros((pc.size + 63) // 64, dtype=np.uint64)
    u = lib().oracle_bitmap(_ptr(pc), pc.size, _ptr(bm))
    return bm, int(u)
