"""Streaming / in-situ mode: a trace analyzed as a sequence
of fixed-size batches, the paper's operating point being a "4MB" device buffer (P:323,
P:971) = 524,288 records per call.

Every batch is one pasta_analyze call with PASTA_NO_FINALIZE over records [a, b). Its
kernel offsets are the global kernel offsets clipped to [a, b) and rebased, and its
per-kernel output pointers start at row k0 (the kernel holding record a), so kernels
cut between batches simply accumulate into the same global row (counts are sums over
any partition of the records). One pasta_finalize at the end derives
the bitmap, unique pages, footprints and WS. Host-side planning only; the calls can be
captured once into a CUDA graph and replayed (see bench.py --stream-batch).
"""
from __future__ import annotations

import numpy as np


def plan_batches(kernel_offsets, n: int, batch: int):
    """[(a, b, k0, sub_offsets)] covering [0, n) in batches of `batch` records.

    sub_offsets (int64, len = kernels overlapping [a, b) + 1) are the kernel offsets of
    the batch relative to a; k0 is the global index of its first kernel."""
    ko = np.asarray(kernel_offsets, dtype=np.int64)
    out = []
    for a in range(0, n, batch):
        b = min(n, a + batch)
        k0 = int(np.searchsorted(ko, a, side="right")) - 1
        k1 = int(np.searchsorted(ko, b, side="left"))  # first kernel starting at or after b
        inner = np.clip(ko[k0 + 1:k1] - a, 0, b - a)
        sub = np.concatenate([[0], inner, [b - a]]).astype(np.int64)
        out.append((a, b, k0, sub))
    return out


class BatchRunner:
    """Issues the batch calls of plan_batches on a Trace's stream (all device memory)."""

    def __init__(self, trace, hist, records, kernel_offsets, n: int, batch: int, page_shift: int,
                 stable: bool = True):
        """stable: the records are not written by the kernel that precedes each call on
        the stream (true for a resident trace), so every scan may start loading its
        batch while the previous one finishes (PASTA_REC_STABLE)."""
        import torch

        from . import (PASTA_NO_FINALIZE, PASTA_REC_CHAINED, PASTA_REC_STABLE, pasta_analyze_batches, pasta_batch,
                       pasta_histograms, pasta_records)

        if hist.hotness is not None or hist.tensor_counts is not None:
            # hotness rows are windows of kernels and tensor outputs are per-level rows that
            # the batch structs below do not carry: refuse instead of leaving them zero
            raise ValueError("BatchRunner: streaming supports page / alloc / kernel outputs only "
                             "(no hotness, no tensor level)")
        self.tr, self.hist, self.page_shift = trace, hist, page_shift
        self.batches = plan_batches(kernel_offsets, n, batch)
        dev = records.device
        flat = np.concatenate([s for _, _, _, s in self.batches])
        self.offs = torch.from_numpy(flat).to(dev)
        self.calls = []
        pos = 0
        W = hist.words
        for a, b, k0, sub in self.batches:
            hs = pasta_histograms(
                hist.page_counts.data_ptr(), hist.alloc_counts.data_ptr(), hist.totals.data_ptr(),
                hist.page_bitmap.data_ptr() if hist.page_bitmap is not None else None,
                hist.kernel_alloc_counts.data_ptr() + 8 * k0 * hist.max_ids
                if hist.kernel_alloc_counts is not None else None,
                hist.kernel_stats.data_ptr() + 8 * 4 * k0 if hist.kernel_stats is not None else None,
                hist.kernel_page_bitmap.data_ptr() + 8 * W * k0 if hist.kernel_page_bitmap is not None else None,
                PASTA_NO_FINALIZE, 0, None)
            self.calls.append((records.data_ptr() + 8 * a, b - a, self.offs.data_ptr() + 8 * pos, len(sub) - 1, hs))
            pos += len(sub)
        # after the first batch every call follows a scan of this handle into the same
        # outputs: chained (no wait before working, completion still in order)
        flags = PASTA_REC_STABLE if stable else 0
        chain_flags = (PASTA_REC_STABLE | PASTA_REC_CHAINED) if stable else 0
        self.array = (pasta_batch * len(self.calls))()
        for i, (addr, nrec, offs, nk, hs) in enumerate(self.calls):
            self.array[i] = pasta_batch(pasta_records(addr, offs, nk, chain_flags if i else flags), nrec, hs)
        self._submit = pasta_analyze_batches

    def run(self):
        """Enqueue every batch with one pasta_analyze_batches call (graph-capturable: no
        host synchronization). Nothing else may be enqueued on the trace's stream
        between the batches."""
        self._submit(self.tr.h, self.array, self.page_shift)


class StreamRing:
    """The same batches through ONE persistent consumer (pasta_stream_open / push /
    close, include/pasta.h): the host publishes the batch descriptors of a resident trace
    into a device ring of `slots` descriptors while the consumer runs; no launch per
    batch. Outputs as BatchRunner (no finalize: call Trace.finalize after)."""

    def __init__(self, trace, hist, records, kernel_offsets, n: int, batch: int, page_shift: int, slots: int = 64):
        import torch

        from . import pasta_stream_batch

        if batch % 2 or n % 2:
            raise ValueError("StreamRing: batches must hold an even number of records")
        self.tr, self.hist, self.page_shift, self.slots, self.batch = trace, hist, page_shift, slots, batch
        self.batches = plan_batches(kernel_offsets, n, batch)
        flat = np.concatenate([s for _, _, _, s in self.batches])
        self.offs = torch.from_numpy(flat).to(records.device)
        arr = (pasta_stream_batch * len(self.batches))()
        pos = 0
        for i, (a, b, k0, sub) in enumerate(self.batches):
            arr[i] = pasta_stream_batch(records.data_ptr() + 8 * a, b - a, self.offs.data_ptr() + 8 * pos,
                                        len(sub) - 1, k0)
            pos += len(sub)
        self.array = arr
        self.s = None

    def start(self):
        """Launch the consumer on the trace's stream (asynchronous)."""
        from . import pasta_stream_open

        self.s = pasta_stream_open(self.tr.h, self.page_shift, self.slots, self.batch, self.hist.struct())

    def push_all(self):
        """Publish every batch (the host waits whenever the ring is full), then the end."""
        from . import pasta_stream_close, pasta_stream_push

        pasta_stream_push(self.s, self.array)
        pasta_stream_close(self.s)

    def run(self):
        self.start()
        self.push_all()

    def destroy(self):
        """Wait for the consumer and free the ring."""
        from . import pasta_stream_destroy

        if self.s is not None:
            pasta_stream_destroy(self.s)
            self.s = None
