"""Multi-GPU merge of per-shard results -- collectives only.

Trace shards are kernel-aligned contiguous record ranges, one per rank; every rank
registers the identical allocation list. Every count output is a pointwise sum over
any partition of the records, so:

* page / alloc counts and the additive totals merge with ONE all_reduce(SUM) of the
  packed int64 buffer [page_counts | alloc_counts | totals] (two's-complement int64
  sums are bit-identical to u64 modular sums);
* the page bitmap merges by OR: NCCL has no bitwise-OR reduction (torch refuses
  ReduceOp.BOR on NCCL), so ranks all_gather their bitmaps and the pasta_bitmap_or
  kernel ORs them and recounts unique pages;
* WS_obj (a max over kernels) merges with all_reduce(MAX);
* MAX_MEM_REFERENCED_KERNEL (totals slots 7-8, an (index, records) pair per rank with
  the index global through Histograms.kernel_row0) merges by ARGMAX: the pairs are
  gathered and pasta_peer_reduce(PASTA_PEER_ARGMAX) keeps the one with the most records,
  ties to the lowest kernel (R24). Exact for kernel-aligned shards, whose kernel
  rows are disjoint; for arbitrary cuts merge_kernel_rows + pasta_finalize on the merged
  rows recompute it;
* per-kernel rows are disjoint across ranks for kernel-aligned shards; for arbitrary
  cuts merge_kernel_rows sums the straddling rows.
Compute stays in the CUDA kernels; these helpers only move data.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


# totals slots merged by MAX (working sets, R11; tensor level R18), the (index, records)
# pair of MAX_MEM_REFERENCED_KERNEL merged by ARGMAX (R24); the rest are sums
_WS_SLOTS = (4, 6)  # PASTA_T_WS_OBJ, PASTA_T_WS_TENSOR
_MK = 7  # PASTA_T_MAX_KERNEL, PASTA_T_MAX_KERNEL + 1 = PASTA_T_MAX_KERNEL_RECORDS


def merge_counts(packed: torch.Tensor, group=None):
    """all_reduce(SUM) of the packed count buffer, in place."""
    dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    return packed


def gather_bitmaps(bitmap: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """[world * words] concatenation of every rank's bitmap (rank-major)."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty(world * bitmap.numel(), dtype=bitmap.dtype, device=bitmap.device)
    dist.all_gather_into_tensor(out, bitmap, group=group)
    return out


def merge_max(x: torch.Tensor, group=None):
    dist.all_reduce(x, op=dist.ReduceOp.MAX, group=group)
    return x


def gather_pairs(pair: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """[world * 2] rank-major concatenation of every rank's (index, records) pair."""
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty(world * 2, dtype=pair.dtype, device=pair.device)
    dist.all_gather_into_tensor(out, pair.contiguous(), group=group)
    return out


def merge_max_kernel(trace, totals: torch.Tensor, saved_pair: torch.Tensor, gathered: torch.Tensor, group=None):
    """totals[7:9] = the ARGMAX over ranks of the saved (index, records) pairs (one
    pasta_peer_reduce over the gathered rows, local memory)."""
    from . import PASTA_PEER_ARGMAX

    world = dist.get_world_size(group)
    gather_pairs(saved_pair, group, out=gathered)
    trace.peer_reduce([gathered.data_ptr() + 16 * r for r in range(world)], 0, 2,
                      totals.data_ptr() + 8 * _MK, op=PASTA_PEER_ARGMAX)


def merge_kernel_rows(rows_local: torch.Tensor, k0: int, n_kernels_total: int, group=None) -> torch.Tensor:
    """Global [n_kernels_total, C] rows from each rank's local rows [k1-k0, C] starting at
    kernel k0 (rows of a kernel cut between ranks are summed)."""
    C = rows_local.shape[1]
    full = torch.zeros(n_kernels_total, C, dtype=rows_local.dtype, device=rows_local.device)
    full[k0:k0 + rows_local.shape[0]] += rows_local
    dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


def reduce_scatter_counts(pages_padded: torch.Tensor, out: torch.Tensor, group=None) -> torch.Tensor:
    """SUM of every rank's padded page counts; rank r receives shard r (pages
    [r*S, (r+1)*S), S = len(pages_padded) / world)."""
    dist.reduce_scatter_tensor(out, pages_padded, op=dist.ReduceOp.SUM, group=group)
    return out


def gather_candidates(pages: torch.Tensor, counts: torch.Tensor, out_pages: torch.Tensor, out_counts: torch.Tensor,
                      group=None):
    """[world * k] rank-major concatenation of every rank's local top-k candidates."""
    dist.all_gather_into_tensor(out_pages, pages, group=group)
    dist.all_gather_into_tensor(out_counts, counts, group=group)
    return out_pages, out_counts


class Merger:
    """One merge step for a Trace's Histograms after a local analyze (with finalize):
    SUM of counts, OR of bitmaps (+ unique pages), MAX of WS_obj."""

    def __init__(self, trace, hist, group=None):
        self.tr, self.hist, self.group = trace, hist, group
        self.world = dist.get_world_size(group)
        self.gathered = torch.empty(self.world * hist.words, dtype=torch.int64, device=hist.packed.device)
        self.ws = torch.empty(len(_WS_SLOTS), dtype=torch.int64, device=hist.packed.device)
        self.mk = torch.empty(2, dtype=torch.int64, device=hist.packed.device)
        self.mk_all = torch.empty(2 * self.world, dtype=torch.int64, device=hist.packed.device)

    def merge(self):
        from . import T_UNIQUE_PAGES

        h = self.hist
        self.ws.copy_(h.totals[list(_WS_SLOTS)])
        self.mk.copy_(h.totals[_MK:_MK + 2])
        merge_counts(h.packed, self.group)
        merge_max_kernel(self.tr, h.totals, self.mk, self.mk_all, self.group)
        gather_bitmaps(h.page_bitmap, self.group, out=self.gathered)
        self.tr.bitmap_or(self.gathered, self.world, h.words, h.page_bitmap,
                          h.totals[T_UNIQUE_PAGES:T_UNIQUE_PAGES + 1])
        merge_max(self.ws, self.group)
        h.totals[list(_WS_SLOTS)] = self.ws


def _topk_buffers(self, ks, dev, alloc):
    """Top-K buffers of a merger: ONE selection for k_max = max(ks) (local list, the g
    gathered candidate lists, the merged list); the other k are prefixes of the merged
    top-k_max list (R10's order is total), copied by pasta_topk_prefix."""
    self.ks = tuple(dict.fromkeys(int(k) for k in ks))
    self.kmax = max(self.ks)
    km = self.kmax
    self.loc = (alloc(km, dtype=torch.int64, device=dev), alloc(km, dtype=torch.int64, device=dev),
                alloc(1, dtype=torch.int64, device=dev))
    self.cand = (torch.empty(self.world * km, dtype=torch.int64, device=dev),
                 torch.empty(self.world * km, dtype=torch.int64, device=dev))
    self.out = {k: (torch.empty(k, dtype=torch.int64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
                    torch.empty(1, dtype=torch.int64, device=dev)) for k in self.ks}


def _topk_prefixes(self):
    rest = [k for k in self.ks if k != self.kmax]
    if rest:
        self.tr.topk_prefix(self.out[self.kmax], self.kmax, rest, [self.out[k] for k in rest])


class ShardedMerger:
    """Merge with the page counts left sharded (strong scaling):

    * all_reduce(SUM) of the small part [alloc_counts | totals], all_reduce(MAX) of WS;
    * reduce_scatter(SUM) of the page counts: rank r holds the merged counts of pages
      [r*S, (r+1)*S) (half the bytes of an all_reduce, and no rank holds all P);
    * all_gather of the local page bitmaps + pasta_bitmap_or -> the global bitmap and
      unique pages on every rank (NCCL has no OR);
    * top-K: each rank selects the top-k of its shard (pasta_topk), the candidates are
      all_gathered and pasta_topk_merge picks the global top-k (exact: a page of the
      global top-k is in its own shard's top-k).
    Histograms must be allocated with pad_pages_to = world * 64."""

    def __init__(self, trace, hist, ks, group=None):
        self.tr, self.hist, self.group = trace, hist, group
        self.world = dist.get_world_size(group)
        assert hist.P_pad % (self.world * 64) == 0, "allocate Histograms with pad_pages_to = world * 64"
        dev = hist.packed.device
        self.S = hist.P_pad // self.world
        self.shard = torch.empty(self.S, dtype=torch.int64, device=dev)
        self.gathered = torch.empty(self.world * hist.words, dtype=torch.int64, device=dev)
        self.ws = torch.empty(len(_WS_SLOTS), dtype=torch.int64, device=dev)
        self.mk = torch.empty(2, dtype=torch.int64, device=dev)
        self.mk_all = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
        _topk_buffers(self, ks, dev, torch.empty)

    def merge(self):
        from . import T_UNIQUE_PAGES

        h = self.hist
        self.ws.copy_(h.totals[list(_WS_SLOTS)])
        self.mk.copy_(h.totals[_MK:_MK + 2])
        dist.all_reduce(h.small, op=dist.ReduceOp.SUM, group=self.group)
        merge_max_kernel(self.tr, h.totals, self.mk, self.mk_all, self.group)
        reduce_scatter_counts(h.pages_padded, self.shard, self.group)
        gather_bitmaps(h.page_bitmap, self.group, out=self.gathered)
        self.tr.bitmap_or(self.gathered, self.world, h.words, h.page_bitmap,
                          h.totals[T_UNIQUE_PAGES:T_UNIQUE_PAGES + 1])
        merge_max(self.ws, self.group)
        h.totals[list(_WS_SLOTS)] = self.ws
        km = self.kmax
        lp, lc, _ = self.tr.topk(self.shard, km, out=self.loc)
        cp, cc = self.cand
        gather_candidates(lp, lc, cp, cc, self.group)
        self.tr.topk_merge(cp, cc, self.world, km, self.S, self.out[km])
        _topk_prefixes(self)
        return self.out


class PeerMerger:
    """ShardedMerger's results through peer memory instead of NCCL data movement
    (DESIGN.md section 5). Every rank maps the other ranks' result buffers once, with
    CUDA IPC handles exported and opened by libpasta in the trace handle's own device
    context (pasta_ipc_export / pasta_ipc_open, lazy peer access: NVLink / NVSwitch loads
    at run time); the handles travel over the process group once. A merge is then:

    1. barrier -- every rank's local analyze is complete;
    2. pasta_peer_reduce: my page shard of every rank -> merged counts + the shard's
       bitmap words + its unique-page count (one kernel); pasta_peer_reduce_small: the
       small part [alloc counts | totals | tensor counts] of every rank, SUM except
       WS_OBJ / WS_TENSOR (MAX), the MAX_MEM_REFERENCED_KERNEL pair (ARGMAX) and
       UNIQUE_PAGES (recomputed below) -- one kernel; the shard's top-k per K;
    3. barrier -- every shard, bitmap word, count and candidate list is ready;
    4. pasta_peer_gather: the peers' shard bitmaps into my page bitmap, the merged small
       part into my histograms, the shards' unique-page counts added up, the peers'
       candidates -- ONE kernel; pasta_topk_merge per K;
    5. barrier -- nobody reads this rank's buffers any more (the next step may zero them).

    With an NCCL group the barriers are stream-ordered (an all_reduce of one word on the
    trace's stream): the merge never waits on the host. With gloo (tests: several ranks
    on one GPU) they are host barriers after a stream synchronize.

    Outputs as ShardedMerger: hist.small merged, hist.page_bitmap and totals[UNIQUE_PAGES]
    global, the rank's merged page shard in `shard`, the global top-k lists (returned),
    totals[MAX_KERNEL, MAX_KERNEL_RECORDS] by ARGMAX (exact for kernel-aligned shards with
    Histograms.kernel_row0 = the shard's first kernel). Histograms must be allocated with
    pad_pages_to = world * 64."""

    def __init__(self, trace, hist, ks, group=None):
        self.tr, self.hist, self.group = trace, hist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        assert hist.P_pad % (self.world * 64) == 0, "allocate Histograms with pad_pages_to = world * 64"
        dev = hist.packed.device
        self.dev = dev
        self.nccl = dist.get_backend(group) == "nccl"
        self.S = hist.P_pad // self.world
        self.Sw = self.S // 64
        self.shard = torch.zeros(self.S, dtype=torch.int64, device=dev)
        self.shard_bm = torch.zeros(self.Sw, dtype=torch.int64, device=dev)
        self.pop = torch.zeros(1, dtype=torch.int64, device=dev)
        self.small_out = torch.zeros_like(hist.small)
        self.flag = torch.zeros(1, dtype=torch.int64, device=dev)
        _topk_buffers(self, ks, dev, torch.zeros)
        mine = [hist.packed, self.shard_bm, self.pop, self.loc[0], self.loc[1]]
        torch.cuda.synchronize(dev)
        # own buffers are used directly; the others' through libpasta's IPC mappings
        handles = [trace.ipc_export(t) for t in mine] if self.world > 1 else []
        allh = [None] * self.world
        dist.all_gather_object(allh, (dev.index if dev.index is not None else torch.cuda.current_device(), handles),
                               group=group)
        self.peers, self._opened, err = [], [], None
        try:
            for r, (devr, hs) in enumerate(allh):
                if r == self.rank:
                    self.peers.append([t.data_ptr() for t in mine])
                    continue
                if devr != dev.index:
                    trace.enable_peer(devr)
                ptrs = [trace.ipc_open(hb) for hb in hs]
                self._opened += ptrs
                self.peers.append(ptrs)
        except Exception as exc:  # e.g. no peer access between these GPUs
            err = f"rank {self.rank}: {exc!r}"
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)  # every rank takes the same decision
        bad = [e for e in errs if e]
        if bad:
            self.close()
            raise RuntimeError("peer mapping failed: " + "; ".join(bad))
        self._plan()

    def _plan(self):
        """The fixed argument lists of every merge (addresses never change)."""
        from . import PASTA_COPY, PASTA_COPY_ADD, PASTA_PEER_ARGMAX, PASTA_PEER_MAX, PASTA_PEER_ZERO, T_UNIQUE_PAGES

        h, W, S, Sw = self.hist, self.world, self.S, self.Sw
        P_pad, mi = h.P_pad, h.max_ids
        self.n_small = h.small.numel()
        self.src_shard = [p[0] + 8 * self.rank * S for p in self.peers]
        self.src_small = [p[0] + 8 * P_pad for p in self.peers]
        u = mi + T_UNIQUE_PAGES
        self.slots = [(mi + s, PASTA_PEER_MAX) for s in _WS_SLOTS] + [(mi + _MK, PASTA_PEER_ARGMAX),
                                                                       (u, PASTA_PEER_ZERO)]
        so, hs = self.small_out.data_ptr(), h.small.data_ptr()
        cp = []
        # the peers' shard bitmap words -> my global bitmap (its padding words stay out)
        for r, p in enumerate(self.peers):
            n = min(Sw, h.words - r * Sw)
            if n > 0:
                cp.append((p[1], h.page_bitmap.data_ptr() + 8 * r * Sw, n, PASTA_COPY))
        # merged small part -> my histograms; unique pages = sum of the shards' counts: the
        # one-word entries of one word run on one thread in table order (copy, then adds)
        cp.append((so, hs, u, PASTA_COPY))
        cp.append((so + 8 * u, hs + 8 * u, 1, PASTA_COPY))
        if self.n_small > u + 1:
            cp.append((so + 8 * (u + 1), hs + 8 * (u + 1), self.n_small - u - 1, PASTA_COPY))
        for p in self.peers:
            cp.append((p[2], hs + 8 * u, 1, PASTA_COPY_ADD))
        cpp, ccc, k = self.cand[0], self.cand[1], self.kmax
        for r, p in enumerate(self.peers):
            cp.append((p[3], cpp.data_ptr() + 8 * r * k, k, PASTA_COPY))
            cp.append((p[4], ccc.data_ptr() + 8 * r * k, k, PASTA_COPY))
        assert len(cp) <= 120, "too many peer copies for one pasta_peer_gather"
        self.copies = cp

    def _barrier(self):
        if self.nccl:
            dist.all_reduce(self.flag, group=self.group)  # stream-ordered (NCCL on the current stream)
        else:
            self.tr.sync()
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=self.group)

    def merge(self):
        tr = self.tr
        with torch.cuda.stream(tr.stream):
            self.pop.zero_()
            self._barrier()  # every rank's local analyze is complete
            tr.peer_reduce(self.src_shard, 0, self.S, self.shard, self.shard_bm, self.pop)
            tr.peer_reduce_small(self.src_small, 0, self.n_small, self.slots, self.small_out)
            tr.topk(self.shard, self.kmax, out=self.loc)
            self._barrier()  # every shard, bitmap word, count and candidate list is ready
            tr.peer_gather(self.copies)
            tr.topk_merge(self.cand[0], self.cand[1], self.world, self.kmax, self.S, self.out[self.kmax])
            _topk_prefixes(self)
            self._barrier()  # nobody reads this rank's buffers any more
        return self.out

    def close(self):
        for ptr in self._opened:
            try:
                self.tr.ipc_close(ptr)
            except Exception:
                pass
        self._opened = []
