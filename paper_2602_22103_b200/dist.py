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
        self.ks = tuple(ks)
        self.loc = {k: (torch.empty(k, dtype=torch.int64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
                        torch.empty(1, dtype=torch.int64, device=dev)) for k in self.ks}
        self.cand = {k: (torch.empty(self.world * k, dtype=torch.int64, device=dev),
                         torch.empty(self.world * k, dtype=torch.int64, device=dev)) for k in self.ks}
        self.out = {k: (torch.empty(k, dtype=torch.int64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
                        torch.empty(1, dtype=torch.int64, device=dev)) for k in self.ks}

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
        for k in self.ks:
            lp, lc, _ = self.tr.topk(self.shard, k, out=self.loc[k])
            cp, cc = self.cand[k]
            gather_candidates(lp, lc, cp, cc, self.group)
            self.tr.topk_merge(cp, cc, self.world, k, self.S, self.out[k])
        return self.out


class PeerMerger:
    """ShardedMerger's results through peer memory instead of NCCL data movement
    (DESIGN.md section 5): every rank maps the other ranks' result buffers once (CUDA
    IPC handles exchanged over the process group; NVLink / NVSwitch loads at run time)
    and one pasta_peer_reduce kernel per merge reads its shard of every rank's page
    counts, writing the merged counts together with the shard's bitmap words and
    unique-page count. A second phase (after a barrier) copies the shard bitmaps,
    unique counts and top-k candidates of the peers the same way. The process group
    carries only the handle exchange and the barriers.

    Outputs as ShardedMerger: hist.small merged (SUMs; WS slots MAX), hist.page_bitmap
    and totals[UNIQUE_PAGES] global, the rank's merged page shard in `shard`, and the
    global top-k lists (returned), totals[MAX_KERNEL, MAX_KERNEL_RECORDS] by ARGMAX (exact
    for kernel-aligned shards with Histograms.kernel_row0 = the shard's first kernel).
    Histograms must be allocated with pad_pages_to = world * 64."""

    def __init__(self, trace, hist, ks, group=None):
        from torch.multiprocessing.reductions import reduce_tensor

        self.tr, self.hist, self.group = trace, hist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        assert hist.P_pad % (self.world * 64) == 0, "allocate Histograms with pad_pages_to = world * 64"
        dev = hist.packed.device
        self.S = hist.P_pad // self.world
        self.Sw = self.S // 64
        self.shard = torch.zeros(self.S, dtype=torch.int64, device=dev)
        self.shard_bm = torch.zeros(self.Sw, dtype=torch.int64, device=dev)
        self.pop = torch.zeros(1, dtype=torch.int64, device=dev)
        self.small_out = torch.zeros_like(hist.small)
        self.bm_full = torch.zeros(self.world * self.Sw, dtype=torch.int64, device=dev)
        self.ks = tuple(ks)
        self.loc = {k: (torch.zeros(k, dtype=torch.int64, device=dev), torch.zeros(k, dtype=torch.int64, device=dev),
                        torch.zeros(1, dtype=torch.int64, device=dev)) for k in self.ks}
        self.cand = {k: (torch.empty(self.world * k, dtype=torch.int64, device=dev),
                         torch.empty(self.world * k, dtype=torch.int64, device=dev)) for k in self.ks}
        self.out = {k: (torch.empty(k, dtype=torch.int64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
                        torch.empty(1, dtype=torch.int64, device=dev)) for k in self.ks}
        mine = [hist.packed, self.shard_bm, self.pop]
        for k in self.ks:
            mine += [self.loc[k][0], self.loc[k][1]]
        torch.cuda.synchronize(dev)
        shared = [reduce_tensor(t) for t in mine] if self.world > 1 else []  # own buffers are used directly
        allh = [None] * self.world
        dist.all_gather_object(allh, (dev.index if dev.index is not None else torch.cuda.current_device(), shared),
                               group=group)
        self.peers, err = [], None
        try:
            for r, (devr, hs) in enumerate(allh):
                if r == self.rank:
                    self.peers.append(mine)
                    continue
                if devr != hist.packed.device.index:
                    trace.enable_peer(devr)
                self.peers.append([fn(*args) for fn, args in hs])
        except Exception as exc:  # e.g. no peer access between these GPUs
            err = f"rank {self.rank}: {exc!r}"
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)  # every rank takes the same decision
        bad = [e for e in errs if e]
        if bad:
            self.peers = []
            raise RuntimeError("peer mapping failed: " + "; ".join(bad))

    def _addr(self, t, elem=0):
        return t.data_ptr() + 8 * elem

    def merge(self):
        from . import PASTA_PEER_ARGMAX, PASTA_PEER_MAX, T_UNIQUE_PAGES

        h, tr, W, S = self.hist, self.tr, self.world, self.S
        P_pad = h.P_pad
        self.pop.zero_()
        torch.cuda.synchronize(h.packed.device)
        tr.sync()
        dist.barrier(group=self.group)  # every rank's local analyze is complete
        # phase 1: my page shard of every rank -> merged counts + bitmap words + popcount
        tr.peer_reduce([self._addr(p[0], self.rank * S) for p in self.peers], 0, S, self.shard, self.shard_bm,
                       self.pop)
        n_small = h.small.numel()
        tr.peer_reduce([self._addr(p[0], P_pad) for p in self.peers], 0, n_small, self.small_out)
        for slot in _WS_SLOTS:
            e = h.max_ids + slot
            tr.peer_reduce([self._addr(p[0], P_pad + e) for p in self.peers], 0, 1, self._addr(self.small_out, e),
                           op=PASTA_PEER_MAX)
        e = h.max_ids + _MK
        tr.peer_reduce([self._addr(p[0], P_pad + e) for p in self.peers], 0, 2, self._addr(self.small_out, e),
                       op=PASTA_PEER_ARGMAX)
        for k in self.ks:
            tr.topk(self.shard, k, out=self.loc[k])
        tr.sync()
        dist.barrier(group=self.group)  # every shard, bitmap word, popcount and candidate list is ready
        # phase 2: the peers' shard bitmaps, unique counts and candidates
        for r, p in enumerate(self.peers):
            tr.peer_reduce([p[1]], 0, self.Sw, self._addr(self.bm_full, r * self.Sw))
        tr.peer_reduce([p[2] for p in self.peers], 0, 1, self._addr(self.small_out, h.max_ids + T_UNIQUE_PAGES))
        for i, k in enumerate(self.ks):
            cp, cc = self.cand[k]
            for r, p in enumerate(self.peers):
                tr.peer_reduce([p[3 + 2 * i]], 0, k, self._addr(cp, r * k))
                tr.peer_reduce([p[4 + 2 * i]], 0, k, self._addr(cc, r * k))
        tr.sync()
        dist.barrier(group=self.group)  # nobody reads this rank's buffers any more
        h.small.copy_(self.small_out)
        h.page_bitmap.copy_(self.bm_full[:h.words])
        for k in self.ks:
            cp, cc = self.cand[k]
            tr.topk_merge(cp, cc, W, k, S, self.out[k])
        return self.out
