"""Multi-GPU merge logic on CPU: world_size 2 (and 4) with the gloo backend.

Each rank analyzes its kernel-aligned shard with the oracle (the CUDA path needs a
GPU; the merge under test is collectives only), packs the results exactly like
paper_2602_22103_b200.Histograms ([page_counts | alloc_counts | totals]) and merges
them with the product helpers of paper_2602_22103_b200.dist: all_reduce(SUM) of the
packed counts, all_gather of bitmaps (the OR itself is the pasta_bitmap_or CUDA
kernel, tested on the GPU; here the gathered rows are OR-ed by the test),
all_reduce(MAX) of WS_obj, and merge_kernel_rows for arbitrary cuts. The merged
result must equal the oracle over the whole trace (SPEC S:291-299 partition fold).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tracegen

TOTALS = 9  # include/pasta.h PASTA_TOTALS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_shard(p, j0, j1, k0, k1, aligned):
    rec = tracegen.host_records(p, j0, j1)
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        o.register_alloc(b, s)
    ko = [int(x) for x in p.kernel_offsets]
    if aligned:
        sub = [x - j0 for x in ko[k0:k1 + 1]]
    else:  # arbitrary cut: kernels overlapping [j0, j1), clipped
        ka = max(k for k in range(len(ko) - 1) if ko[k] <= j0) if j1 > j0 else 0
        kb = min(k for k in range(1, len(ko)) if ko[k] >= j1)
        sub = [0] + [min(max(x - j0, 0), j1 - j0) for x in ko[ka + 1:kb]] + [j1 - j0]
        k0, k1 = ka, kb
    o.analyze(rec, sub, p.page_shift, kernel_rows=True, kernel_pages=True)
    return o, k0, k1


def _worker(rank, world, port, aligned, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22103_b200 import dist as pdist

        p = tracegen.build_plan("tiny", seed=11, n=1 << 17)
        if aligned:
            j0, j1, k0, k1 = p.shard(rank, world)
        else:
            j0, j1 = p.n * rank // world + 777 * rank, p.n * (rank + 1) // world + (777 * (rank + 1) if rank + 1 < world else 0)
            k0 = k1 = 0
        o, k0, k1 = _oracle_shard(p, j0, j1, k0, k1, aligned)
        P, A = o.page_counts.size, len(p.allocs)
        packed = torch.zeros(P + A + TOTALS, dtype=torch.int64)
        packed[:P] = torch.from_numpy(o.page_counts.view(np.int64))
        packed[P:P + A] = torch.from_numpy(o.alloc_counts.view(np.int64))
        packed[P + A:P + A + 3] = torch.from_numpy(o.totals.view(np.int64))
        bm, _ = o.bitmap()
        fp, ws = o.footprints()
        pdist.merge_counts(packed)
        gathered = pdist.gather_bitmaps(torch.from_numpy(bm.view(np.int64)))
        wst = torch.tensor([ws], dtype=torch.int64)
        pdist.merge_max(wst)
        rows = torch.from_numpy(o.kernel_rows.view(np.int64).copy())
        full_rows = pdist.merge_kernel_rows(rows, k0, p.n_kernels)
        # MAX_MEM_REFERENCED_KERNEL: the shard's (global index, records) pair, as finalize
        # writes it into totals[7:9] with kernel_row0 = k0; gathered for the ARGMAX merge
        per = o.kernel_rows.sum(axis=1, dtype=np.uint64) + o.kun
        i = int(np.argmax(per))
        pairs = pdist.gather_pairs(torch.tensor([k0 + i, int(per[i])], dtype=torch.int64))
        if rank == 0:
            out_q.put({"packed": packed.numpy().copy(), "gathered": gathered.numpy().copy(), "ws": int(wst[0]),
                       "rows": full_rows.numpy().copy(), "shard": (j0, j1, k0, k1),
                       "pairs": pairs.numpy().copy()})
    finally:
        dist.destroy_process_group()


def _run(world, aligned):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, aligned, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return res


@pytest.fixture(autouse=True)
def _lib(built):
    return built


@pytest.mark.parametrize("world,aligned", [(2, True), (2, False), (4, True)])
def test_gloo_merge_equals_whole_trace(world, aligned):
    res = _run(world, aligned)
    p = tracegen.build_plan("tiny", seed=11, n=1 << 17)
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        o.register_alloc(b, s)
    o.analyze(tracegen.host_records(p), p.kernel_offsets, p.page_shift, kernel_rows=True)
    P, A = o.page_counts.size, len(p.allocs)
    packed = res["packed"].view(np.uint64)
    assert np.array_equal(packed[:P], o.page_counts)
    assert np.array_equal(packed[P:P + A], o.alloc_counts)
    assert np.array_equal(packed[P + A:P + A + 3], o.totals)
    W = (P + 63) // 64
    merged_bm = np.bitwise_or.reduce(res["gathered"].view(np.uint64).reshape(world, W), axis=0)
    bm, _ = o.bitmap()
    assert np.array_equal(merged_bm, bm)  # OR of shard bitmaps == bitmap of merged counts
    fp, ws = o.footprints()
    if aligned:  # kernel-aligned shards: per-kernel rows are disjoint, so WS = max of shard WS
        assert res["ws"] == ws
        # ... and the ARGMAX of the shards' (index, records) pairs (most records, ties to
        # the lowest index: the rule of pasta_peer_reduce(PASTA_PEER_ARGMAX), tested on the
        # GPU) is the whole trace's MAX_MEM_REFERENCED_KERNEL (R24)
        pairs = res["pairs"].reshape(world, 2)
        best = min(range(world), key=lambda r: (-int(pairs[r, 1]), int(pairs[r, 0])))
        assert int(pairs[best, 0]) == o.max_kernel()
    assert np.array_equal(res["rows"].view(np.uint64), o.kernel_rows)


def test_shard_plan_is_kernel_aligned_and_covering():
    for name in ["tiny", "rn50", "llama"]:
        p = tracegen.build_plan(name)
        ko = [int(x) for x in p.kernel_offsets]
        for world in (1, 2, 4, 8):
            prev = 0
            for r in range(world):
                j0, j1, k0, k1 = p.shard(r, world)
                assert j0 == prev and ko[k0] == j0 and ko[k1] == j1
                prev = j1
                if name == "llama":  # balanced within one kernel's worth of records
                    assert abs((j1 - j0) - p.n / world) <= max(np.diff(ko)) + 1
            assert prev == p.n


def _worker_sharded(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22103_b200 import dist as pdist

        p = tracegen.build_plan("tiny", seed=5, n=1 << 17)
        j0, j1, k0, k1 = p.shard(rank, world)
        o, _, _ = _oracle_shard(p, j0, j1, k0, k1, True)
        P = o.page_counts.size
        P_pad = (P + 64 * world - 1) // (64 * world) * (64 * world)
        pages = torch.zeros(P_pad, dtype=torch.int64)
        pages[:P] = torch.from_numpy(o.page_counts.view(np.int64))
        S = P_pad // world
        shard = torch.empty(S, dtype=torch.int64)
        pdist.reduce_scatter_counts(pages, shard)
        K = 16
        lp, lc, _ = oracle.topk(shard.numpy().view(np.uint64), K)  # stands in for pasta_topk on the shard
        cp = torch.empty(world * K, dtype=torch.int64)
        cc = torch.empty(world * K, dtype=torch.int64)
        pdist.gather_candidates(torch.from_numpy(lp.view(np.int64).copy()), torch.from_numpy(lc.view(np.int64).copy()),
                                cp, cc)
        if rank == 0:
            out_q.put({"shard0": shard.numpy().copy(), "cp": cp.numpy().copy(), "cc": cc.numpy().copy(), "S": S})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_topk_flow(world):
    """reduce_scatter of the page counts + shard-local top-K + all_gather of candidates:
    the best K of the union (global page ids) is the global top-K."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = tracegen.build_plan("tiny", seed=5, n=1 << 17)
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, s in p.allocs:
        o.register_alloc(b, s)
    o.analyze(tracegen.host_records(p), p.kernel_offsets, p.page_shift)
    S = res["S"]
    assert np.array_equal(res["shard0"].view(np.uint64)[: min(S, o.page_counts.size)], o.page_counts[:S])
    K = 16
    cp, cc = res["cp"].view(np.uint64), res["cc"].view(np.uint64)
    cand = [(int(c), int(pg) + (i // K) * S) for i, (pg, c) in enumerate(zip(cp, cc)) if c]
    cand.sort(key=lambda x: (-x[0], x[1]))
    rp, rc, rf = oracle.topk(o.page_counts, K)
    assert [pg for _, pg in cand[:K]] == [int(x) for x in rp[:rf]]
    assert [c for c, _ in cand[:K]] == [int(x) for x in rc[:rf]]


def _worker_tensors(rank, world, port, out_q):
    """Two-level shards (objects = pool chunks, tensors = allocations; NEXT f3): the packed
    buffer carries the tensor counts after the totals, WS_obj and WS_tensor merge by MAX."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22103_b200 import dist as pdist

        p = tracegen.build_plan("tiny", seed=13, n=1 << 17)
        j0, j1, k0, k1 = p.shard(rank, world)
        o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.objects), len(p.objects), max_live_tensors=len(p.allocs),
                               max_tensor_ids=len(p.allocs))
        for b, s in p.objects:
            o.register_alloc(b, s)
        for b, s in p.allocs:
            o.register_tensor(b, s)
        ko = [int(x) for x in p.kernel_offsets]
        o.analyze(tracegen.host_records(p, j0, j1), [x - j0 for x in ko[k0:k1 + 1]], p.page_shift, kernel_rows=True)
        P, A, T = o.page_counts.size, len(p.objects), len(p.allocs)
        packed = torch.zeros(P + A + TOTALS + T, dtype=torch.int64)
        packed[:P] = torch.from_numpy(o.page_counts.view(np.int64))
        packed[P:P + A] = torch.from_numpy(o.alloc_counts.view(np.int64))
        tot = np.zeros(TOTALS, dtype=np.uint64)
        tot[:3] = o.totals
        tot[5] = o.untensored
        tot[4] = o.footprints()[1]
        tot[6] = o.tensor_footprints()[1]
        packed[P + A:P + A + TOTALS] = torch.from_numpy(tot.view(np.int64))
        packed[P + A + TOTALS:] = torch.from_numpy(o.tensor_counts.view(np.int64))
        totals = packed[P + A:P + A + TOTALS]
        ws = totals[list(pdist._WS_SLOTS)].clone()
        pdist.merge_counts(packed)
        pdist.merge_max(ws)
        totals[list(pdist._WS_SLOTS)] = ws
        if rank == 0:
            out_q.put({"packed": packed.numpy().copy()})
    finally:
        dist.destroy_process_group()


def test_gloo_merge_tensor_level():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tensors, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = tracegen.build_plan("tiny", seed=13, n=1 << 17)
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.objects), len(p.objects), max_live_tensors=len(p.allocs),
                           max_tensor_ids=len(p.allocs))
    for b, s in p.objects:
        o.register_alloc(b, s)
    for b, s in p.allocs:
        o.register_tensor(b, s)
    o.analyze(tracegen.host_records(p), p.kernel_offsets, p.page_shift, kernel_rows=True)
    P, A = o.page_counts.size, len(p.objects)
    packed = res["packed"].view(np.uint64)
    tot = packed[P + A:P + A + TOTALS]
    assert np.array_equal(packed[:P], o.page_counts)
    assert np.array_equal(packed[P:P + A], o.alloc_counts)
    assert np.array_equal(packed[P + A + TOTALS:], o.tensor_counts)
    assert tot[:3].tolist() == o.totals.tolist() and int(tot[5]) == o.untensored
    assert int(tot[4]) == o.footprints()[1] and int(tot[6]) == o.tensor_footprints()[1]
