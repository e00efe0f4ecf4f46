"""GPU tests of the peer-memory merge: pasta_peer_reduce against
plain numpy sums / maxes / bitmaps, and dist.PeerMerger with two processes on one GPU
(CUDA IPC mappings of each other's buffers, a gloo group for the handle exchange and
barriers) against the oracle over the whole trace (SPEC S:291-299 partition fold).
The box has one GPU, so the peer loads stay on the device; on an NVSwitch box the
same mappings are NVLink loads."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2602_22103_b200 as pb  # noqa: E402
import oracle  # noqa: E402
import tracegen  # noqa: E402
from tests.harness import u64  # noqa: E402

DEV = torch.device("cuda:0")


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(DEV)


@pytest.mark.parametrize("g", [1, 3, 8, 16])
def test_peer_reduce_sum_bitmap_max(g):
    rng = np.random.default_rng(g)
    n_all = 64 * 1001
    srcs = []
    for r in range(g):
        a = rng.integers(0, 1 << 64, size=n_all, dtype=np.uint64)
        a[rng.random(n_all) < 0.7] = 0  # zero pages
        srcs.append(a)
    srcs[0][:64 * 3] = 0  # words with no set bit in any source
    for a in srcs[1:]:
        a[:64 * 3] = 0
    dsrc = [_t(a) for a in srcs]
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    lo, n = 64 * 7, 64 * 990
    out = torch.zeros(n, dtype=torch.int64, device=DEV)
    bm = torch.zeros(n // 64, dtype=torch.int64, device=DEV)
    pop = torch.full((1,), 5, dtype=torch.int64, device=DEV)
    tr.peer_reduce(dsrc, lo, n, out, bm, pop)
    mx = torch.zeros(n - 3, dtype=torch.int64, device=DEV)
    tr.peer_reduce(dsrc, lo + 1, n - 3, mx, op=pb.PASTA_PEER_MAX)
    tr.sync()
    with np.errstate(over="ignore"):
        ref = np.zeros(n, dtype=np.uint64)
        for a in srcs:
            ref += a[lo:lo + n]
    assert np.array_equal(u64(out), ref)
    bits = (ref != 0).reshape(-1, 64)
    ref_bm = (bits.astype(np.uint64) << np.arange(64, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
    assert np.array_equal(u64(bm), ref_bm)
    assert int(u64(pop)[0]) == 5 + int((ref != 0).sum())
    ref_max = np.max(np.stack([a[lo + 1:lo + 1 + n - 3] for a in srcs]), axis=0)
    assert np.array_equal(u64(mx), ref_max)
    # misaligned bitmap ranges, too many sources, MAX with a bitmap: EINVAL
    for args, kw in (((dsrc, lo + 1, n, out, bm), {}), ((dsrc, lo, n - 1, out, bm), {}),
                     ((dsrc * 17, lo, 64, out), {}), ((dsrc, lo, n, out, bm), {"op": pb.PASTA_PEER_MAX})):
        with pytest.raises(pb.PastaError):
            tr.peer_reduce(*args, **kw)
    tr.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, two):
    import traceback

    try:
        _work(rank, world, port, q, two)
    except BaseException:  # report instead of leaving the parent waiting on the queue
        q.put(("error", rank, traceback.format_exc()))
        raise


def _work(rank, world, port, q, two):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22103_b200 import dist as pdist

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        p = tracegen.build_plan("tiny", seed=17)
        j0, j1, k0, k1 = p.shard(rank, world)
        rec = torch.empty(j1 - j0, dtype=torch.int64, device=dev)
        tracegen.device_records(tracegen.DevicePlan(p, dev), rec, j0, j1)
        ko = torch.from_numpy((p.kernel_offsets[k0:k1 + 1] - np.uint64(j0)).view(np.int64).copy()).to(dev)
        objs = p.objects if two else p.allocs
        kw = dict(max_live_tensors=len(p.allocs), max_tensor_ids=len(p.allocs)) if two else {}
        tr = pb.Trace(dev, p.va_lo, p.va_hi, len(objs), len(objs), **kw)
        for b, s in objs:
            tr.register_alloc(b, s)
        if two:
            for b, s in p.allocs:
                tr.register_tensor(b, s)
        hist = tr.histograms(p.page_shift, n_kernels=k1 - k0, kernel_rows=True, pad_pages_to=64 * world,
                             kernel_row0=k0)
        merger = pdist.PeerMerger(tr, hist, (16, 3))
        for step in range(2):  # a second merge on re-analyzed buffers (barrier discipline)
            hist.zero_()
            tr.analyze(rec, p.page_shift, hist, kernel_offsets=ko)
            outs = merger.merge()
            tr.sync()
            torch.cuda.synchronize()
        q.put((rank, u64(merger.shard).copy(), u64(hist.small).copy(), u64(hist.page_bitmap).copy(),
               {k: tuple(u64(x).copy() for x in v) for k, v in outs.items()}, merger.S))
        dist.barrier()
        tr.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,two", [(2, False), (3, False), (2, True)])
def test_peer_merger_ranks_on_one_gpu(world, two):
    """two = objects (4 MiB blocks) + tensors (the allocations): tensor counts (SUM),
    untensored total and WS_tensor (MAX) merged too."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, two)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get()
        assert r[0] != "error", f"rank {r[1]} failed:\n{r[2]}"
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0

    p = tracegen.build_plan("tiny", seed=17)
    objs = p.objects if two else p.allocs
    kw = dict(max_live_tensors=len(p.allocs), max_tensor_ids=len(p.allocs)) if two else {}
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(objs), len(objs), **kw)
    for b, s in objs:
        o.register_alloc(b, s)
    if two:
        for b, s in p.allocs:
            o.register_tensor(b, s)
    o.analyze(tracegen.host_records(p), p.kernel_offsets, p.page_shift, kernel_rows=True)
    bm, uniq = o.bitmap()
    S = res[0][5]
    pages = np.zeros(world * S, dtype=np.uint64)
    pages[:len(o.page_counts)] = o.page_counts
    A = len(objs)
    for r in range(world):
        _, shard, small, pbm, outs, _ = res[r]
        assert np.array_equal(shard, pages[r * S:(r + 1) * S]), f"rank {r}: merged page shard"
        assert np.array_equal(small[:A], o.alloc_counts[:A]), f"rank {r}: alloc counts"
        tot = small[len(o.alloc_counts):len(o.alloc_counts) + pb.TOTALS]
        assert tot[:3].tolist() == o.totals.tolist(), f"rank {r}: totals"
        assert int(tot[3]) == uniq, f"rank {r}: unique pages"
        fp, ws = o.footprints()
        assert int(tot[4]) == ws, f"rank {r}: WS_obj (MAX)"
        mk = o.max_kernel()
        assert int(tot[pb.T_MAX_KERNEL]) == mk, f"rank {r}: MAX_MEM_REFERENCED_KERNEL (ARGMAX)"
        per = o.kernel_rows.sum(axis=1, dtype=np.uint64) + o.kun
        assert int(tot[pb.T_MAX_KERNEL_RECORDS]) == int(per[mk]), f"rank {r}: its records"
        assert np.array_equal(pbm, bm), f"rank {r}: bitmap"
        if two:
            T = len(p.allocs)
            assert np.array_equal(small[A + pb.TOTALS:A + pb.TOTALS + T], o.tensor_counts), f"rank {r}: tensor counts"
            assert int(tot[pb.T_UNTENSORED]) == o.untensored, f"rank {r}: untensored"
            assert int(tot[pb.T_WS_TENSOR]) == o.tensor_footprints()[1], f"rank {r}: WS_tensor (MAX)"
        for k in (16, 3):
            rp, rc, rf = oracle.topk(o.page_counts, k)
            assert int(outs[k][2][0]) == rf and np.array_equal(outs[k][0], rp) and np.array_equal(outs[k][1], rc), \
                f"rank {r}: top-{k}"


def test_peer_merger_world1_nccl():
    """PeerMerger through an NCCL group (the bench's N > 1 configuration, here at world
    size 1): the handle exchange and barriers run on NCCL, and the merged results equal
    the single-GPU ones."""
    import torch.distributed as dist

    from paper_2602_22103_b200 import dist as pdist

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=DEV)
    try:
        p = tracegen.build_plan("tiny", seed=19)
        rec = torch.empty(p.n, dtype=torch.int64, device=DEV)
        tracegen.device_records(tracegen.DevicePlan(p, DEV), rec)
        ko = torch.from_numpy(p.kernel_offsets.view(np.int64).copy()).to(DEV)
        tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
        for b, s in p.allocs:
            tr.register_alloc(b, s)
        hist = tr.histograms(p.page_shift, n_kernels=p.n_kernels, kernel_rows=True, pad_pages_to=64)
        tr.analyze(rec, p.page_shift, hist, kernel_offsets=ko)
        ref = tuple(u64(x).copy() for x in tr.topk(hist.page_counts, 16))
        tr.sync()
        totals, bm = u64(hist.totals).copy(), u64(hist.page_bitmap).copy()
        outs = pdist.PeerMerger(tr, hist, (16,)).merge()
        tr.sync()
        torch.cuda.synchronize()
        assert all(np.array_equal(u64(a), b) for a, b in zip(outs[16], ref))
        assert np.array_equal(u64(hist.totals), totals)  # every slot, the ARGMAX pair included
        o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
        for b, s in p.allocs:
            o.register_alloc(b, s)
        o.analyze(tracegen.host_records(p), p.kernel_offsets, p.page_shift, kernel_rows=True)
        assert int(totals[pb.T_MAX_KERNEL]) == o.max_kernel()
        assert np.array_equal(u64(hist.page_bitmap), bm)
        tr.close()
    finally:
        dist.destroy_process_group()


def test_peer_argmax_pairs():
    """PASTA_PEER_ARGMAX: the (index, records) pair with the most records, ties to the
    lowest index (the MAX_MEM_REFERENCED_KERNEL merge, R24), over 1-16 sources; n != 2
    is EINVAL."""
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    rng = np.random.default_rng(5)
    for g in (1, 2, 3, 8, 16):
        for trial in range(20):
            vals = rng.integers(0, 4, size=g).astype(np.uint64)  # many ties
            if trial % 5 == 0:
                vals[rng.integers(0, g)] = np.uint64((1 << 64) - 1)
            idx = rng.permutation(10 * g)[:g].astype(np.uint64)
            buf = torch.from_numpy(np.stack([idx, vals], axis=1).reshape(-1).view(np.int64).copy()).to(DEV)
            out = torch.zeros(2, dtype=torch.int64, device=DEV)
            tr.peer_reduce([buf.data_ptr() + 16 * r for r in range(g)], 0, 2, out, op=pb.PASTA_PEER_ARGMAX)
            tr.sync()
            best = max(range(g), key=lambda r: (int(vals[r]), -int(idx[r])))
            assert u64(out).tolist() == [int(idx[best]), int(vals[best])], (g, trial)
    with pytest.raises(pb.PastaError) as ei:
        tr.peer_reduce([buf], 0, 3, out, op=pb.PASTA_PEER_ARGMAX)
    assert ei.value.status == pb.PASTA_EINVAL
    tr.close()


def test_enable_peer_status_codes():
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    tr.enable_peer(DEV.index or 0)  # own device: nothing to enable
    for bad in (-1, torch.cuda.device_count()):
        with pytest.raises(pb.PastaError) as ei:
            tr.enable_peer(bad)
        assert ei.value.status == pb.PASTA_EINVAL
    tr.close()


def test_peer_reduce_small_slots():
    """pasta_peer_reduce_small: SUM except MAX slots, an ARGMAX pair (ties to the lowest
    index) and ZERO slots, over 1-16 sources, one launch; bad slots are EINVAL."""
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    rng = np.random.default_rng(11)
    n = 70_001
    for g in (1, 2, 5, 16):
        srcs = [rng.integers(0, 1 << 62, size=n + 9, dtype=np.uint64) for _ in range(g)]
        am = 777
        for a in srcs:
            a[3 + am + 1] = rng.integers(0, 3)  # tied values at the ARGMAX pair
        dsrc = [_t(a) for a in srcs]
        slots = [(5, pb.PASTA_PEER_MAX), (n - 1, pb.PASTA_PEER_MAX), (am, pb.PASTA_PEER_ARGMAX),
                 (42, pb.PASTA_PEER_ZERO)]
        out = torch.zeros(n, dtype=torch.int64, device=DEV)
        tr.peer_reduce_small(dsrc, 3, n, slots, out)
        tr.sync()
        with np.errstate(over="ignore"):
            ref = np.zeros(n, dtype=np.uint64)
            for a in srcs:
                ref += a[3:3 + n]
        for i in (5, n - 1):
            ref[i] = max(a[3 + i] for a in srcs)
        best = max(range(g), key=lambda r: (int(srcs[r][3 + am + 1]), -int(srcs[r][3 + am])))
        ref[am], ref[am + 1] = srcs[best][3 + am], srcs[best][3 + am + 1]
        ref[42] = 0
        assert np.array_equal(u64(out), ref), g
    out = torch.zeros(8, dtype=torch.int64, device=DEV)
    for bad in ([(8, pb.PASTA_PEER_MAX)], [(7, pb.PASTA_PEER_ARGMAX)], [(0, pb.PASTA_PEER_SUM)],
                [(0, pb.PASTA_PEER_ZERO)] * 17):
        with pytest.raises(pb.PastaError) as ei:
            tr.peer_reduce_small(dsrc, 0, 8, bad, out)
        assert ei.value.status == pb.PASTA_EINVAL
    tr.close()


def test_peer_gather_copies_and_ordered_adds():
    """pasta_peer_gather: copies and atomic adds of many entries in one launch; one-word
    entries into the same word apply in table order (a copy, then adds)."""
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    rng = np.random.default_rng(12)
    srcs = [rng.integers(0, 1 << 40, size=int(m), dtype=np.uint64) for m in rng.integers(1, 50_000, size=40)]
    dsrc = [_t(a) for a in srcs]
    dst = torch.zeros(sum(a.size for a in srcs) + 1, dtype=torch.int64, device=DEV)
    copies, off = [], 0
    for a, d in zip(srcs, dsrc):
        copies.append((d, dst.data_ptr() + 8 * off, a.size, pb.PASTA_COPY))
        off += a.size
    word = dst.data_ptr() + 8 * off
    ones = [_t(np.array([v], dtype=np.uint64)) for v in (5, 7, 11, 13)]
    copies.append((ones[0], word, 1, pb.PASTA_COPY))
    copies += [(o, word, 1, pb.PASTA_COPY_ADD) for o in ones[1:]]
    tr.peer_gather(copies)
    tr.sync()
    ref = np.concatenate(srcs + [np.array([5 + 7 + 11 + 13], dtype=np.uint64)])
    assert np.array_equal(u64(dst), ref)
    with pytest.raises(pb.PastaError):
        tr.peer_gather(copies * 4)  # > 120 entries
    with pytest.raises(pb.PastaError):
        tr.peer_gather([(dsrc[0], dst, 4, 9)])  # bad op
    tr.close()


def test_ipc_export_status_codes():
    """pasta_ipc_export of a caching-allocator tensor (an address inside a larger block):
    offset recorded; a host pointer is EINVAL; opening one's own handle in the exporting
    process is refused by the driver (ECUDA), closing an unknown pointer is ENOENT."""
    import ctypes

    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    big = torch.zeros(1 << 20, dtype=torch.int64, device=DEV)
    hb = tr.ipc_export(big[1000:])
    h = pb.pasta_ipc_handle.from_buffer_copy(hb)
    assert h.offset >= 8000 and h.block_bytes >= 8 << 20 and h.device == (DEV.index or 0)
    host = ctypes.create_string_buffer(64)
    with pytest.raises(pb.PastaError) as ei:
        tr.ipc_export(ctypes.addressof(host))
    assert ei.value.status == pb.PASTA_EINVAL
    with pytest.raises(pb.PastaError) as ei:
        tr.ipc_open(hb)
    assert ei.value.status == pb.PASTA_ECUDA
    with pytest.raises(pb.PastaError) as ei:
        tr.ipc_close(big.data_ptr())
    assert ei.value.status == pb.PASTA_ENOENT
    tr.close()
