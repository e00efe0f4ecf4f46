#!/usr/bin/env python3
"""Benchmark of the PASTA trace-analysis hot path on B200 (one JSON line on rank 0).

A *step* is one pass of the whole hot path (S1 range lookup, S2
page / alloc / per-kernel histograms, S3 bitmap + popcount + per-kernel footprints and
WS, S4 top-K, S5 merge when N > 1) over the workload's synthetic trace, records
already resident in HBM. The default workload is BASELINE config 5 ("llama": 10 * 2^30
8-byte records, 10,000 kernels, ~1,200 tensors, 64 GiB window at 4 KiB pages); it is
sharded kernel-aligned across the N ranks (strong scaling: the same trace for every N).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama] [--impl ours|reference]

N > 1 is launched with torchrun (one process per GPU, NCCL): ranks merge their
histograms with one all_reduce(SUM) of the packed counts, all_gather their page bitmaps
and OR them with the pasta_bitmap_or kernel (NCCL has no OR), then each rank selects
top-K from the merged counts. Times are CUDA events on the launching stream, max over
ranks. `--impl reference` times the CPU oracle (the deliberately slow, correct program)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "trace records analyzed/s (G rec/s) and HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "G rec/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama",
                    choices=["tiny", "rn50", "gpt2m", "uvm", "llama", "s_perm", "s_hot", "s_manyranges"],
                    help="BASELINE config (default: llama, the headline) or a SURVEY section 8d stress row")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--records", "--n", dest="n", type=int, default=None,
                    help="override the record count (testing only)")
    ap.add_argument("--e2e-records", type=int, default=1 << 31, help="cap of the pinned host trace for e2e")
    ap.add_argument("--cpu-sample", type=int, default=1 << 28,
                    help="records in the single-thread oracle's bounded sample")
    ap.add_argument("--cpu-sample-all", type=int, default=1 << 31,
                    help="records in the all-core oracle's bounded sample")
    ap.add_argument("--ref-sample", type=int, default=1 << 28, help="records per --impl reference step (all cores)")
    ap.add_argument("--stream-batch", type=int, default=0,
                    help="also time streaming mode: one pasta_analyze per batch of this many records "
                         "(524288 = the paper's 4 MB buffer), captured in a CUDA graph")
    ap.add_argument("--merge", default="peer", choices=["peer", "nccl"],
                    help="N > 1 merge: peer = pasta_peer_reduce over CUDA-IPC-mapped peer memory (dist.PeerMerger), "
                         "nccl = reduce_scatter / all_gather + pasta_bitmap_or (dist.ShardedMerger)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config):
    """dram bytes per scan launch from the committed ncu --set full summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "scan_traffic.json")) as f:
            d = json.load(f)
        return d.get(config)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent NVML sampling of SM clock and throttle reasons while the
    timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle leg
def host_cpu():
    """(logical CPUs this process may use, CPU model name from /proc/cpuinfo)."""
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        n = os.cpu_count() or 1
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return n, model


def oracle_prepare(plan, n_sample, threads=1):
    """The first n_sample records of the workload (host generator, on `threads` threads)
    and their kernel segments (whole kernel prefix + the cut kernel's head). Not timed."""
    import tracegen

    n_sample = min(n_sample, plan.n)
    rec = np.empty(n_sample, dtype=np.uint64)
    step = max(1 << 20, -(-n_sample // max(1, threads)))
    parts = [(j, min(n_sample, j + step)) for j in range(0, n_sample, step)]
    ths = [threading.Thread(target=tracegen.host_records, args=(plan, j0, j1, rec[j0:j1])) for j0, j1 in parts]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    ko = plan.kernel_offsets.astype(np.int64)
    k1 = int(np.searchsorted(ko, n_sample, side="right")) - 1
    sub = [int(x) for x in ko[: k1 + 1]]
    if sub[-1] != n_sample:
        sub.append(n_sample)
    return rec, sub


def oracle_run(plan, rec, sub, threads=1):
    """Time the oracle (as it stands) over the prepared sample: the whole path (lookup,
    histograms, per-kernel rows, bitmap, footprints, top-K). threads == 1: the single-
    thread oracle_analyze; threads > 1: OracleTrace.analyze_parallel (the same C
    definition on kernel-aligned slabs, per-thread arrays summed)."""
    import oracle

    o = oracle.OracleTrace(plan.va_lo, plan.va_hi, len(plan.allocs), len(plan.allocs))
    for b, s in plan.allocs:
        o.register_alloc(b, s)
    t0 = time.perf_counter()
    if threads > 1:
        o.analyze_parallel(rec, sub, plan.page_shift, kernel_rows=True, kernel_pages=plan.want_kernel_pages,
                           threads=threads)
    else:
        o.analyze(rec, sub, plan.page_shift, kernel_rows=True, kernel_pages=plan.want_kernel_pages)
    o.bitmap()
    o.footprints()
    for K in plan.topk:
        o.topk(K)
    return time.perf_counter() - t0


def cpu_baseline(plan, args):
    """The oracle timed on this host's cores (rank 0, N = 1 leg): all cores on a bounded
    sample (the headline `value`) and one thread on a smaller one (the paper's CPU tools
    are "typically single" threaded). Generation excluded."""
    nproc, model = host_cpu()
    rec, sub = oracle_prepare(plan, args.cpu_sample_all, threads=nproc)
    dt_all = oracle_run(plan, rec, sub, threads=nproc)
    n_all, nk_all = rec.size, len(sub) - 1
    del rec
    rec, sub = oracle_prepare(plan, args.cpu_sample, threads=nproc)
    dt_one = oracle_run(plan, rec, sub, threads=1)
    n_one, nk_one = rec.size, len(sub) - 1
    return {"value": n_all / dt_all / 1e9, "unit": UNIT, "cores": nproc, "kind": "oracle",
            "sample": f"first {n_all} records ({nk_all} kernel segments) of the {args.config} plan, {nproc} threads "
                      f"(OracleTrace.analyze_parallel), generation excluded",
            "nproc": nproc, "cpu_model": model,
            "single_thread": {"value": n_one / dt_one / 1e9, "unit": UNIT, "cores": 1,
                              "sample": f"first {n_one} records ({nk_one} kernel segments), 1 thread"}}


def run_reference(args):
    import tracegen

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    plan = tracegen.build_plan(args.config, args.seed, args.n)
    nproc, model = host_cpu()
    rec, sub = oracle_prepare(plan, args.ref_sample, threads=nproc)
    n_s = rec.size
    times = []
    for i in range(args.warmup + args.steps):
        dt = oracle_run(plan, rec, sub, threads=nproc)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = n_s * len(times) / tot / 1e9
    sample = (f"first {n_s} records ({len(sub) - 1} kernel segments) of the {args.config} plan per step, "
              f"{nproc} threads (OracleTrace.analyze_parallel), generation excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / len(times) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": args.config, "n_records": n_s, "sample_of": plan.n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": sample,
                             "nproc": nproc, "cpu_model": model},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our leg
# Test-only: PASTA_BENCH_GLOO=1 runs the N > 1 path with a gloo group and every rank on
# cuda:0 (one GPU, several processes), so the multi-rank code is exercised on a one-GPU
# box (tests/test_bench_contract.py). The peer merge works there through CUDA IPC; the
# NCCL merge needs the nccl backend.
_GLOO = os.environ.get("PASTA_BENCH_GLOO") == "1"


def _dist_barrier(local):
    import torch.distributed as dist

    if _GLOO:
        dist.barrier()
    else:
        dist.barrier(device_ids=[local])


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _GLOO else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch

    import paper_2602_22103_b200 as pb
    import tracegen
    from paper_2602_22103_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if _GLOO:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist

        if _GLOO:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    plan = tracegen.build_plan(args.config, args.seed, args.n)
    j0, j1, k0, k1 = plan.shard(rank, world)
    n_loc = j1 - j0
    nk_loc = k1 - k0
    P = plan.n_pages
    stream = torch.cuda.current_stream(dev)

    # ---- inputs resident in HBM (generation not timed) ----
    dp = tracegen.DevicePlan(plan, dev)
    rec = torch.empty(max(1, n_loc), dtype=torch.int64, device=dev)
    tracegen.device_records(dp, rec, j0, j1)
    ko_loc = torch.from_numpy((plan.kernel_offsets[k0:k1 + 1].astype(np.int64) - j0)).to(dev)
    del dp
    torch.cuda.synchronize()

    A = len(plan.allocs)
    tr = pb.Trace(dev, plan.va_lo, plan.va_hi, A, A, stream=stream)
    for b, s in plan.allocs:
        tr.register_alloc(b, s)
    hist = tr.histograms(plan.page_shift, n_kernels=nk_loc, kernel_rows=plan.want_kernel_rows,
                         kernel_pages=plan.want_kernel_pages, pad_pages_to=64 * world, kernel_row0=k0)
    # N > 1: each rank merges its page shard from every rank's counts over peer memory
    # (dist.PeerMerger) or through NCCL (dist.ShardedMerger); top-K from shard candidates
    merger, merge_kind = None, None
    if world > 1:
        if args.merge == "peer":
            try:
                merger, merge_kind = pdist.PeerMerger(tr, hist, plan.topk, group), "peer"
            except Exception as exc:  # no peer access / IPC on this node: the NCCL merge
                print(f"bench: peer merge unavailable ({exc!r}); using the NCCL merge", file=sys.stderr)
        if merger is None:
            merger, merge_kind = pdist.ShardedMerger(tr, hist, plan.topk, group), "nccl"
    ks = list(dict.fromkeys(plan.topk))
    top_outs = [(torch.empty(k, dtype=torch.int64, device=dev), torch.empty(k, dtype=torch.int64, device=dev),
                 torch.empty(1, dtype=torch.int64, device=dev)) for k in ks]
    top_out = top_outs[ks.index(max(ks))]

    def step():
        hist.zero_()
        tr.analyze(rec, plan.page_shift, hist, kernel_offsets=ko_loc, n=n_loc, finalize=True)
        if merger is not None:
            merger.merge()
        else:  # every top-k list of the config from one selection (pasta_topk_many)
            tr.topk_many(hist.page_counts, ks, top_outs)

    def barrier():
        if world > 1:
            _dist_barrier(local)
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    tr.reset_timing()
    tr.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    tr.set_timing(False)
    phases, launches = tr.timing()
    ms_max = _max_over_ranks(ms, dev) if world > 1 else ms

    # ---- correctness guard (cheap invariants on the merged result) ----
    tot = hist.totals.cpu().numpy().view(np.uint64)
    assert int(tot[0]) == plan.n, (int(tot[0]), plan.n)
    dump = os.environ.get("PASTA_BENCH_DUMP")
    if dump:  # test hook: every merged output of one more step, per rank (tests/test_bench_contract.py)
        step()
        if merger is not None:
            tops = {k: tuple(t.cpu().numpy().view(np.uint64).copy() for t in merger.out[k]) for k in plan.topk}
            shard, S = merger.shard.cpu().numpy().view(np.uint64).copy(), merger.S
        else:
            tops = {k: tuple(t.cpu().numpy().view(np.uint64).copy() for t in o)
                    for k, o in tr.topk_many(hist.page_counts, ks).items()}
            shard, S = hist.page_counts.cpu().numpy().view(np.uint64).copy(), P
        torch.cuda.synchronize()
        np.savez(f"{dump}.rank{rank}.npz", shard=shard, S=S, small=hist.small.cpu().numpy().view(np.uint64),
                 bitmap=hist.page_bitmap.cpu().numpy().view(np.uint64),
                 **{f"top{k}_{i}": v for k, t in tops.items() for i, v in enumerate(t)})

    gb_scan = 8.0 * n_loc / 1e9
    scan_ms = phases["scan"] / args.steps
    peak, peak_src = peaks()
    achieved = gb_scan / (scan_ms / 1e3) if scan_ms > 0 else None
    value = plan.n * args.steps / (ms_max / 1e3) / 1e9

    # ---- e2e: same metric through the C ABI from pinned HOST memory ----
    stream_res = None
    if args.stream_batch:
        stream_res = run_stream(args, plan, rec, n_loc, ko_loc, nk_loc, dev, int(hist.totals[0].item()))
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, plan, tr, hist, rec, n_loc, ko_loc, j0, k0, world, group, local, dev, ks, top_outs)
    del rec
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(plan, args)
    if rank == 0:
        traffic = ncu_traffic(args.config)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (tracegen plan, seed %d; records generated on the device, untimed)" % args.seed,
            "config": {"workload": plan.name, "n_records": plan.n, "kernels": plan.n_kernels, "allocs": A,
                       "page_shift": plan.page_shift, "window_bytes": plan.va_hi - plan.va_lo, "pages": P,
                       "topk": plan.topk, "kernel_rows": plan.want_kernel_rows,
                       "kernel_pages": plan.want_kernel_pages,
                       "shard": "kernel-aligned contiguous, %d records on rank 0" % n_loc,
                       "merge": merge_kind,
                       "l2": "inputs (%.1f GiB/rank) larger than L2; no flush" % (8 * n_loc / 2**30)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "pasta scan_kernel", "algorithmic_bytes_per_launch": 8 * n_loc,
                         "avg_launch_ms": scan_ms, "peak_source": peak_src},
            "phases_ms_per_step": {k: v / args.steps for k, v in phases.items()},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "frac_of_8TBs_spec": (achieved / 8000.0) if achieved else None,
        }
        if stream_res is not None:
            line["stream"] = stream_res
        print(json.dumps(line), flush=True)
    if world > 1:
        _dist_barrier(local)
        torch.distributed.destroy_process_group()


def run_stream(args, plan, rec, n_loc, ko_loc, nk_loc, dev, expect_records):
    """Streaming mode (NEXT f2): the same records analyzed as fixed-size batches, one
    pasta_analyze (NO_FINALIZE) per batch plus one pasta_finalize, on a dedicated stream;
    timed eagerly and as one CUDA-graph replay of all the calls."""
    import torch

    import paper_2602_22103_b200 as pb
    from paper_2602_22103_b200.stream import BatchRunner

    s = torch.cuda.Stream(dev)
    A = len(plan.allocs)
    tr = pb.Trace(dev, plan.va_lo, plan.va_hi, A, A, stream=s)
    for b, sz in plan.allocs:
        tr.register_alloc(b, sz)
    h = tr.histograms(plan.page_shift, n_kernels=nk_loc, kernel_rows=plan.want_kernel_rows,
                      kernel_pages=plan.want_kernel_pages)
    runner = BatchRunner(tr, h, rec, ko_loc.cpu().numpy(), n_loc, args.stream_batch, plan.page_shift)

    def once():
        h.zero_()
        runner.run()
        tr.finalize(plan.page_shift, h, n_kernels=nk_loc)

    with torch.cuda.stream(s):
        once()  # also uploads the range table
    s.synchronize()
    assert int(h.totals[0].item()) == expect_records
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            once()
        e1.record(s)
    s.synchronize()
    eager_ms = e0.elapsed_time(e1) / reps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        once()
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    s.synchronize()
    graph_ms = e0.elapsed_time(e1) / reps
    assert int(h.totals[0].item()) == expect_records
    calls = len(runner.calls)
    # persistent ring consumer: one launch, the host publishing batch descriptors into a
    # ring of 256 while it runs (events on the consumer's stream around open .. close)
    from paper_2602_22103_b200.stream import StreamRing

    ring_ms = []
    ring = StreamRing(tr, h, rec, ko_loc.cpu().numpy(), n_loc - (n_loc % 2), args.stream_batch, plan.page_shift,
                      slots=256)
    for rep in range(1 + reps):
        h.zero_()
        torch.cuda.synchronize(dev)
        e0.record(s)
        ring.run()
        e1.record(s)
        ring.destroy()
        s.synchronize()
        if rep:
            ring_ms.append(e0.elapsed_time(e1))
    assert int(h.totals[0].item()) == n_loc - (n_loc % 2)
    ring_t = sum(ring_ms) / len(ring_ms)
    tr.close()
    return {"batch_records": args.stream_batch, "calls": calls, "unit": "G rec/s",
            "graph_value": n_loc / (graph_ms / 1e3) / 1e9, "graph_ms": graph_ms,
            "eager_value": n_loc / (eager_ms / 1e3) / 1e9, "eager_ms": eager_ms,
            "graph_us_per_call": graph_ms * 1e3 / calls,
            "ring_value": (n_loc - n_loc % 2) / (ring_t / 1e3) / 1e9, "ring_ms": ring_t,
            "ring_us_per_batch": ring_t * 1e3 / len(ring.batches), "ring_slots": 256,
            "ring_path": "pasta_stream_open + pasta_stream_push (host publishes while the consumer runs) + close"}


def run_e2e(args, plan, tr, hist, rec, n_loc, ko_loc, j0, k0, world, group, local, dev, ks, top_outs):
    """End to end through the public API: every step copies its records from pinned
    host memory (inside pasta_analyze, chunked and overlapped with the scan), runs the
    whole path, and reads the results (totals + top-K) back to the host."""
    import torch

    top_out = top_outs[ks.index(max(ks))]

    import paper_2602_22103_b200 as pb

    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    # every rank of this node pins its own host copy: share 40 % of the node's free RAM
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    n_e = max(1, min(n_loc, args.e2e_records, int(avail * 0.4) // max(1, local_world) // 8))
    # the e2e trace is the kernel-aligned prefix of this rank's shard that fits in RAM
    ko_loc_np = ko_loc.cpu().numpy()
    kcut = int(np.searchsorted(ko_loc_np, n_e, side="right")) - 1
    if kcut >= 1:
        n_e = int(ko_loc_np[kcut])
        ko_e = ko_loc_np[: kcut + 1]
    else:  # the first kernel alone exceeds the cap: cut it
        ko_e = np.array([0, n_e], dtype=np.int64)
    host = torch.empty(n_e, dtype=torch.int64, pin_memory=True)
    host.copy_(rec[:n_e])
    ko_h = torch.from_numpy(ko_e.astype(np.int64)).pin_memory()
    h_e = tr.histograms(plan.page_shift, n_kernels=len(ko_e) - 1, kernel_rows=plan.want_kernel_rows,
                        kernel_pages=plan.want_kernel_pages, pad_pages_to=64 * world, kernel_row0=k0)
    from paper_2602_22103_b200 import dist as pdist

    merger = None
    if world > 1:  # the same merge as the device-resident step
        if args.merge == "peer":
            try:
                merger = pdist.PeerMerger(tr, h_e, plan.topk, group)
            except Exception as exc:
                print(f"bench: e2e peer merge unavailable ({exc!r}); using the NCCL merge", file=sys.stderr)
        if merger is None:
            merger = pdist.ShardedMerger(tr, h_e, plan.topk, group)
    res_host = torch.empty(pb.TOTALS + 2 * top_out[0].numel() + 1, dtype=torch.int64, pin_memory=True)
    K = top_out[0].numel()

    def step():
        h_e.zero_()
        tr.analyze(host, plan.page_shift, h_e, kernel_offsets=ko_h, n=n_e, host=True)
        if merger is not None:
            outs = merger.merge()
            res = outs[max(plan.topk)]
        else:
            tr.topk_many(h_e.page_counts, ks, top_outs)
            res = top_out
        T = pb.TOTALS
        res_host[:T].copy_(h_e.totals, non_blocking=True)
        res_host[T:T + K].copy_(res[0], non_blocking=True)
        res_host[T + K:T + 2 * K].copy_(res[1], non_blocking=True)
        res_host[T + 2 * K:].copy_(res[2], non_blocking=True)

    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        _dist_barrier(local)
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    n_tot = n_e * world
    out = {"value": n_tot * steps / (ms / 1e3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * n_e + ko_h.numel() * 8,
           "d2h_bytes_per_step": res_host.numel() * 8, "records_per_rank": n_e, "steps": steps,
           "path": "pasta_analyze(PASTA_REC_HOST) from pinned host memory + finalize + top-K + D2H of results",
           "sample": "kernel-aligned prefix of each rank's shard (%d of %d records)" % (n_e, n_loc)}
    del host
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
