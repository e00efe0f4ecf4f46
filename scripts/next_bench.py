"""Throughput of the SURVEY §8(f) NEXT rows at full size, each against the same scan
without the feature, on one B200 (one JSON line per variant on stdout).

    python scripts/next_bench.py [--reps 5] [--warmup 2] [--only uvm,rich,peer]

uvm (BASELINE config 4: 4e9 8-byte records, 2 MiB blocks, 2,000 kernels, per-kernel
rows + per-kernel page bitmaps):
  base       the §8(a) scan as bench.py runs it on this config
  hot        + f1 hotness matrix, windows of 20 kernels (100 windows x 204,800 blocks)
  twolevel   + f3 objects (pool chunks) and tensors (allocations), tensor rows
  twolevel+hot
gpt2m rich (f4: 2e9 16-byte records, grid window = all kernels, writes + bytes).
peer (S5 merge kernel pasta_peer_reduce at the llama shard size, g = 8 local sources;
134 MB of sources, so partly L2-resident across repetitions).

Times: the library's own CUDA events around the scan launch on its stream
(pasta_get_timing "scan" / "finalize"), averaged over --reps passes after --warmup.
Algorithmic bytes = 8 B (16 B rich) per record; peak = MEASURED_PEAKS.json hbm_gbs.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_22103_b200 as pb  # noqa: E402
import tracegen  # noqa: E402

DEV = torch.device("cuda:0")


def peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def timed(tr, fn, reps, warmup):
    for _ in range(warmup):
        fn()
    tr.sync()
    tr.reset_timing()
    tr.set_timing(True)
    for _ in range(reps):
        fn()
    tr.sync()
    ph, _ = tr.timing()
    tr.set_timing(False)
    return {k: v / reps for k, v in ph.items() if v}


def line(cfg, variant, n, bytes_per_rec, ph, pk, extra=None):
    ms = ph["scan"]
    gbs = bytes_per_rec * n / ms / 1e6
    d = {"config": cfg, "variant": variant, "n_records": n, "scan_ms": round(ms, 3),
         "finalize_ms": round(ph.get("finalize", 0.0), 3), "G_rec_s": round(n / ms / 1e6, 1),
         "algorithmic_GB_s": round(gbs, 1), "peak_GB_s": pk, "frac": round(gbs / pk, 4)}
    d.update(extra or {})
    print(json.dumps(d), flush=True)


def uvm(args, pk):
    p = tracegen.build_plan("uvm")
    dp = tracegen.DevicePlan(p, DEV)
    rec = torch.empty(p.n, dtype=torch.int64, device=DEV)
    tracegen.device_records(dp, rec)
    ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.uint64).view(np.int64).copy()).to(DEV)
    nk, wk = p.n_kernels, 20
    for variant in ("base", "hot", "twolevel", "twolevel+hot"):
        two = variant.startswith("twolevel")
        hot = variant.endswith("hot")
        objs = p.objects if two else p.allocs
        kw = dict(max_live_tensors=len(p.allocs), max_tensor_ids=len(p.allocs)) if two else {}
        tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(objs), len(objs), **kw)
        for b, s in objs:
            tr.register_alloc(b, s)
        if two:
            for b, s in p.allocs:
                tr.register_tensor(b, s)
        h = tr.histograms(p.page_shift, n_kernels=nk, kernel_rows=True, kernel_pages=p.want_kernel_pages,
                          window_kernels=wk if hot else 0)

        def run():
            h.zero_()
            tr.analyze(rec, p.page_shift, h, kernel_offsets=ko)
        ph = timed(tr, run, args.reps, args.warmup)
        extra = {"objects": len(objs), "tensors": len(p.allocs) if two else 0, "kernels": nk,
                 "blocks": h.P, "page_shift": p.page_shift}
        if hot:
            extra.update({"window_kernels": wk, "windows": h.n_windows})
        line("uvm", variant, p.n, 8, ph, pk, extra)
        tr.close()
        del h
    del rec
    torch.cuda.empty_cache()


def rich(args, pk):
    from tracegen.rich import rich_device

    p = tracegen.build_plan("gpt2m")
    n = p.n
    ko = torch.from_numpy(np.asarray(p.kernel_offsets, dtype=np.int64)).to(DEV)
    dp = tracegen.DevicePlan(p, DEV)
    for mix, blk in ((0.0, 0), (0.05, 5), (0.05, 0)):
        rec = torch.empty((n, 2), dtype=torch.int64, device=DEV)
        step = 1 << 27
        tmp = torch.empty(step, dtype=torch.int64, device=DEV)
        for j0 in range(0, n, step):
            j1 = min(n, j0 + step)
            tracegen.device_records(dp, tmp[:j1 - j0], j0, j1)
            rec[j0:j1] = rich_device(tmp[:j1 - j0], ko, seed=11, j0=j0, mix=mix, block_log2=blk)
        del tmp
        kmax = int(np.searchsorted(np.asarray(p.kernel_offsets, dtype=np.int64), n, side="left"))
        tr = pb.Trace(DEV, p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
        for b, s in p.allocs:
            tr.register_alloc(b, s)
        h = tr.histograms(p.page_shift, n_kernels=kmax + 1, kernel_rows=True)
        rx = tr.rich_outputs(p.page_shift)

        def run():
            tr.analyze_rich(rec, 0, kmax, p.page_shift, h, rx, finalize=False)
        ph = timed(tr, run, args.reps, args.warmup)
        line("gpt2m", f"rich mix={mix} burst=2^{blk}" if mix else "rich", n, 16, ph, pk,
             {"concurrent_kernel_fraction": mix, "burst_records": (1 << blk) if mix else 0})
        tr.close()
        del rec, h, rx
        torch.cuda.empty_cache()


def peer(args, pk):
    """S5 merge kernel (pasta_peer_reduce) at the llama shard size for g = 8: rank 0's
    shard of 2,097,152 pages from 8 sources, with bitmap words and popcount. The sources
    are local here (one GPU), so this measures the kernel against HBM, not NVLink."""
    g, S = 8, (1 << 24) // 8
    srcs = [torch.randint(0, 1 << 20, (S,), dtype=torch.int64, device=DEV) for _ in range(g)]
    out = torch.empty(S, dtype=torch.int64, device=DEV)
    bm = torch.empty(S // 64, dtype=torch.int64, device=DEV)
    pop = torch.zeros(1, dtype=torch.int64, device=DEV)
    tr = pb.Trace(DEV, 0, 1 << 32, 1, 1)
    ph = timed(tr, lambda: tr.peer_reduce(srcs, 0, S, out, bm, pop), args.reps * 20, args.warmup)
    ms = ph["merge"]
    byts = 8 * S * g + 8 * S + S // 8
    print(json.dumps({"config": "llama shard, g=8 (local sources)", "variant": "peer_reduce", "pages": S,
                      "merge_ms": round(ms, 4), "algorithmic_GB_s": round(byts / ms / 1e6, 1), "peak_GB_s": pk,
                      "frac": round(byts / ms / 1e6 / pk, 4)}), flush=True)
    tr.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--only", default="uvm,rich,peer")
    args = ap.parse_args()
    pk = peak()
    only = args.only.split(",")
    if "uvm" in only:
        uvm(args, pk)
    if "rich" in only:
        rich(args, pk)
    if "peer" in only:
        peer(args, pk)


if __name__ == "__main__":
    main()
