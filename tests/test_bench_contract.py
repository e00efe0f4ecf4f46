"""bench.py keeps the driver's JSON contract: the reference arm on CPU (the oracle on a
bounded sample; runs here), and our arm on the GPU at the tiny config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-sample", "65536"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["steps"] == 1 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "llama"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line_tiny():
    d = _run(["--config", "tiny", "--steps", "3", "--warmup", "3", "--cpu-sample", "65536", "--e2e-records",
              "1048576"])
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["dtype"] == "u64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and 0 < r["frac"] == pytest.approx(
        r["achieved"] / r["peak"])
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_two_rank_bench_on_one_gpu(tmp_path):
    """The N > 1 bench path (kernel-aligned shards, dist.PeerMerger through libpasta's
    CUDA IPC mappings, max-over-ranks timing, e2e with the same merge) as two processes
    on one GPU with a gloo group (PASTA_BENCH_GLOO=1; the driver's multi-GPU runs use
    NCCL), and EVERY merged output of both ranks (page shard, alloc counts, totals incl.
    unique pages / WS_obj / the MAX_MEM_REFERENCED_KERNEL pair, bitmap, top-K) equal to
    the oracle over the whole trace."""
    import socket

    import numpy as np

    import oracle
    import paper_2602_22103_b200 as pb
    import tracegen

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n = 300_000_000
    dump = str(tmp_path / "merged")
    env = dict(os.environ, PASTA_BENCH_GLOO="1", PASTA_BENCH_DUMP=dump)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "gpt2m",
           "--records", str(n), "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-records", "4194304"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["merge"] == "peer" and d["value"] > 0
    assert d["phases_ms_per_step"]["merge"] > 0 and d["e2e"]["value"] > 0

    p = tracegen.build_plan("gpt2m", 42, n)
    o = oracle.OracleTrace(p.va_lo, p.va_hi, len(p.allocs), len(p.allocs))
    for b, sz in p.allocs:
        o.register_alloc(b, sz)
    o.analyze_parallel(lambda j0, j1: tracegen.host_records(p, j0, j1), p.kernel_offsets, p.page_shift,
                       kernel_rows=True)
    bm, uniq = o.bitmap()
    _, ws = o.footprints()
    mk = o.max_kernel()
    per = o.kernel_rows.sum(axis=1, dtype=np.uint64) + o.kun
    A = len(p.allocs)
    for r in range(2):
        z = np.load(f"{dump}.rank{r}.npz")
        S = int(z["S"])
        pages = np.zeros(2 * S, dtype=np.uint64)
        pages[:len(o.page_counts)] = o.page_counts
        assert np.array_equal(z["shard"], pages[r * S:(r + 1) * S]), f"rank {r}: merged page shard"
        small = z["small"]
        assert np.array_equal(small[:A], o.alloc_counts), f"rank {r}: alloc counts"
        tot = small[A:A + pb.TOTALS]
        assert tot[:3].tolist() == o.totals.tolist(), f"rank {r}: records / unattributed / out of window"
        assert int(tot[pb.T_UNIQUE_PAGES]) == uniq, f"rank {r}: unique pages"
        assert int(tot[pb.T_WS_OBJ]) == ws, f"rank {r}: WS_obj"
        assert int(tot[pb.T_MAX_KERNEL]) == mk and int(tot[pb.T_MAX_KERNEL_RECORDS]) == int(per[mk]), \
            f"rank {r}: MAX_MEM_REFERENCED_KERNEL"
        assert np.array_equal(z["bitmap"], bm), f"rank {r}: bitmap"
        for k in p.topk:
            rp, rc, rf = oracle.topk(o.page_counts, k)
            assert int(z[f"top{k}_2"][0]) == rf, f"rank {r}: found top-{k}"
            assert np.array_equal(z[f"top{k}_0"], rp) and np.array_equal(z[f"top{k}_1"], rc), f"rank {r}: top-{k}"
