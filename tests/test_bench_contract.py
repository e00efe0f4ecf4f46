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
def test_two_rank_bench_on_one_gpu():
    """The N > 1 bench path (kernel-aligned shards, dist.PeerMerger through CUDA IPC,
    max-over-ranks timing, e2e with the same merge) as two processes on one GPU with a
    gloo group (PASTA_BENCH_GLOO=1; the driver's multi-GPU runs use NCCL)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, PASTA_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "gpt2m",
           "--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-records", "4194304"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["merge"] == "peer" and d["value"] > 0
    assert d["phases_ms_per_step"]["merge"] > 0 and d["e2e"]["value"] > 0
