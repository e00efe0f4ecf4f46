"""Rich 16-byte records (NEXT f4) from a plan's 8-byte address records.

Layout (SPEC S:39-42 MemAccessInfo; include/pasta.h pasta_rich_record): u64 address,
u32 grid_id, u16 size_bytes, u8 flags (bit 0 is_write, bit 1 shared space), u8 zero.
Input infrastructure only (no analysis arithmetic). Record j of kernel segment k gets,
from h = splitmix64(seed + j):

* grid_id = grid_base + k, except with probability ``mix`` grid_base + k - 1 when
  k > 0: kernels overlapping in time (concurrent streams), so grid ids are not sorted
  within a slice. The draw is made per block of 2^block_log2 records (from
  hb = splitmix64(seed + (j >> block_log2)): hb & 0xFFFF < mix * 2^16), so 0 mixes
  single records and 5 mixes warp-sized bursts;
* size_bytes = 1 << ((h >> 16) & 7) (1 .. 128);
* is_write iff ((h >> 24) & 3) == 0 (25 %);
* shared space iff ((h >> 32) & 127) == 0 (1/128).

Two implementations: ``rich_host`` (numpy) and ``rich_device`` (torch ops on the
device), cross-checked in tests/test_gpu_rich.py.
"""
from __future__ import annotations

import numpy as np

RICH_DTYPE = np.dtype([("addr", "<u8"), ("grid", "<u4"), ("size", "<u2"), ("flags", "u1"), ("pad", "u1")])
assert RICH_DTYPE.itemsize == 16

_C1, _C2, _C3 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _splitmix_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(_C1)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C2)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C3)
        return z ^ (z >> np.uint64(31))


def rich_host(addr: np.ndarray, kernel_offsets, seed: int, grid_base: int = 0, mix: float = 0.05,
              j0: int = 0, block_log2: int = 0) -> np.ndarray:
    """addr: records j0 .. j0 + n - 1; kernel_offsets: global offsets."""
    addr = np.ascontiguousarray(addr, dtype=np.uint64)
    n = addr.size
    ko = np.asarray(kernel_offsets, dtype=np.int64)
    jj = np.arange(j0, j0 + n, dtype=np.int64)
    j = jj.astype(np.uint64)
    k = np.searchsorted(ko, jj, side="right") - 1
    h = _splitmix_np(j + np.uint64(seed))
    hb = _splitmix_np((j >> np.uint64(block_log2)) + np.uint64(seed))
    thr = np.uint64(int(mix * 65536))
    prev = ((hb & np.uint64(0xFFFF)) < thr) & (k > 0)
    out = np.zeros(n, dtype=RICH_DTYPE)
    out["addr"] = addr
    out["grid"] = (grid_base + k - prev.astype(np.int64)).astype(np.uint32)
    out["size"] = (np.uint64(1) << ((h >> np.uint64(16)) & np.uint64(7))).astype(np.uint16)
    wr = ((h >> np.uint64(24)) & np.uint64(3)) == 0
    sh = ((h >> np.uint64(32)) & np.uint64(127)) == 0
    out["flags"] = wr.astype(np.uint8) | (sh.astype(np.uint8) << 1)
    return out


def _srl(x, s: int):
    """Logical right shift of int64 tensors holding u64 bit patterns."""
    import torch

    return torch.bitwise_and(torch.bitwise_right_shift(x, s), (1 << (64 - s)) - 1)


def _wrap(c: int) -> int:
    return c - (1 << 64) if c >= 1 << 63 else c


def _splitmix_t(x, seed: int):
    z = x + _wrap((seed + _C1) & ((1 << 64) - 1))
    z = (z ^ _srl(z, 30)) * _wrap(_C2)
    z = (z ^ _srl(z, 27)) * _wrap(_C3)
    return z ^ _srl(z, 31)


def rich_device(addr, kernel_offsets, seed: int, grid_base: int = 0, mix: float = 0.05, j0: int = 0,
                block_log2: int = 0):
    """addr: int64 CUDA tensor; kernel_offsets: int64 CUDA tensor (global offsets);
    records are global indices j0 .. j0 + n - 1. Returns an int64 tensor [n, 2] whose
    bytes are the RICH_DTYPE records."""
    import torch

    n = addr.numel()
    dev = addr.device
    j = torch.arange(j0, j0 + n, dtype=torch.int64, device=dev)
    k = torch.searchsorted(kernel_offsets, j, right=True) - 1
    h = _splitmix_t(j, seed)
    hb = _splitmix_t(_srl(j, block_log2) if block_log2 else j, seed)
    thr = int(mix * 65536)
    prev = ((hb & 0xFFFF) < thr) & (k > 0)
    grid = grid_base + k - prev.to(torch.int64)
    size = torch.bitwise_left_shift(torch.ones_like(h), _srl(h, 16) & 7)
    wr = (_srl(h, 24) & 3) == 0
    sh = (_srl(h, 32) & 127) == 0
    flags = wr.to(torch.int64) | (sh.to(torch.int64) << 1)
    out = torch.empty((n, 2), dtype=torch.int64, device=dev)
    out[:, 0] = addr
    out[:, 1] = (grid & 0xFFFFFFFF) | (size << 32) | (flags << 48)
    return out
