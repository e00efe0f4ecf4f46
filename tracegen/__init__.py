"""tracegen -- seeded synthetic trace generator (test/bench input infrastructure).

Shared by the oracle side and the CUDA side of the parity contract, from a module of
its own that holds none of the analysis method's arithmetic. Two independent
implementations of tracegen/GENERATOR.md: ``host_records`` (C, libtracegen_host.so)
and ``device_records`` (CUDA, libtracegen_dev.so).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .plan import CONFIGS, Plan, build_plan, splitmix64  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_host = None
_dev = None


def _load_host():
    global _host
    if _host is None:
        path = os.path.join(_HERE, "libtracegen_host.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.tracegen_host.restype = ctypes.c_int
        lib.tracegen_host.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_void_p]
        lib.tracegen_splitmix64.restype = ctypes.c_uint64
        lib.tracegen_splitmix64.argtypes = [ctypes.c_uint64]
        _host = lib
    return _host


def _load_dev():
    global _dev
    if _dev is None:
        path = os.path.join(_HERE, "libtracegen_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.tracegen_device.restype = ctypes.c_int
        lib.tracegen_device.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        _dev = lib
    return _dev


def host_records(plan: Plan, j0: int = 0, j1: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Records j0..j1-1 of ``plan`` generated on the host (C implementation)."""
    if j1 is None:
        j1 = plan.n
    lib = _load_host()
    st = np.ascontiguousarray(plan.streams, dtype=np.uint64)
    cdf = np.ascontiguousarray(plan.cdf, dtype=np.uint64)
    if out is None:
        out = np.empty(j1 - j0, dtype=np.uint64)
    assert out.dtype == np.uint64 and out.flags.c_contiguous and out.size >= j1 - j0
    rc = lib.tracegen_host(st.ctypes.data, st.shape[0], cdf.ctypes.data, j0, j1, out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"tracegen_host failed ({rc})")
    return out[: j1 - j0]


class DevicePlan:
    """Plan tables resident on a CUDA device (torch tensors own the memory)."""

    def __init__(self, plan: Plan, device):
        import torch

        self.plan = plan
        self.streams = torch.from_numpy(plan.streams.view(np.int64).copy()).to(device)
        self.cdf = torch.from_numpy(plan.cdf.view(np.int64).copy()).to(device)


def device_records(dplan: DevicePlan, out, j0: int = 0, j1: int | None = None, stream=None):
    """Write records j0..j1-1 into the int64/uint64 CUDA tensor ``out`` (CUDA
    implementation), asynchronously on ``stream`` (default: torch current stream)."""
    import torch

    if j1 is None:
        j1 = dplan.plan.n
    assert out.is_cuda and out.element_size() == 8 and out.is_contiguous() and out.numel() >= j1 - j0
    if stream is None:
        stream = torch.cuda.current_stream(out.device)
    lib = _load_dev()
    rc = lib.tracegen_device(dplan.streams.data_ptr(), dplan.streams.shape[0], dplan.cdf.data_ptr(), j0, j1,
                             out.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"tracegen_device failed ({rc})")
    return out
