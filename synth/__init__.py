"""Seeded, counter-based synthetic inputs shared by the CUDA path's tests/bench
and the oracle's tests (see synth.h).  Holds none of the method's arithmetic.

host_fill(...)   -> numpy array, via libsynth_host.so (gcc)
device_fill(...) -> torch CUDA tensor, via libsynth_cuda.so (nvcc, sm_100a)

Both produce identical bits for identical (kind, seed, start, n, lo, hi), so a
shard [start, start+n) of a global array is the same on every GPU count.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

F32_U01, F64_U01, F32_S11, F64_S11, I32_RANGE, I64_RANGE, I64_FULL = range(7)
F32_RAMP, F64_RAMP, I32_RAMP, I64_RAMP = range(7, 11)

KIND_DTYPE = {
    F32_U01: np.float32, F64_U01: np.float64, F32_S11: np.float32, F64_S11: np.float64,
    I32_RANGE: np.int32, I64_RANGE: np.int64, I64_FULL: np.int64,
    F32_RAMP: np.float32, F64_RAMP: np.float64, I32_RAMP: np.int32, I64_RAMP: np.int64,
}

# Seeds: x = 1, y = 2, ints/scan = 3, max/min = 4.
SEED_X, SEED_Y, SEED_INT, SEED_MAXMIN = 1, 2, 3, 4

_host = None
_cuda = None


def _load(name):
    path = os.path.join(HERE, name)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `python __graft_entry__.py build` (or make -C synth)")
    return ctypes.CDLL(path)


def _host_lib():
    global _host
    if _host is None:
        lib = _load("libsynth_host.so")
        lib.synth_fill_host.restype = ctypes.c_int
        lib.synth_fill_host.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        _host = lib
    return _host


def _cuda_lib():
    global _cuda
    if _cuda is None:
        lib = _load("libsynth_cuda.so")
        lib.synth_fill_cuda.restype = ctypes.c_int
        lib.synth_fill_cuda.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _cuda = lib
    return _cuda


def host_fill(kind, seed, n, start=0, lo=0, hi=0, out=None):
    """Return (or fill `out` with) elements [start, start+n) of stream (kind, seed)."""
    dt = KIND_DTYPE[kind]
    if out is None:
        out = np.empty(n, dtype=dt)
    assert out.dtype == dt and out.flags.c_contiguous and out.size == n
    rc = _host_lib().synth_fill_host(kind, seed, start, n, lo, hi, out.ctypes.data if n else None)
    if rc != 0:
        raise ValueError(f"synth_fill_host rejected kind={kind} n={n} lo={lo} hi={hi}")
    return out


def device_fill(kind, seed, n, start=0, lo=0, hi=0, out=None, device=None):
    """Fill a CUDA tensor with elements [start, start+n) of stream (kind, seed)."""
    import torch
    tdt = {np.float32: torch.float32, np.float64: torch.float64,
           np.int32: torch.int32, np.int64: torch.int64}[KIND_DTYPE[kind]]
    if out is None:
        out = torch.empty(n, dtype=tdt, device=device or "cuda")
    assert out.dtype == tdt and out.is_cuda and out.is_contiguous() and out.numel() == n
    stream = torch.cuda.current_stream(out.device).cuda_stream
    rc = _cuda_lib().synth_fill_cuda(kind, seed, start, n, lo, hi, out.data_ptr() if n else None, stream)
    if rc != 0:
        raise RuntimeError(f"synth_fill_cuda failed rc={rc} kind={kind} n={n}")
    return out
