"""GPUArray operations on torch CUDA tensors (§3.2.1).

torch supplies device memory and the stream (plumbing); every operation is
one call through the C ABI (include/gpuarray.h) into an sm_100a kernel:

    axpbyz(a, x, b, y)    z = a*x + b*y        ElementwiseKernel
    axpbz(a, x, b)        z = a*x + b          (Listing 1 doubling: a=2, b=-0.0)
    reduce(op, map, x, y) map-then-reduce       ReductionKernel
    dot / sum / norm2sq / max / min             instances of reduce
    scan(x, exclusive)    prefix sum

Reductions return a 0-d tensor that stays on the GPU ("a GPUArray scalar
still residing on the GPU"); `.item()` is the `.get()`.
All calls are asynchronous on torch's current stream.
Errors raise: ValueError for shapes/arguments, TypeError
for dtypes, RuntimeError for CUDA failures.
"""
import builtins

import torch

from . import _abi
from ._abi import (GA_C64, GA_C128, GA_F32, GA_F64, GA_I32, GA_I64, GA_MAP_CONJ_MUL, GA_MAP_ID, GA_MAP_MUL,
                   GA_MAP_SQUARE, GA_OP_MAX, GA_OP_MIN, GA_OP_SUM, GA_SCAN_EXCLUSIVE, GA_SCAN_INCLUSIVE, check,
                   make_scalar)

SUM, MAX, MIN = GA_OP_SUM, GA_OP_MAX, GA_OP_MIN
ID, MUL, SQUARE, CONJ_MUL = GA_MAP_ID, GA_MAP_MUL, GA_MAP_SQUARE, GA_MAP_CONJ_MUL

_DT = {torch.float32: GA_F32, torch.float64: GA_F64, torch.int32: GA_I32, torch.int64: GA_I64,
       torch.complex64: GA_C64, torch.complex128: GA_C128}
_REAL_OF = {torch.complex64: torch.float32, torch.complex128: torch.float64}


def ga_dtype(t):
    try:
        return _DT[t]
    except KeyError:
        raise TypeError(f"unsupported dtype {t}; expected float32/float64/int32/int64/complex64/complex128") from None


def _check_array(name, t):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dim() != 1:
        raise ValueError(f"{name} must be 1-D (got shape {tuple(t.shape)})")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    ga_dtype(t.dtype)


def _same(x, other, name):
    _check_array(name, other)
    if other.shape != x.shape:  # "All these instances are required to have the same length" PAPER.md:457-458
        raise ValueError(f"{name} has length {other.numel()}, x has {x.numel()}")
    if other.dtype != x.dtype:
        raise TypeError(f"{name} has dtype {other.dtype}, x has {x.dtype}")
    if other.device != x.device:
        raise ValueError(f"{name} is on {other.device}, x on {x.device}")


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(t):
    """torch's current stream on t's device as a cudaStream_t (int)."""
    if _raw_stream is not None:  # no Stream object per call (~µs of host time)
        return _raw_stream(t.device.index)
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t):
    return t.data_ptr() if t.numel() else None


# --------------------------------------------------------------- workspaces
# One zero-filled workspace per (kernel family, device, stream); the kernels
# keep it valid across calls (epoch-tagged reduce slots / epoch-tagged scan
# status), so it is zeroed at allocation and then only when its epoch could
# wrap: the scan epoch has 30 bits and the reduce tag 31, so a workspace is
# re-zeroed (on the call's stream, stream-ordered) every WRAP_CALLS calls,
# long before a stale word could match a recycled epoch.  Reduce and scan
# workspaces have different layouts and are never shared; scan workspaces are
# also kept apart by element size (the status layout is tagged word by word
# for every size, so sharing would be correct too — tests/
# test_scan_workspace_gpu.py shares one on purpose).
WRAP_CALLS = 1 << 29
_ws = {}


def workspace(kind, device, stream, nbytes):
    key = (kind, device.index, stream)
    e = _ws.get(key)
    if e is None or e[0].numel() < nbytes:
        size = builtins.max(nbytes, 1 << 16)
        if e is not None:
            size = builtins.max(size, 2 * e[0].numel())
        e = [torch.zeros(size, dtype=torch.uint8, device=device), 0]
        _ws[key] = e
    e[1] += 1
    if e[1] >= WRAP_CALLS:
        e[0].zero_()  # torch's current stream on this device == the call's stream
        e[1] = 1
    return e[0]


# --------------------------------------------------------------- elementwise
def axpbyz(a, x, b, y, out=None):
    """z = a*x + b*y in one pass; floats round as RN(RN(a*x)+RN(b*y)) (R1).
    a and b are converted to x's dtype first (numpy-sized scalars, R2)."""
    _check_array("x", x)
    _same(x, y, "y")
    if out is None:
        out = torch.empty_like(x)
    else:
        _same(x, out, "out")
    dt = ga_dtype(x.dtype)
    check(_abi.gpuarray_axpbyz(dt, x.numel(), make_scalar(dt, a), _ptr(x), make_scalar(dt, b), _ptr(y), _ptr(out),
                               _stream(x)))
    return out


def axpbyz_ds(a, x, b, y, out=None, a_num=None, a_den=None, b_num=None, b_den=None):
    """axpbyz whose coefficients may carry device-resident factors: the
    effective a is RN(a * RN(a_num / a_den)) (missing tensor = 1), read when
    the kernel runs (float32/float64; the factors are 1-element tensors of
    x's dtype, e.g. reduction results left on the GPU)."""
    _check_array("x", x)
    _same(x, y, "y")
    if out is None:
        out = torch.empty_like(x)
    else:
        _same(x, out, "out")
    dt = ga_dtype(x.dtype)

    def ptr(t):
        if t is None:
            return None
        if t.numel() != 1 or t.dtype != x.dtype or t.device != x.device:
            raise ValueError("device scalar factors must be 1-element tensors of x's dtype and device")
        return t.data_ptr()
    check(_abi.gpuarray_axpbyz_ds(dt, x.numel(), _abi.make_dscalar(dt, a, ptr(a_num), ptr(a_den)), _ptr(x),
                                  _abi.make_dscalar(dt, b, ptr(b_num), ptr(b_den)), _ptr(y), _ptr(out), _stream(x)))
    return out


def axpbz(a, x, b, out=None):
    """z = a*x + b in one pass (RN(RN(a*x)+b))."""
    _check_array("x", x)
    if out is None:
        out = torch.empty_like(x)
    else:
        _same(x, out, "out")
    dt = ga_dtype(x.dtype)
    check(_abi.gpuarray_axpbz(dt, x.numel(), make_scalar(dt, a), _ptr(x), make_scalar(dt, b), _ptr(out),
                              _stream(x)))
    return out


def stencil3(l, d, u, x, diag=None, out=None):
    """y[i] = l*x[i-1] + d_i*x[i] + u*x[i+1] (boundary terms omitted, every
    step RN, R25); d_i = diag[i] when a diagonal array is given.  The
    operator of the CG workload."""
    _check_array("x", x)
    if out is None:
        out = torch.empty_like(x)
    else:
        _same(x, out, "out")
    if diag is not None:
        _same(x, diag, "diag")
    dt = ga_dtype(x.dtype)
    check(_abi.gpuarray_stencil3(dt, x.numel(), make_scalar(dt, l), make_scalar(dt, d), make_scalar(dt, u),
                                 _ptr(diag) if diag is not None else None, _ptr(x), _ptr(out), _stream(x)))
    return out


# --------------------------------------------------------------- fused CG steps (NEXT-4)
def _dfactor(t, x, name):
    if t is None:
        return None
    if t.numel() != 1 or t.dtype != x.dtype or t.device != x.device:
        raise ValueError(f"{name} must be a 1-element tensor of x's dtype and device")
    return t.data_ptr()


def _scalar_out(out, x):
    if out is None:
        return torch.empty((), dtype=x.dtype, device=x.device)
    if out.numel() != 1 or out.dtype != x.dtype or out.device != x.device:
        raise ValueError("out must be a 1-element tensor of x's dtype on x's device")
    return out


def cg_direction(r, p_in, p_out, ap, beta=1.0, beta_num=None, beta_den=None, l=-1.0, d=2.0, u=-1.0, diag=None,
                 out=None):
    """One kernel: p_out = r + beta p_in, ap = A p_out (A = tridiag(l, d_i, u)),
    returns p_out . ap as a 0-d device tensor.  beta is RN(beta *
    RN(beta_num / beta_den)) with device factors (gpuarray_cg_direction)."""
    _check_array("r", r)
    for name, t in (("p_in", p_in), ("p_out", p_out), ("ap", ap)):
        _same(r, t, name)
    if diag is not None:
        _same(r, diag, "diag")
    out = _scalar_out(out, r)
    dt = ga_dtype(r.dtype)
    s = _stream(r)
    nb = _abi.gpuarray_reduce_workspace_bytes(dt, r.numel())
    w = workspace("reduce", r.device, s, nb)
    check(_abi.gpuarray_cg_direction(dt, r.numel(), _abi.make_dscalar(dt, beta, _dfactor(beta_num, r, "beta_num"),
                                                                      _dfactor(beta_den, r, "beta_den")),
                                     _ptr(r), _ptr(p_in), _ptr(p_out), make_scalar(dt, l), make_scalar(dt, d),
                                     make_scalar(dt, u), _ptr(diag) if diag is not None else None, _ptr(ap),
                                     out.data_ptr(), w.data_ptr(), w.numel(), s))
    return out


def cg_update(x, r, p, ap, alpha=1.0, alpha_num=None, alpha_den=None, out=None):
    """One kernel: x += alpha p, r -= alpha ap (in place), returns r . r of
    the updated r as a 0-d device tensor (gpuarray_cg_update)."""
    _check_array("x", x)
    for name, t in (("r", r), ("p", p), ("ap", ap)):
        _same(x, t, name)
    out = _scalar_out(out, x)
    dt = ga_dtype(x.dtype)
    s = _stream(x)
    nb = _abi.gpuarray_reduce_workspace_bytes(dt, x.numel())
    w = workspace("reduce", x.device, s, nb)
    check(_abi.gpuarray_cg_update(dt, x.numel(), _abi.make_dscalar(dt, alpha, _dfactor(alpha_num, x, "alpha_num"),
                                                                   _dfactor(alpha_den, x, "alpha_den")),
                                  _ptr(x), _ptr(r), _ptr(p), _ptr(ap), out.data_ptr(), w.data_ptr(), w.numel(), s))
    return out


# --------------------------------------------------------------- operators / cumath
_BINARY = (_abi.GA_EW_MUL, _abi.GA_EW_DIV, _abi.GA_EW_MAX, _abi.GA_EW_MIN)


def elementwise(op, x, y=None, out=None):
    """z = op(x[, y]) in one pass (gpuarray_elementwise)."""
    _check_array("x", x)
    if op in _BINARY:
        if y is None:
            raise ValueError("binary operator needs y")
        _same(x, y, "y")
    if out is None:
        out = torch.empty_like(x)
    else:
        _same(x, out, "out")
    check(_abi.gpuarray_elementwise(op, ga_dtype(x.dtype), x.numel(), _ptr(x), _ptr(y) if op in _BINARY else None,
                                    _ptr(out), _stream(x)))
    return out


def multiply(x, y, out=None):
    return elementwise(_abi.GA_EW_MUL, x, y, out)


def divide(x, y, out=None):
    return elementwise(_abi.GA_EW_DIV, x, y, out)


def maximum(x, y, out=None):
    return elementwise(_abi.GA_EW_MAX, x, y, out)


def minimum(x, y, out=None):
    return elementwise(_abi.GA_EW_MIN, x, y, out)


def sqrt(x, out=None):
    return elementwise(_abi.GA_EW_SQRT, x, None, out)


def fabs(x, out=None):
    return elementwise(_abi.GA_EW_ABS, x, None, out)


def negative(x, out=None):
    return elementwise(_abi.GA_EW_NEG, x, None, out)


def exp(x, out=None):
    return elementwise(_abi.GA_EW_EXP, x, None, out)


def log(x, out=None):
    return elementwise(_abi.GA_EW_LOG, x, None, out)


def sin(x, out=None):
    return elementwise(_abi.GA_EW_SIN, x, None, out)


def cos(x, out=None):
    return elementwise(_abi.GA_EW_COS, x, None, out)


# --------------------------------------------------------------- map-reduce
def reduce(op, map_, x, y=None, out_dtype=None, out=None, nccl_comm=None):
    """Fold map(x, y) with op from its neutral element; returns a 0-d device
    tensor of out_dtype (default: x.dtype).  With `nccl_comm` (an ncclComm_t
    as an int), x is this rank's shard and the result is the fold over every
    rank's shard (gpuarray_reduce_sharded: local kernel + one NCCL
    allreduce on the current stream)."""
    _check_array("x", x)
    has_y = map_ in (MUL, CONJ_MUL)
    if has_y:
        if y is None:
            raise ValueError("maps MUL / CONJ_MUL need y")
        _same(x, y, "y")
    if out_dtype is None:  # |x|^2 of complex data is real
        out_dtype = _REAL_OF.get(x.dtype, x.dtype) if map_ == SQUARE else x.dtype
    if out is None:
        out = torch.empty((), dtype=out_dtype, device=x.device)
    elif out.numel() != 1 or out.dtype != out_dtype or out.device != x.device:
        raise ValueError("out must be a 1-element tensor of out_dtype on x's device")
    in_dt, out_dt = ga_dtype(x.dtype), ga_dtype(out_dtype)
    s = _stream(x)
    nb = _abi.gpuarray_reduce_workspace_bytes(out_dt, x.numel())
    w = workspace("reduce", x.device, s, nb)
    if nccl_comm is not None:
        check(_abi.gpuarray_reduce_sharded(op, map_, in_dt, out_dt, x.numel(), _ptr(x), _ptr(y) if has_y else None,
                                           out.data_ptr(), w.data_ptr(), w.numel(), nccl_comm, s))
        return out
    check(_abi.gpuarray_reduce(op, map_, in_dt, out_dt, x.numel(), _ptr(x), _ptr(y) if has_y else None,
                               out.data_ptr(), w.data_ptr(), w.numel(), s))
    return out


def dot(x, y, out_dtype=None, out=None):
    """Listing 3b: map x[i]*y[i], reduce a+b, neutral 0."""
    return reduce(SUM, MUL, x, y, out_dtype=out_dtype, out=out)


def vdot(x, y, out=None):
    """sum conj(x[i]) * y[i] (equal to dot for real data)."""
    return reduce(SUM, CONJ_MUL, x, y, out=out)


def sum(x, out_dtype=None, out=None):  # noqa: A001 - numpy-patterned name
    return reduce(SUM, ID, x, out_dtype=out_dtype, out=out)


def norm2sq(x, out_dtype=None, out=None):
    """Squared 2-norm: map x[i]*x[i] (|x[i]|^2 for complex, into the real
    type), reduce a+b (x is read once)."""
    return reduce(SUM, SQUARE, x, out_dtype=out_dtype, out=out)


def max(x, out=None):  # noqa: A001
    return reduce(MAX, ID, x, out=out)


def min(x, out=None):  # noqa: A001
    return reduce(MIN, ID, x, out=out)


# --------------------------------------------------------------- scan
def scan(x, exclusive=False, out=None, carry=None, op=SUM, out_dtype=None, nccl_comm=None):
    """Scan with reduction expression `op` (SUM / MAX / MIN) over int32,
    int64 (wrapping), float32, float64.  `out_dtype`
    (default x.dtype) may widen int32 -> int64 or float32 -> float64: the
    scan then runs in the wide type (NEXT-2).  `carry` is an optional 1-D
    device tensor of out_dtype whose elements are all folded in front (a
    sharded scan's offset).  With `nccl_comm` (an ncclComm_t as an int), x is
    this rank's shard and out its part of the scan of the global array
    (gpuarray_scan_sharded: local reduce, NCCL allgather of the shard
    totals, local scan with their prefix as carry-in)."""
    _check_array("x", x)
    out_dtype = x.dtype if out_dtype is None else out_dtype
    if out is None:
        out = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    else:
        _check_array("out", out)
        if out.shape != x.shape:
            raise ValueError(f"out has length {out.numel()}, x has {x.numel()}")
        if out.dtype != out_dtype or out.device != x.device:
            raise TypeError(f"out must be a {out_dtype} tensor on {x.device}")
    in_dt, dt = ga_dtype(x.dtype), ga_dtype(out_dtype)
    if carry is not None:
        _check_array("carry", carry)
        if carry.dtype != out_dtype or carry.device != x.device:
            raise TypeError("carry must match out_dtype and x's device")
        cptr, ccount = _ptr(carry), carry.numel()
    else:
        cptr, ccount = None, 0
    s = _stream(x)
    kind = GA_SCAN_EXCLUSIVE if exclusive else GA_SCAN_INCLUSIVE
    esize = x.element_size() if out_dtype == x.dtype else 8
    if nccl_comm is not None:
        nb = _abi.gpuarray_scan_sharded_workspace_bytes(dt, x.numel())
        w = workspace(f"scan_sharded{esize}", x.device, s, nb)
        check(_abi.gpuarray_scan_sharded(op, kind, in_dt, dt, x.numel(), _ptr(x), _ptr(out), cptr, ccount,
                                         w.data_ptr(), w.numel(), nccl_comm, s))
        return out
    nb = _abi.gpuarray_scan_workspace_bytes(dt, x.numel())
    w = workspace(f"scan{esize}", x.device, s, nb)
    check(_abi.gpuarray_scan(op, kind, in_dt, dt, x.numel(), _ptr(x), _ptr(out), cptr, ccount, w.data_ptr(),
                             w.numel(), s))
    return out


def launch_count():
    """Kernels launched by libgpuarray.so in this process."""
    return _abi.gpuarray_launch_count()
