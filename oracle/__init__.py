"""Python face of the CPU oracle (oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product package
paper_1304_5553_b200 never imports it (tests/test_isolation.py checks).

Every function is a thin ctypes call into oracle.c, which cites the PAPER.md
passage it follows.  Inputs are numpy arrays; results are numpy arrays or
Python scalars.  Parity pins: tests/test_oracle.py.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

F32, F64, I32, I64 = 0, 1, 2, 3
SUM, MAX, MIN = 0, 1, 2
MAP_ID, MAP_MUL, MAP_SQUARE = 0, 1, 2
INCLUSIVE, EXCLUSIVE = 0, 1

_DT = {np.dtype(np.float32): F32, np.dtype(np.float64): F64,
       np.dtype(np.int32): I32, np.dtype(np.int64): I64}

CFLAGS = ["-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared"]


def build(force=False):
    """Compile oracle.c with gcc (no FMA contraction, no fast-math)."""
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, src, "-lm"])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        vp, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        f32 = ctypes.c_float
        for name, st in (("f32", f32), ("f64", d), ("i32", i32), ("i64", i64)):
            fn = getattr(L, f"oracle_axpbyz_{name}")
            fn.restype = None
            fn.argtypes = [i64, st, vp, st, vp, vp]
            fn = getattr(L, f"oracle_axpbz_{name}")
            fn.restype = None
            fn.argtypes = [i64, st, vp, st, vp]
        L.oracle_sum_f32.restype = d
        L.oracle_sum_f32.argtypes = [ctypes.c_int, i64, vp, vp, ctypes.POINTER(d)]
        L.oracle_sum_f64.restype = d
        L.oracle_sum_f64.argtypes = [ctypes.c_int, i64, vp, vp, ctypes.POINTER(d)]
        L.oracle_sum_int.restype = i64
        L.oracle_sum_int.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, vp, vp]
        L.oracle_maxmin_f32.restype = d
        L.oracle_maxmin_f32.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp]
        L.oracle_maxmin_f64.restype = d
        L.oracle_maxmin_f64.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp]
        L.oracle_maxmin_int.restype = i64
        L.oracle_maxmin_int.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, vp, vp]
        L.oracle_scan_i32.restype = None
        L.oracle_scan_i32.argtypes = [ctypes.c_int, i64, vp, vp, i32]
        L.oracle_scan_i64.restype = None
        L.oracle_scan_i64.argtypes = [ctypes.c_int, i64, vp, vp, i64]
        L.oracle_scan_maxmin_f32.restype = None
        L.oracle_scan_maxmin_f32.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, f32]
        L.oracle_scan_maxmin_f64.restype = None
        L.oracle_scan_maxmin_f64.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, d]
        L.oracle_scan_maxmin_int.restype = None
        L.oracle_scan_maxmin_int.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, vp, vp, i64]
        for nm in ("oracle_axpbyz_c64", "oracle_axpbyz_c128"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [i64, vp, vp, vp, vp, vp]
        L.oracle_sum_complex.restype = None
        L.oracle_sum_complex.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, vp, vp]
        L.oracle_norm2_complex.restype = d
        L.oracle_norm2_complex.argtypes = [ctypes.c_int, i64, vp]
        for nm in ("oracle_ewmap_f32", "oracle_ewmap_f64"):
            getattr(L, nm).restype = None
            getattr(L, nm).argtypes = [ctypes.c_int, i64, vp, vp, vp]
        L.oracle_ewmap_int.restype = None
        L.oracle_ewmap_int.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, vp]
        L.oracle_stencil3_f64.restype = None
        L.oracle_stencil3_f64.argtypes = [i64, d, d, d, vp, vp, vp]
        L.oracle_stencil3_f32.restype = None
        L.oracle_stencil3_f32.argtypes = [i64, f32, f32, f32, vp, vp, vp]
        L.oracle_scan_sum_float.restype = None
        L.oracle_scan_sum_float.argtypes = [ctypes.c_int, ctypes.c_int, i64, vp, vp, d, vp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def _c(a, dt=None):
    a = np.ascontiguousarray(a, dtype=dt)
    return a


def _name(dt):
    return {F32: "f32", F64: "f64", I32: "i32", I64: "i64"}[_DT[np.dtype(dt)]]


def axpbyz(a, x, b, y):
    """z = a*x + b*y elementwise; a, b are cast to x.dtype (R2)."""
    x = _c(x)
    y = _c(y, x.dtype)
    assert x.shape == y.shape and x.ndim == 1
    z = np.empty_like(x)
    st = x.dtype.type
    getattr(lib(), f"oracle_axpbyz_{_name(x.dtype)}")(x.size, st(a).item(), _ptr(x), st(b).item(), _ptr(y), _ptr(z))
    return z


def axpbz(a, x, b):
    """z = a*x + b elementwise (Listing 1/2 doubling is a=2, b=0)."""
    x = _c(x)
    z = np.empty_like(x)
    st = x.dtype.type
    getattr(lib(), f"oracle_axpbz_{_name(x.dtype)}")(x.size, st(a).item(), _ptr(x), st(b).item(), _ptr(z))
    return z


def reduce(op, map_, x, y=None, out_dtype=None, return_sumabs=False):
    """Map-reduce.  Float SUM returns a float64 near-exact
    value (Neumaier); integer SUM returns a Python int wrapped to out_dtype;
    MAX/MIN returns a value of the input dtype."""
    x = _c(x)
    if map_ == MAP_MUL:
        y = _c(y, x.dtype)
        assert y.shape == x.shape
    else:
        y = None
    in_dt = _DT[x.dtype]
    out_dt = _DT[np.dtype(out_dtype)] if out_dtype is not None else in_dt
    L = lib()
    n = x.size
    if op == SUM:
        if in_dt in (F32, F64):
            sa = ctypes.c_double(0.0)
            fn = L.oracle_sum_f32 if in_dt == F32 else L.oracle_sum_f64
            r = fn(map_, n, _ptr(x), _ptr(y), ctypes.byref(sa))
            return (r, sa.value) if return_sumabs else r
        r = int(L.oracle_sum_int(map_, in_dt, out_dt, n, _ptr(x), _ptr(y)))
        return (r, None) if return_sumabs else r
    if in_dt == F32:
        r = np.float32(L.oracle_maxmin_f32(op, map_, n, _ptr(x), _ptr(y)))
    elif in_dt == F64:
        r = np.float64(L.oracle_maxmin_f64(op, map_, n, _ptr(x), _ptr(y)))
    else:
        r = int(L.oracle_maxmin_int(op, map_, in_dt, n, _ptr(x), _ptr(y)))
    return (r, None) if return_sumabs else r


MAP_CONJ_MUL = 3


def axpbyz_complex(a, x, b, y):
    """z = a*x + b*y for complex64/complex128 (PAPER.md:385-394 + R24): the
    complex products written out component-wise, every operation RN, no FMA."""
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y, dtype=x.dtype)
    assert x.dtype in (np.complex64, np.complex128) and x.shape == y.shape and x.ndim == 1
    ct = x.dtype
    av = np.array([a], dtype=ct)
    bv = np.array([b], dtype=ct)
    z = np.empty_like(x)
    fn = lib().oracle_axpbyz_c64 if ct == np.complex64 else lib().oracle_axpbyz_c128
    fn(x.size, av.ctypes.data, _ptr(x), bv.ctypes.data, _ptr(y), _ptr(z))
    return z


def reduce_complex(map_, x, y=None, return_sumabs=False):
    """Complex sum (MAP_ID), dot (MAP_MUL: sum x*y), vdot (MAP_CONJ_MUL: sum
    conj(x)*y) as a near-exact complex128; MAP_SQUARE gives sum |x_i|^2 as a
    float64."""
    x = np.ascontiguousarray(x)
    is128 = int(x.dtype == np.complex128)
    if map_ == MAP_SQUARE:
        return lib().oracle_norm2_complex(is128, x.size, _ptr(x))
    if map_ != MAP_ID:
        y = np.ascontiguousarray(y, dtype=x.dtype)
    out = np.zeros(2)
    sa = ctypes.c_double(0.0)
    lib().oracle_sum_complex(map_, is128, x.size, _ptr(x), _ptr(y) if map_ != MAP_ID else None, out.ctypes.data,
                             ctypes.byref(sa))
    r = complex(out[0], out[1])
    return (r, sa.value) if return_sumabs else r


NEUTRAL = {
    (MAX, np.dtype(np.float32)): -np.inf, (MIN, np.dtype(np.float32)): np.inf,
    (MAX, np.dtype(np.float64)): -np.inf, (MIN, np.dtype(np.float64)): np.inf,
    (MAX, np.dtype(np.int32)): np.iinfo(np.int32).min, (MIN, np.dtype(np.int32)): np.iinfo(np.int32).max,
    (MAX, np.dtype(np.int64)): np.iinfo(np.int64).min, (MIN, np.dtype(np.int64)): np.iinfo(np.int64).max,
}


def scan(kind, x, carry=None, out=None, op=SUM, return_sumabs=False, out_dtype=None):
    """Scan with reduction expression `op`; the exclusive
    head / inclusive start is `carry` (default: the neutral element, R13).
    Integer SUM wraps in the element type; float SUM returns the exact prefix
    sums as float64 (and, with return_sumabs, |c| + sum |x_j| per position);
    MAX / MIN fold with maxNum/minNum and return the element type.
    out_dtype widens first (int32 -> int64, float32 -> float64: the result
    dtype is a parameter): the scan of the exactly converted
    elements, i.e. the scan run in the wide type (R27)."""
    x = _c(x)
    if out_dtype is not None and np.dtype(out_dtype) != x.dtype:
        if (x.dtype, np.dtype(out_dtype)) not in ((np.dtype(np.int32), np.dtype(np.int64)),
                                                  (np.dtype(np.float32), np.dtype(np.float64))):
            raise TypeError(f"no widening scan {x.dtype} -> {np.dtype(out_dtype)}")
        x = x.astype(out_dtype)  # exact conversion
    L = lib()
    if op == SUM and x.dtype.kind == "f":
        res = np.empty(x.size, np.float64)
        sa = np.empty(x.size, np.float64) if return_sumabs else None
        L.oracle_scan_sum_float(kind, _DT[x.dtype], x.size, _ptr(x), _ptr(res), float(carry or 0.0), _ptr(sa))
        return (res, sa) if return_sumabs else res
    if out is None:
        out = np.empty_like(x)
    if op == SUM:
        fn = {np.dtype(np.int32): L.oracle_scan_i32, np.dtype(np.int64): L.oracle_scan_i64}[x.dtype]
        fn(kind, x.size, _ptr(x), _ptr(out), int(np.array(carry or 0).astype(x.dtype)))
        return out
    c = NEUTRAL[(op, x.dtype)] if carry is None else carry
    if x.dtype == np.float32:
        L.oracle_scan_maxmin_f32(op, kind, x.size, _ptr(x), _ptr(out), float(c))
    elif x.dtype == np.float64:
        L.oracle_scan_maxmin_f64(op, kind, x.size, _ptr(x), _ptr(out), float(c))
    else:
        L.oracle_scan_maxmin_int(op, kind, _DT[x.dtype], x.size, _ptr(x), _ptr(out), int(c))
    return out


def stencil3(l, d, u, x, diag=None):
    """y_i = l*x_{i-1} + d_i*x_i + u*x_{i+1}, boundary terms omitted, each
    step RN left to right (R25); d_i = diag[i] when diag is given."""
    x = _c(x)
    y = np.empty_like(x)
    if diag is not None:
        diag = _c(diag, x.dtype)
    st = x.dtype.type
    fn = lib().oracle_stencil3_f64 if x.dtype == np.float64 else lib().oracle_stencil3_f32
    fn(x.size, st(l).item(), st(d).item(), st(u).item(), _ptr(diag) if diag is not None else None, _ptr(x), _ptr(y))
    return y


EW_MUL, EW_DIV, EW_SQRT, EW_ABS, EW_NEG, EW_EXP, EW_LOG, EW_SIN, EW_COS, EW_MAX, EW_MIN = range(11)
EW_BINARY = (EW_MUL, EW_DIV, EW_MAX, EW_MIN)


def ewmap(op, x, y=None):
    """z = op(x[, y]) elementwise (R26)."""
    x = _c(x)
    if op in EW_BINARY:
        y = _c(y, x.dtype)
        assert y.shape == x.shape
    else:
        y = None
    z = np.empty_like(x)
    L = lib()
    if x.dtype == np.float32:
        L.oracle_ewmap_f32(op, x.size, _ptr(x), _ptr(y), _ptr(z))
    elif x.dtype == np.float64:
        L.oracle_ewmap_f64(op, x.size, _ptr(x), _ptr(y), _ptr(z))
    else:
        L.oracle_ewmap_int(op, _DT[x.dtype], x.size, _ptr(x), _ptr(y), _ptr(z))
    return z
