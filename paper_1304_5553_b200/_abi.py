"""Thin ctypes binding of include/gpuarray.h — argument marshalling only.

Every function here has the name and argument order of its C entry point and
passes raw device pointers, sizes and the CUDA stream handle straight
through; all compute happens in libgpuarray.so's sm_100a kernels.  There is
no fallback: if the library is missing, importing this module raises.
"""
import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libgpuarray.so")

GA_F32, GA_F64, GA_I32, GA_I64, GA_C64, GA_C128 = 0, 1, 2, 3, 4, 5
GA_OP_SUM, GA_OP_MAX, GA_OP_MIN = 0, 1, 2
GA_MAP_ID, GA_MAP_MUL, GA_MAP_SQUARE, GA_MAP_CONJ_MUL = 0, 1, 2, 3
GA_SCAN_INCLUSIVE, GA_SCAN_EXCLUSIVE = 0, 1
GA_OK, GA_ERR_INVALID_ARGUMENT, GA_ERR_UNSUPPORTED, GA_ERR_WORKSPACE, GA_ERR_CUDA, GA_ERR_NCCL = 0, 1, 2, 3, 4, 5

# Every symbol include/gpuarray.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "gpuarray_axpbyz", "gpuarray_axpbz", "gpuarray_reduce_workspace_bytes", "gpuarray_reduce",
    "gpuarray_scan_workspace_bytes", "gpuarray_scan", "gpuarray_status_string", "gpuarray_last_error",
    "gpuarray_abi_version", "gpuarray_launch_count", "gpuarray_xgpu_buffer_bytes", "gpuarray_reduce_xgpu",
    "gpuarray_stencil3", "gpuarray_axpbyz_ds", "gpuarray_elementwise", "gpuarray_cg_direction",
    "gpuarray_cg_update", "gpuarray_reduce_sharded", "gpuarray_scan_sharded_workspace_bytes",
    "gpuarray_scan_sharded",
)


class ga_scalar_t(ctypes.Structure):
    """Layout-identical to the C struct: {int32 dtype; int32 reserved; union v}
    (24 bytes).  The 16-byte union is carried as two raw 8-byte words
    (little-endian: a 4-byte member sits in the low half of `bits`) because
    ctypes cannot pass unions by value portably."""
    _fields_ = [("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32), ("bits", ctypes.c_uint64),
                ("bits_hi", ctypes.c_uint64)]


class ga_dscalar_t(ctypes.Structure):
    """{ga_scalar_t scale; const void *num; const void *den} (40 bytes)."""
    _fields_ = [("scale", ga_scalar_t), ("num", ctypes.c_void_p), ("den", ctypes.c_void_p)]


def make_dscalar(dt, scale, num=None, den=None):
    d = ga_dscalar_t()
    d.scale = make_scalar(dt, scale)
    d.num = num
    d.den = den
    return d


def make_scalar(dt, value):
    """ga_scalar_t holding `value` converted to dtype `dt` (RN for floats, R2)."""
    import struct
    if dt == GA_F32:
        raw = struct.pack("<f", float(value)) + b"\0\0\0\0"  # struct rounds to nearest float32
    elif dt == GA_F64:
        raw = struct.pack("<d", float(value))
    elif dt == GA_I32:
        raw = struct.pack("<i", ((int(value) + (1 << 31)) % (1 << 32)) - (1 << 31)) + b"\0\0\0\0"
    elif dt == GA_I64:
        raw = struct.pack("<q", ((int(value) + (1 << 63)) % (1 << 64)) - (1 << 63))
    elif dt == GA_C64:
        c = complex(value)
        raw = struct.pack("<ff", c.real, c.imag)
    elif dt == GA_C128:
        c = complex(value)
        raw = struct.pack("<dd", c.real, c.imag)
    else:
        raise ValueError(f"bad dtype {dt}")
    raw = raw.ljust(16, b"\0")
    s = ga_scalar_t()
    s.dtype = dt
    s.reserved = 0
    s.bits, s.bits_hi = struct.unpack("<QQ", raw)
    return s


class GpuArrayError(RuntimeError):
    def __init__(self, status, detail):
        super().__init__(f"{_status_name(status)}: {detail}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python paper_1304_5553_b200/build.py). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, sz, st = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
    lib.gpuarray_axpbyz.restype = st
    lib.gpuarray_axpbyz.argtypes = [st, i64, ga_scalar_t, vp, ga_scalar_t, vp, vp, vp]
    lib.gpuarray_axpbz.restype = st
    lib.gpuarray_axpbz.argtypes = [st, i64, ga_scalar_t, vp, ga_scalar_t, vp, vp]
    lib.gpuarray_reduce_workspace_bytes.restype = sz
    lib.gpuarray_reduce_workspace_bytes.argtypes = [st, i64]
    lib.gpuarray_reduce.restype = st
    lib.gpuarray_reduce.argtypes = [st, st, st, st, i64, vp, vp, vp, vp, sz, vp]
    lib.gpuarray_scan_workspace_bytes.restype = sz
    lib.gpuarray_scan_workspace_bytes.argtypes = [st, i64]
    lib.gpuarray_scan.restype = st
    lib.gpuarray_scan.argtypes = [st, st, st, st, i64, vp, vp, vp, i64, vp, sz, vp]
    lib.gpuarray_status_string.restype = ctypes.c_char_p
    lib.gpuarray_status_string.argtypes = [st]
    lib.gpuarray_last_error.restype = ctypes.c_char_p
    lib.gpuarray_last_error.argtypes = []
    lib.gpuarray_abi_version.restype = ctypes.c_int
    lib.gpuarray_abi_version.argtypes = []
    lib.gpuarray_launch_count.restype = ctypes.c_uint64
    lib.gpuarray_launch_count.argtypes = []
    lib.gpuarray_xgpu_buffer_bytes.restype = sz
    lib.gpuarray_xgpu_buffer_bytes.argtypes = []
    lib.gpuarray_reduce_xgpu.restype = st
    lib.gpuarray_reduce_xgpu.argtypes = [st, st, st, st, i64, vp, vp, vp, vp, sz, vp, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_uint64, st, vp]
    lib.gpuarray_elementwise.restype = st
    lib.gpuarray_elementwise.argtypes = [st, st, i64, vp, vp, vp, vp]
    lib.gpuarray_axpbyz_ds.restype = st
    lib.gpuarray_axpbyz_ds.argtypes = [st, i64, ga_dscalar_t, vp, ga_dscalar_t, vp, vp, vp]
    lib.gpuarray_stencil3.restype = st
    lib.gpuarray_stencil3.argtypes = [st, i64, ga_scalar_t, ga_scalar_t, ga_scalar_t, vp, vp, vp, vp]
    lib.gpuarray_cg_direction.restype = st
    lib.gpuarray_cg_direction.argtypes = [st, i64, ga_dscalar_t, vp, vp, vp, ga_scalar_t, ga_scalar_t, ga_scalar_t, vp,
                                          vp, vp, vp, sz, vp]
    lib.gpuarray_reduce_sharded.restype = st
    lib.gpuarray_reduce_sharded.argtypes = [st, st, st, st, i64, vp, vp, vp, vp, sz, vp, vp]
    lib.gpuarray_scan_sharded_workspace_bytes.restype = sz
    lib.gpuarray_scan_sharded_workspace_bytes.argtypes = [st, i64]
    lib.gpuarray_scan_sharded.restype = st
    lib.gpuarray_scan_sharded.argtypes = [st, st, st, st, i64, vp, vp, vp, i64, vp, sz, vp, vp]
    lib.gpuarray_cg_update.restype = st
    lib.gpuarray_cg_update.argtypes = [st, i64, ga_dscalar_t, vp, vp, vp, vp, vp, vp, sz, vp]
    return lib


LIB = _load()


def _status_name(s):
    return LIB.gpuarray_status_string(s).decode()


def gpuarray_axpbyz(dt, n, a, x, b, y, z, stream):
    return LIB.gpuarray_axpbyz(dt, n, a, x, b, y, z, stream)


def gpuarray_axpbz(dt, n, a, x, b, z, stream):
    return LIB.gpuarray_axpbz(dt, n, a, x, b, z, stream)


def gpuarray_reduce_workspace_bytes(out_dt, n):
    return LIB.gpuarray_reduce_workspace_bytes(out_dt, n)


def gpuarray_reduce(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, stream):
    return LIB.gpuarray_reduce(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, stream)


def gpuarray_xgpu_buffer_bytes():
    return LIB.gpuarray_xgpu_buffer_bytes()


GA_XGPU_ALL, GA_XGPU_EXCLUSIVE_PREFIX = 0, 1


def gpuarray_reduce_xgpu(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, peer_buffers, rank, world,
                         seq, fold, stream):
    return LIB.gpuarray_reduce_xgpu(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, peer_buffers,
                                    rank, world, seq, fold, stream)


def gpuarray_scan_workspace_bytes(dt, n):
    return LIB.gpuarray_scan_workspace_bytes(dt, n)


def gpuarray_scan(op, kind, in_dt, out_dt, n, in_, out, carry, carry_count, workspace, workspace_bytes, stream):
    return LIB.gpuarray_scan(op, kind, in_dt, out_dt, n, in_, out, carry, carry_count, workspace, workspace_bytes,
                             stream)


def gpuarray_reduce_sharded(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, nccl_comm, stream):
    return LIB.gpuarray_reduce_sharded(op, map_, in_dt, out_dt, n, x, y, out, workspace, workspace_bytes, nccl_comm,
                                       stream)


def gpuarray_scan_sharded_workspace_bytes(out_dt, n):
    return LIB.gpuarray_scan_sharded_workspace_bytes(out_dt, n)


def gpuarray_scan_sharded(op, kind, in_dt, out_dt, n, in_, out, carry, carry_count, workspace, workspace_bytes,
                          nccl_comm, stream):
    return LIB.gpuarray_scan_sharded(op, kind, in_dt, out_dt, n, in_, out, carry, carry_count, workspace,
                                     workspace_bytes, nccl_comm, stream)


GA_EW_MUL, GA_EW_DIV, GA_EW_SQRT, GA_EW_ABS, GA_EW_NEG, GA_EW_EXP, GA_EW_LOG, GA_EW_SIN, GA_EW_COS, GA_EW_MAX, \
    GA_EW_MIN = range(11)


def gpuarray_elementwise(op, dt, n, x, y, z, stream):
    return LIB.gpuarray_elementwise(op, dt, n, x, y, z, stream)


def gpuarray_axpbyz_ds(dt, n, a, x, b, y, z, stream):
    return LIB.gpuarray_axpbyz_ds(dt, n, a, x, b, y, z, stream)


def gpuarray_stencil3(dt, n, l, d, u, diag, x, y, stream):
    return LIB.gpuarray_stencil3(dt, n, l, d, u, diag, x, y, stream)


def gpuarray_status_string(status):
    return _status_name(status)


def gpuarray_last_error():
    return LIB.gpuarray_last_error().decode()


def gpuarray_abi_version():
    return LIB.gpuarray_abi_version()


def gpuarray_launch_count():
    return LIB.gpuarray_launch_count()


def check(status):
    """Raise per the paper's exception model: ValueError for
    argument/workspace errors, TypeError for uninstantiated dtype/op combos,
    GpuArrayError (a RuntimeError) for CUDA errors."""
    if status == GA_OK:
        return
    detail = gpuarray_last_error()
    msg = f"{_status_name(status)}: {detail}"
    if status in (GA_ERR_INVALID_ARGUMENT, GA_ERR_WORKSPACE):
        raise ValueError(msg)
    if status == GA_ERR_UNSUPPORTED:
        raise TypeError(msg)
    raise GpuArrayError(status, detail)


def gpuarray_cg_direction(dt, n, beta, r, p_in, p_out, l, d, u, diag, ap, pap, workspace, workspace_bytes, stream):
    return LIB.gpuarray_cg_direction(dt, n, beta, r, p_in, p_out, l, d, u, diag, ap, pap, workspace, workspace_bytes,
                                     stream)


def gpuarray_cg_update(dt, n, alpha, x, r, p, ap, rr, workspace, workspace_bytes, stream):
    return LIB.gpuarray_cg_update(dt, n, alpha, x, r, p, ap, rr, workspace, workspace_bytes, stream)
