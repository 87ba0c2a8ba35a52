"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/gpuarray.h declares, and validates arguments synchronously
(no kernel is launched for invalid calls, so these run without a GPU)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gpuarray.h")).read()
    return sorted(set(re.findall(r"\b(gpuarray_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def abi():
    from conftest import product_build
    product_build()
    from paper_1304_5553_b200 import _abi
    return _abi


def test_exports_every_declared_symbol(abi):
    declared = header_symbols()
    assert len(declared) == 20
    assert sorted(abi.EXPORTS) == declared
    for name in declared:
        assert hasattr(abi.LIB, name), name


def test_nm_shows_c_linkage(abi):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_symbols():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_version_and_strings(abi):
    assert abi.gpuarray_abi_version() == 5
    assert abi.gpuarray_status_string(abi.GA_OK) == "GA_OK"
    assert abi.gpuarray_status_string(abi.GA_ERR_CUDA) == "GA_ERR_CUDA"
    assert abi.gpuarray_status_string(abi.GA_ERR_NCCL) == "GA_ERR_NCCL"
    assert abi.gpuarray_status_string(99) == "GA_ERR_UNKNOWN"


def test_workspace_sizes(abi):
    assert abi.gpuarray_reduce_workspace_bytes(abi.GA_F32, 1 << 30) == 128 + 32 * 32768 + 32 * 256
    assert abi.gpuarray_xgpu_buffer_bytes() == 2 * 64 * 32
    a = abi.gpuarray_scan_workspace_bytes(abi.GA_I32, 1 << 30)
    assert a == 256 + 8 * ((1 << 30) // 4096)
    b = abi.gpuarray_scan_workspace_bytes(abi.GA_I64, 1 << 20)
    tiles = (1 << 20) // 4096  # status for the smaller (fallback) tile of 4096 elements
    assert b == 256 + tiles * 16  # two tagged 64-bit words per tile for 8-byte types
    assert abi.gpuarray_scan_workspace_bytes(abi.GA_F32, 100) == 256 + 8   # float scans too
    assert abi.gpuarray_scan_workspace_bytes(abi.GA_F64, 4096) == 256 + 16


def test_argument_validation_is_synchronous(abi):
    f32 = abi.make_scalar(abi.GA_F32, 1.0)
    f64 = abi.make_scalar(abi.GA_F64, 1.0)
    E = abi.GA_ERR_INVALID_ARGUMENT
    assert abi.gpuarray_axpbyz(abi.GA_F32, -1, f32, None, f32, None, None, None) == E
    assert abi.gpuarray_axpbyz(abi.GA_F32, 0, f32, None, f32, None, None, None) == abi.GA_OK  # no-op
    assert abi.gpuarray_axpbyz(abi.GA_F32, 4, f32, 4096, f64, 8192, 12288, None) == E        # scalar dtype
    assert "scalar dtype" in abi.gpuarray_last_error()
    assert abi.gpuarray_axpbyz(abi.GA_F32, 4, f32, None, f32, 8192, 12288, None) == E         # NULL x
    assert abi.gpuarray_axpbyz(abi.GA_F32, 16, f32, 4096, f32, 8192, 4100, None) == E         # partial overlap
    assert abi.gpuarray_axpbyz(7, 4, f32, 4096, f32, 8192, 12288, None) == E                  # bad dtype
    assert abi.gpuarray_axpbz(abi.GA_F32, 4, f32, 4096, f64, 12288, None) == E
    ws = abi.gpuarray_reduce_workspace_bytes(abi.GA_F32, 4)
    R = abi.gpuarray_reduce
    assert R(5, 0, 0, 0, 4, 4096, None, 64, 128, ws, None) == E                                # bad op
    assert R(0, 5, 0, 0, 4, 4096, None, 64, 128, ws, None) == E                                # bad map
    assert R(0, abi.GA_MAP_CONJ_MUL, 0, 0, 4, 4096, None, 64, 128, ws, None) == E              # CONJ_MUL without y
    assert R(1, 0, abi.GA_C64, abi.GA_C64, 4, 4096, None, 64, 128, ws, None) == abi.GA_ERR_UNSUPPORTED  # max of complex
    assert R(0, 2, abi.GA_C64, abi.GA_C64, 4, 4096, None, 64, 128, ws, None) == abi.GA_ERR_UNSUPPORTED  # |x|^2 -> real
    assert R(0, abi.GA_MAP_MUL, 0, 0, 4, 4096, None, 64, 128, ws, None) == E                   # MUL without y
    assert R(0, 0, 0, 0, 4, 4096, None, None, 128, ws, None) == E                              # no out
    assert R(0, 0, 0, 0, 4, 4096, None, 64, 128, ws - 1, None) == abi.GA_ERR_WORKSPACE
    assert R(0, 0, 0, 0, 4, 4096, None, 64, None, ws, None) == abi.GA_ERR_WORKSPACE
    S = abi.gpuarray_scan
    sw = abi.gpuarray_scan_workspace_bytes(abi.GA_I32, 100)
    I32, I64 = abi.GA_I32, abi.GA_I64
    assert S(5, 0, I32, I32, 100, 4096, 8192, None, 0, 64, sw, None) == E                    # bad op
    assert S(0, 0, 9, 9, 100, 4096, 8192, None, 0, 64, sw, None) == E                        # bad dtype
    assert S(0, 0, abi.GA_C64, abi.GA_C64, 100, 4096, 8192, None, 0, 64, sw, None) == abi.GA_ERR_UNSUPPORTED
    assert S(0, 0, I64, I32, 100, 4096, 8192, None, 0, 64, sw, None) == abi.GA_ERR_UNSUPPORTED  # narrowing
    assert S(0, 0, I32, abi.GA_F64, 100, 4096, 8192, None, 0, 64, sw, None) == abi.GA_ERR_UNSUPPORTED
    assert S(0, 3, I32, I32, 100, 4096, 8192, None, 0, 64, sw, None) == E                    # bad kind
    assert S(0, 0, I32, I32, 100, 4096, 8192, None, 2, 64, sw, None) == E                    # carry NULL
    assert S(0, 0, I32, I32, 100, 4096, 4100, None, 0, 64, sw, None) == E                    # partial overlap
    sw64 = abi.gpuarray_scan_workspace_bytes(I64, 100)
    assert S(0, 0, I32, I64, 100, 4096, 4096, None, 0, 64, sw64, None) == E                  # widening in place
    assert "in place" in abi.gpuarray_last_error()
    assert S(0, 0, I32, I32, 100, 4096, 8192, None, 0, 64, sw - 1, None) == abi.GA_ERR_WORKSPACE
    assert S(0, 0, I32, I32, 0, None, None, None, 0, None, 0, None) == abi.GA_OK           # n == 0 no-op


def test_sharded_validation(abi):
    """The sharded entries validate synchronously like the local ones; a NULL
    communicator is an argument error (no NCCL call is made)."""
    E = abi.GA_ERR_INVALID_ARGUMENT
    ws = abi.gpuarray_reduce_workspace_bytes(abi.GA_F32, 4)
    RS = abi.gpuarray_reduce_sharded
    assert RS(0, 0, 0, 0, 4, 4096, None, 64, 128, ws, None, None) == E                       # no comm
    assert RS(1, 0, abi.GA_C64, abi.GA_C64, 4, 4096, None, 64, 128, ws, 0x1000, None) == abi.GA_ERR_UNSUPPORTED
    SS = abi.gpuarray_scan_sharded
    I32, I64 = abi.GA_I32, abi.GA_I64
    sw = abi.gpuarray_scan_sharded_workspace_bytes(I32, 100)
    # reduce workspace + carries (4098 x 8 B, rounded to 256 B) + scan workspace
    red = abi.gpuarray_reduce_workspace_bytes(I32, 100)
    assert sw == (red + 4098 * 8 + 255) // 256 * 256 + abi.gpuarray_scan_workspace_bytes(I32, 100)
    assert SS(0, 0, I32, I32, 100, 4096, 8192, None, 0, 64, sw, None, None) == E              # no comm
    assert SS(0, 0, I32, I32, -1, 4096, 8192, None, 0, 64, sw, 0x1000, None) == E             # n < 0
    assert SS(0, 0, I32, I32, 100, 4096, 8192, None, 3, 64, sw, 0x1000, None) == E            # carry NULL
    assert SS(1, 0, I32, I64, 100, 4096, 8192, None, 0, 64, sw, 0x1000, None) == abi.GA_ERR_UNSUPPORTED
    assert SS(0, 0, I32, I32, 100, 4096, 8192, None, 0, 64, sw - 1, 0x1000, None) == abi.GA_ERR_WORKSPACE


def test_cg_step_validation(abi):
    """The fused CG steps reject bad arguments before any launch."""
    E = abi.GA_ERR_INVALID_ARGUMENT
    F32 = abi.GA_F32
    s32 = abi.make_scalar(F32, 1.0)
    ds = abi.make_dscalar(F32, 1.0)
    ws = abi.gpuarray_reduce_workspace_bytes(F32, 1000)
    D = abi.gpuarray_cg_direction
    # r=4096, p_in=8192, p_out=12288, ap=16384 (1000 floats = 4000 bytes each)
    assert D(abi.GA_I32, 1000, abi.make_dscalar(abi.GA_I32, 1), 4096, 8192, 12288, s32, s32, s32, None, 16384, 64,
             128, ws, None) == abi.GA_ERR_UNSUPPORTED
    assert D(F32, 1000, ds, 4096, 8192, 8192, s32, s32, s32, None, 16384, 64, 128, ws, None) == E  # p_out = p_in
    assert D(F32, 1000, ds, 4096, 8192, 12288, s32, s32, s32, None, 12290, 64, 128, ws, None) == E  # ap in p_out
    assert D(F32, 1000, ds, 4096, 8192, 12288, s32, s32, s32, 16384, 16384, 64, 128, ws, None) == E  # ap = diag
    assert D(F32, 1000, ds, 4096, 8192, 12288, s32, s32, s32, None, 16384, None, 128, ws, None) == E  # no pap
    assert D(F32, 1000, ds, 4096, 8192, 12288, s32, s32, s32, None, 16384, 64, 128, ws - 1, None) == \
        abi.GA_ERR_WORKSPACE
    assert D(F32, 1000, abi.make_dscalar(abi.GA_F64, 1.0), 4096, 8192, 12288, s32, s32, s32, None, 16384, 64, 128,
             ws, None) == E                                                                     # scalar dtype
    U = abi.gpuarray_cg_update
    assert U(F32, 1000, ds, 4096, 4096, 8192, 12288, 64, 128, ws, None) == E                   # x = r
    assert U(F32, 1000, ds, 4096, 8192, 12288, 12300, 64, 128, ws, None) == E                  # p, ap overlap
    assert U(F32, -1, ds, 4096, 8192, 12288, 16384, 64, 128, ws, None) == E
    assert U(abi.GA_C64, 10, ds, 4096, 8192, 12288, 16384, 64, 128, ws, None) == abi.GA_ERR_UNSUPPORTED


def test_python_error_mapping(abi):
    with pytest.raises(ValueError):
        abi.check(abi.GA_ERR_INVALID_ARGUMENT)
    with pytest.raises(TypeError):
        abi.check(abi.GA_ERR_UNSUPPORTED)
    with pytest.raises(RuntimeError):
        abi.check(abi.GA_ERR_CUDA)


def test_scalar_marshalling(abi):
    import struct
    s = abi.make_scalar(abi.GA_F32, 5.7)
    assert struct.unpack("<f", struct.pack("<Q", s.bits)[:4])[0] == struct.unpack("<f", struct.pack("<f", 5.7))[0]
    s = abi.make_scalar(abi.GA_I32, -1)
    assert s.bits == 0xFFFFFFFF
    s = abi.make_scalar(abi.GA_I64, -2)
    assert s.bits == (1 << 64) - 2
    s = abi.make_scalar(abi.GA_C64, 1.5 - 2j)
    assert struct.unpack("<ff", struct.pack("<Q", s.bits)) == (1.5, -2.0) and s.bits_hi == 0
    s = abi.make_scalar(abi.GA_C128, 0.25 + 4j)
    assert struct.unpack("<dd", struct.pack("<QQ", s.bits, s.bits_hi)) == (0.25, 4.0)
    import ctypes
    assert ctypes.sizeof(abi.ga_scalar_t) == 24
