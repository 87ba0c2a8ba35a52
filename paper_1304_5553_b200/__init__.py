"""paper_1304_5553_b200 — a B200-native (sm_100a) implementation of the
GPUArray hot path of arXiv 1304.5553 (PyCUDA/PyOpenCL chapter): fused
elementwise linear combinations, single-pass map-reduce and single-pass
decoupled-look-back scan, behind a C ABI (include/gpuarray.h).

Importing requires the built CUDA library (libgpuarray.so); there is no CPU
fallback.  See DESIGN.md."""
from . import gpuarray  # noqa: F401
from .gpuarray import (axpbyz, axpbyz_ds, axpbz, cg_direction, cg_update, dot, elementwise,  # noqa: F401
                       launch_count, max, min, norm2sq, reduce, scan, stencil3, sum, vdot)

__all__ = ["gpuarray", "axpbyz", "axpbyz_ds", "axpbz", "reduce", "dot", "vdot", "sum", "norm2sq", "max", "min",
           "scan", "elementwise", "stencil3", "cg_direction", "cg_update", "launch_count"]
