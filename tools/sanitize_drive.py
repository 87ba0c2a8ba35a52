"""Exercise every libgpuarray kernel family at small, ragged and unaligned
sizes (no checks: the parity tests do that) so compute-sanitizer can watch
for out-of-bounds accesses, races and barrier misuse:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_drive.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1304_5553_b200 import gpuarray as G  # noqa: E402

dev = torch.device("cuda:0")


def arr(n, dt, off=0):
    buf = (torch.rand(n + off, device=dev) * 10).to(dt)
    return buf[off:]


for n in (1, 7, 33, 1000, 4099, 70_001, 300_007):
    for off in (0, 1):
        for dt in (torch.float32, torch.float64, torch.int32, torch.int64):
            x, y = arr(n, dt, off), arr(n, dt, off)
            G.axpbyz(2, x, 3, y)
            G.axpbz(2, x, 1)
            G.sum(x)
            G.max(x)
            G.min(x)
            G.dot(x, y)
            G.norm2sq(x)
            G.elementwise(G._abi.GA_EW_MUL, x, y)
            G.elementwise(G._abi.GA_EW_MAX, x, y)
            G.elementwise(G._abi.GA_EW_NEG, x)
            for op in (G.SUM, G.MAX, G.MIN):
                G.scan(x, op=op)
                G.scan(x, exclusive=True, op=op, carry=arr(2, dt))
            if dt == torch.int32:
                G.scan(x, out_dtype=torch.int64)
            if dt == torch.float32:
                G.scan(x, out_dtype=torch.float64, exclusive=True)
            if dt.is_floating_point:
                G.elementwise(G._abi.GA_EW_SQRT, x)
                G.elementwise(G._abi.GA_EW_EXP, x)
                G.stencil3(-1, 2, -1, x)
                G.stencil3(-1, 2, -1, x, diag=arr(n, dt, off))
                one = torch.ones(1, dtype=dt, device=dev)
                G.axpbyz_ds(1.0, x, 1.0, y, b_num=one, b_den=one)
                p2, ap = arr(n, dt, off), arr(n, dt, off)
                G.cg_direction(x, y, p2, ap, beta_num=one, beta_den=one)
                G.cg_direction(x, y, p2, ap, beta_num=one, beta_den=one, diag=arr(n, dt, off))
                G.cg_update(arr(n, dt, off), arr(n, dt, off), p2, ap, alpha_num=one, alpha_den=one)
        for cdt in (torch.complex64, torch.complex128):
            xc = torch.randn(n + off, dtype=cdt, device=dev)[off:]
            yc = torch.randn(n + off, dtype=cdt, device=dev)[off:]
            G.axpbyz(1 + 2j, xc, 3, yc)
            G.vdot(xc, yc)
            G.dot(xc, yc)
            G.norm2sq(xc)
    torch.cuda.synchronize()

# multi-group reduction finishes (grids of 129 and 300 blocks: group leaders
# waiting on tagged slots, the grid leader folding group slots), 4-, 8- and
# 16-byte partials on one workspace
for n in (129 * 16384 - 3, 300 * 16384 + 5):
    for dt in (torch.float32, torch.float64, torch.int32, torch.int64):
        x, y = arr(n, dt), arr(n, dt)
        G.sum(x)
        G.max(x)
        G.dot(x, y)
    xc = torch.randn(n, dtype=torch.complex128, device=dev)
    G.vdot(xc, xc)
    G.cg_update(arr(n, torch.float32), arr(n, torch.float32), arr(n, torch.float32), arr(n, torch.float32),
                alpha_num=torch.ones(1, device=dev), alpha_den=torch.ones(1, device=dev))
    torch.cuda.synchronize()

# Ring scans (48 MiB .. 384 / 768 MiB of non-widening input: persistent CTAs,
# TMA bulk stages, mbarriers, register double buffer): every op, in place,
# carry-in, a 16-byte view offset, ragged tails of 1-3 elements past the last
# 16-byte multiple (element-wise tail reads)
for n, dt in (((48 << 20) // 4 + 3, torch.int32), ((64 << 20) // 8 + 1, torch.int64),
              ((64 << 20) // 4 + 2, torch.float32), ((96 << 20) // 8 + 5, torch.float64)):
    for off in (0, 2):
        x = arr(n, dt, off)
        for op in (G.SUM, G.MAX, G.MIN):
            G.scan(x, op=op)
        G.scan(x, exclusive=True, carry=arr(3, dt))
        G.scan(x, exclusive=True, out=x)
        torch.cuda.synchronize()
# L-shape scans (above the ring window; >= 256 super-tiles: the look-back L2
# prefetch of the tile 42 ids ahead is active), in place and out of place,
# plus a ragged tail (8-byte and widened L-shape scans read 1 KiB rows when
# 32-byte aligned and 512-byte rows otherwise: both, via a 2-element
# (16-byte) view offset)
for n, dt in (((4 << 30) // 4 + 12345, torch.int32), ((2 << 30) // 8 + 777, torch.int64),
              ((2 << 30) // 8 + 999, torch.float64)):
    for off in (0, 2):
        x = arr(n, dt, off)
        G.scan(x)
        G.scan(x, exclusive=True, out=x)
        torch.cuda.synchronize()
for dt, wide in ((torch.int32, torch.int64), (torch.float32, torch.float64)):
    x = arr(256 * 98304 + 4321, dt)
    G.scan(x, out_dtype=wide)
    G.scan(x, out_dtype=wide, exclusive=True)
    torch.cuda.synchronize()
print("drive ok", G.launch_count(), "launches")
