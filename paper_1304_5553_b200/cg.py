"""Unpreconditioned conjugate gradients on the GPUArray kernels (SURVEY.md
§8(f) NEXT-4): the paper's "conjugate-gradient-based Krylov solver for large,
sparse linear systems" built from exactly the hot-path
operations — dot, squared 2-norm, axpbyz — plus the three-point stencil
operator (gpuarray_stencil3), for symmetric tridiagonal systems
A = tridiag(l, d_i, l) such as 1-D Poisson (l = -1, d = 2).

Every vector operation is one libgpuarray.so kernel; the two scalars per
iteration (p.Ap and r.r) are brought to the host with .item(), the GPUArray
scalar's `get`, to form alpha and beta.
"""
import math

import torch

from . import gpuarray as G


class CGResult:
    def __init__(self, x, iterations, residual_norms, converged):
        self.x = x
        self.iterations = iterations
        self.residual_norms = residual_norms  # ||r_k||_2, k = 0 .. iterations
        self.converged = converged


def cg(b, offdiag=-1.0, d=2.0, diag=None, x0=None, rtol=1e-10, maxiter=None):
    """Solve A x = b, A = tridiag(offdiag, d_i, offdiag) (d_i = diag[i] if a
    diagonal tensor is given), to ||b - A x|| <= rtol * ||b||."""
    G._check_array("b", b)
    if not b.dtype.is_floating_point or b.is_complex():
        raise TypeError("cg needs a float32 or float64 right-hand side")
    n = b.numel()
    maxiter = n if maxiter is None else maxiter
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = torch.empty_like(b)
    p = torch.empty_like(b)
    ap = torch.empty_like(b)
    G.stencil3(offdiag, d, offdiag, x, diag=diag, out=ap)          # A x0
    G.axpbyz(1.0, b, -1.0, ap, out=r)                               # r = b - A x0
    G.axpbz(1.0, r, -0.0, out=p)                                    # p = r (b = -0.0: exact copy)
    rs = float(G.norm2sq(r).item())
    bnorm = math.sqrt(float(G.norm2sq(b).item()))
    hist = [math.sqrt(rs)]
    k = 0
    while k < maxiter and math.sqrt(rs) > rtol * bnorm:
        G.stencil3(offdiag, d, offdiag, p, diag=diag, out=ap)       # Ap
        pap = float(G.dot(p, ap).item())
        if pap <= 0.0:
            raise ArithmeticError("p.Ap <= 0: the operator is not symmetric positive definite")
        alpha = rs / pap
        G.axpbyz(1.0, x, alpha, p, out=x)                           # x += alpha p
        G.axpbyz(1.0, r, -alpha, ap, out=r)                         # r -= alpha Ap
        rs_new = float(G.norm2sq(r).item())
        G.axpbyz(1.0, r, rs_new / rs, p, out=p)                     # p = r + beta p
        rs = rs_new
        k += 1
        hist.append(math.sqrt(rs))
    return CGResult(x, k, hist, math.sqrt(rs) <= rtol * bnorm)
