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


class GraphCG:
    """CG with every scalar left on the GPU: alpha = rs/pAp and beta =
    rs_new/rs enter the kernels as device-resident factors (ga_dscalar_t), so
    `block` iterations (an even number) are captured ONCE in a CUDA graph at
    construction and replayed by every solve(); the host reads the residual
    only between blocks.  Iteration counts are rounded up to whole blocks (a
    zero numerator keeps a converged iteration finite, see ga_dscalar_t).

    fused=True (default): two kernels per iteration, gpuarray_cg_direction
    (p = r + beta p; Ap; p.Ap) and gpuarray_cg_update (x += alpha p;
    r -= alpha Ap; r.r) — 10 element-sizes of HBM traffic per iteration.
    fused=False: the six single-operation kernels (stencil3, dot, three
    axpbyz_ds, norm2sq) — 14 element-sizes."""

    def __init__(self, n, dtype=torch.float64, offdiag=-1.0, d=2.0, diag=None, block=16, device=None, fused=True):
        if block < 2 or block % 2:
            raise ValueError("block must be an even number >= 2")
        if dtype not in (torch.float32, torch.float64):
            raise TypeError("GraphCG needs float32 or float64")
        dev = torch.device(device or "cuda")
        self.n, self.block, self.dev, self.fused = n, block, dev, fused
        self.offdiag, self.d, self.diag = offdiag, d, diag
        mk = lambda: torch.zeros(n, dtype=dtype, device=dev)  # noqa: E731
        self.b, self.x, self.r, self.p, self.ap = mk(), mk(), mk(), mk(), mk()
        self.p2 = [self.p, mk()] if fused else None  # fused: p ping-pongs (neighbours are read)
        self.rs = [torch.zeros(1, dtype=dtype, device=dev) for _ in range(2)]
        self.pap = torch.zeros(1, dtype=dtype, device=dev)
        self.stream = torch.cuda.Stream(dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):  # warm-up: module loading, workspaces
            self.b.fill_(1.0)
            self._start()
            for k in range(block):
                self._iteration(k)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            for k in range(block):
                self._iteration(k)

    def _start(self):
        G.stencil3(self.offdiag, self.d, self.offdiag, self.x, diag=self.diag, out=self.ap)
        G.axpbyz(1.0, self.b, -1.0, self.ap, out=self.r)
        G.reduce(G.SUM, G.SQUARE, self.r, out=self.rs[0])
        if self.fused:
            # iteration 0 forms p = r + beta*0 with beta = rs0 / 1 (finite)
            self.p2[1].zero_()
            self.rs[1].fill_(1.0)
        else:
            G.axpbz(1.0, self.r, -0.0, out=self.p)

    def _iteration(self, k):
        if self.fused:
            return self._iteration_fused(k)
        cur, nxt = self.rs[k & 1], self.rs[(k + 1) & 1]
        x, r, p, ap, pap = self.x, self.r, self.p, self.ap, self.pap
        G.stencil3(self.offdiag, self.d, self.offdiag, p, diag=self.diag, out=ap)
        G.reduce(G.SUM, G.MUL, p, ap, out=pap)
        G.axpbyz_ds(1.0, x, 1.0, p, out=x, b_num=cur, b_den=pap)      # x += (rs/pAp) p
        G.axpbyz_ds(1.0, r, -1.0, ap, out=r, b_num=cur, b_den=pap)    # r -= (rs/pAp) Ap
        G.reduce(G.SUM, G.SQUARE, r, out=nxt)                          # rs_new
        G.axpbyz_ds(1.0, r, 1.0, p, out=p, b_num=nxt, b_den=cur)      # p = r + (rs_new/rs) p

    def _iteration_fused(self, k):
        cur, prev = self.rs[k & 1], self.rs[(k + 1) & 1]
        pin, pout = self.p2[(k + 1) & 1], self.p2[k & 1]
        G.cg_direction(self.r, pin, pout, self.ap, beta=1.0, beta_num=cur, beta_den=prev, l=self.offdiag, d=self.d,
                       u=self.offdiag, diag=self.diag, out=self.pap)               # p = r + (rs/rs_prev) p; Ap; p.Ap
        G.cg_update(self.x, self.r, pout, self.ap, alpha=1.0, alpha_num=cur, alpha_den=self.pap,
                    out=prev)                                                     # x, r update; rs_new -> rs[(k+1)&1]

    def solve(self, b, x0=None, rtol=1e-10, maxiter=None):
        G._check_array("b", b)
        if b.numel() != self.n or b.dtype != self.b.dtype:
            raise ValueError("b does not match the solver's size / dtype")
        maxiter = self.n if maxiter is None else maxiter
        s = self.stream
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.b.copy_(b)
            if x0 is None:
                self.x.zero_()
            else:
                self.x.copy_(x0)
            self._start()
            bnorm = math.sqrt(float(G.norm2sq(self.b).item()))
            res = math.sqrt(float(self.rs[0].item()))
        hist = [res]
        k, conv = 0, res <= rtol * bnorm
        while not conv and k < maxiter:
            self.graph.replay()
            k += self.block
            res = math.sqrt(float(self.rs[0].item()))  # block is even: rs[0] holds the latest
            hist.append(res)
            conv = res <= rtol * bnorm
        torch.cuda.current_stream(self.dev).wait_stream(s)
        return CGResult(self.x.clone(), k, hist, conv)


def cg_graph(b, offdiag=-1.0, d=2.0, diag=None, x0=None, rtol=1e-10, maxiter=None, block=16, fused=True):
    """One-shot convenience wrapper around GraphCG (captures a graph per call;
    build a GraphCG once to solve repeatedly)."""
    solver = GraphCG(b.numel(), b.dtype, offdiag, d, diag, block, b.device, fused=fused)
    return solver.solve(b, x0=x0, rtol=rtol, maxiter=maxiter)
