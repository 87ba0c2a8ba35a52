"""NEXT-4: the stencil operator (bit-exact vs the oracle) and unpreconditioned
CG built from the hot-path kernels, checked against SPEC.md's acceptance
criterion 9 (S:649-657 area) and numpy's dense solver."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import cg as gcg
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"
NPT = {np.float32: torch.float32, np.float64: torch.float64}


def to_dev(a, offset=0):
    buf = torch.empty(a.size + offset, dtype=NPT[a.dtype.type], device=DEV)
    v = buf[offset:]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 255, 256, 257, 4099, 1_000_003])
@pytest.mark.parametrize("with_diag", [False, True])
def test_stencil3_bit_exact(dt, n, with_diag):
    x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 1, n)
    diag = synth.host_fill(synth.F32_U01 if dt == np.float32 else synth.F64_U01, 2, n) if with_diag else None
    l, d, u = dt(-1.25), dt(2.5), dt(-0.75)
    ref = oracle.stencil3(l, d, u, x, diag=diag)
    for offs in (0, 3):
        got = G.stencil3(float(l), float(d), float(u), to_dev(x, offs),
                         diag=to_dev(diag, offs) if with_diag else None).cpu().numpy()
        assert np.array_equal(bits(got), bits(ref))


def test_cg_spec_poisson_64():
    """SPEC acceptance 9: 1-D Poisson n = 64 in f64 converges with
    ||b - Ax|| <= 1e-10 ||b|| in <= 64 iterations; matches numpy's dense solve."""
    n = 64
    b = torch.ones(n, dtype=torch.float64, device=DEV)
    res = gcg.cg(b, offdiag=-1.0, d=2.0, rtol=1e-10)
    assert res.converged and res.iterations <= 64
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    xs = np.linalg.solve(A, np.ones(n))
    x = res.x.cpu().numpy()
    assert np.max(np.abs(x - xs)) <= 1e-9 * np.max(np.abs(xs))
    # the residual the solver tracked equals the oracle's b - A x
    r = np.ones(n) - oracle.stencil3(-1.0, 2.0, -1.0, x)
    assert np.linalg.norm(r) <= 1e-10 * np.sqrt(n) * 1.0001


def test_cg_spec_2x2():
    """SPEC acceptance 9: [[4,1],[1,3]] x = [1,2] matches the dense solve to 1e-12."""
    b = torch.tensor([1.0, 2.0], dtype=torch.float64, device=DEV)
    diag = torch.tensor([4.0, 3.0], dtype=torch.float64, device=DEV)
    res = gcg.cg(b, offdiag=1.0, diag=diag, rtol=1e-14)
    xs = np.linalg.solve(np.array([[4.0, 1.0], [1.0, 3.0]]), np.array([1.0, 2.0]))
    assert res.iterations <= 2
    assert np.allclose(res.x.cpu().numpy(), xs, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("with_diag", [False, True])
def test_cg_large_consistency(dt, with_diag):
    """n = 2^20, a diagonally dominant tridiagonal system (d = 4 or a random
    diagonal in [4, 5), off-diagonal -1; condition number < 3): CG converges
    in tens of iterations, and the residual the solver tracked agrees with
    ||b - A x|| recomputed by the oracle on the host."""
    n = 1 << 20
    npdt = np.float32 if dt == torch.float32 else np.float64
    bh = synth.host_fill(synth.F32_S11 if npdt == np.float32 else synth.F64_S11, 5, n)
    dh = None
    if with_diag:
        dh = (4.0 + synth.host_fill(synth.F64_U01, 6, n)).astype(npdt)
    b = torch.from_numpy(bh).to(DEV)
    rtol = 1e-5 if dt == torch.float32 else 1e-12
    res = gcg.cg(b, offdiag=-1.0, d=4.0, diag=torch.from_numpy(dh).to(DEV) if with_diag else None, rtol=rtol,
                 maxiter=200)
    assert res.converged and 5 < res.iterations < 60
    x = res.x.cpu().numpy().astype(np.float64)
    r = bh.astype(np.float64) - oracle.stencil3(-1.0, 4.0, -1.0, x, diag=None if dh is None else dh.astype(np.float64))
    u = 2.0 ** -24 if dt == torch.float32 else 2.0 ** -53
    bn = np.linalg.norm(bh.astype(np.float64))
    assert np.linalg.norm(r) <= rtol * bn + 50 * u * bn
    assert abs(np.linalg.norm(r) - res.residual_norms[-1]) <= 50 * u * bn + 0.5 * np.linalg.norm(r)


def test_axpbyz_ds_bit_exact():
    """Device-resident factors: a = RN(scale * RN(num / den)); 0/0 -> 0."""
    n = 100_003
    for dt, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
        x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 1, n)
        y = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 2, n)
        num = torch.tensor([3.3], dtype=tdt, device=DEV)
        den = torch.tensor([-0.7], dtype=tdt, device=DEV)
        got = G.axpbyz_ds(1.5, to_dev(x), -2.0, to_dev(y), a_num=num, b_num=num, b_den=den).cpu().numpy()
        a = dt(dt(1.5) * dt(3.3))
        b = dt(dt(-2.0) * dt(dt(3.3) / dt(-0.7)))
        assert np.array_equal(bits(got), bits(oracle.axpbyz(a, x, b, y)))
        zero = torch.zeros(1, dtype=tdt, device=DEV)
        got = G.axpbyz_ds(1.0, to_dev(x), 5.0, to_dev(y), b_num=zero, b_den=zero).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle.axpbyz(dt(1), x, dt(0), y)))


def test_cg_graph_matches_host_cg_f64():
    """float64: the unfused device-scalar iteration runs the same kernels as
    the host one and forms the same alpha/beta bits (RN(rs/pAp) either way),
    so x and the residuals agree exactly over the same number of iterations.
    The fused iteration reduces p.Ap and r.r in another order (R28): close,
    not identical."""
    n = 1 << 16
    b = torch.from_numpy(synth.host_fill(synth.F64_S11, 7, n)).to(DEV)
    ref = gcg.cg(b, offdiag=-1.0, d=4.0, rtol=0.0, maxiter=32)
    got = gcg.cg_graph(b, offdiag=-1.0, d=4.0, rtol=0.0, maxiter=32, block=16, fused=False)
    assert got.iterations == ref.iterations == 32
    assert torch.equal(got.x, ref.x)
    assert got.residual_norms[-1] == ref.residual_norms[-1]
    fused = gcg.cg_graph(b, offdiag=-1.0, d=4.0, rtol=0.0, maxiter=32, block=16, fused=True)
    assert fused.iterations == 32
    assert torch.allclose(fused.x, ref.x, rtol=1e-9, atol=1e-12)


def test_cg_graph_converges_poisson():
    n = 64
    b = torch.ones(n, dtype=torch.float64, device=DEV)
    res = gcg.cg_graph(b, rtol=1e-10, block=8)
    assert res.converged and res.iterations <= 72
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    assert np.allclose(res.x.cpu().numpy(), np.linalg.solve(A, np.ones(n)), rtol=1e-8, atol=0)


# ------------------------------------------------------------------ fused CG steps (R28)
def _sdata(dt, n, seed, unit=False):
    if dt == np.float32:
        return synth.host_fill(synth.F32_U01 if unit else synth.F32_S11, seed, n)
    return synth.host_fill(synth.F64_U01 if unit else synth.F64_S11, seed, n)


def _dot_tol(dt, n, ref, sumabs):
    u = 2.0 ** -24 if dt == np.float32 else 2.0 ** -53
    rel = 1e-5 if dt == np.float32 else 1e-13
    return max(rel * abs(ref), n * u * sumabs)


FUSED_SIZES = [1, 2, 7, 8, 9, 255, 4099, 100_003, 1_000_003, (1 << 20) + 17]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", FUSED_SIZES)
@pytest.mark.parametrize("with_diag", [False, True])
def test_cg_direction_matches_composition(dt, n, with_diag):
    """p_out, ap bit-exact against the oracle's axpbyz(1, r, beta, p_in) then
    stencil3; p_out . ap within the dot tolerance (R9/R10); beta formed from
    device factors exactly as ga_dscalar_t says (RN(scale * RN(num / den)))."""
    tdt = NPT[dt]
    r, pin = _sdata(dt, n, 11), _sdata(dt, n, 12)
    diag = (dt(3.0) + _sdata(dt, n, 13, unit=True)).astype(dt) if with_diag else None
    l, d, u = dt(-1.25), dt(2.5), dt(-0.75)
    num = torch.tensor([0.37], dtype=tdt, device=DEV)
    den = torch.tensor([-1.9], dtype=tdt, device=DEV)
    beta = dt(dt(2.0) * dt(dt(0.37) / dt(-1.9)))
    p_ref = oracle.axpbyz(dt(1), r, beta, pin)
    ap_ref = oracle.stencil3(l, d, u, p_ref, diag=diag)
    dot_ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_MUL, p_ref, ap_ref, return_sumabs=True)
    for offs in (0, 3):  # vector path, scalar path
        pout = to_dev(np.zeros(n, dt), offs)
        ap = to_dev(np.zeros(n, dt), offs)
        got = G.cg_direction(to_dev(r, offs), to_dev(pin, offs), pout, ap, beta=2.0, beta_num=num, beta_den=den,
                             l=float(l), d=float(d), u=float(u), diag=to_dev(diag, offs) if with_diag else None)
        assert np.array_equal(bits(pout.cpu().numpy()), bits(p_ref))
        assert np.array_equal(bits(ap.cpu().numpy()), bits(ap_ref))
        assert abs(float(got.item()) - dot_ref) <= _dot_tol(dt, n, dot_ref, sa)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", FUSED_SIZES)
def test_cg_update_matches_composition(dt, n):
    """x' = axpbyz(1, x, alpha, p), r' = axpbyz(1, r, -alpha, ap) bit-exact;
    r'.r' within tolerance; alpha = RN(1 * RN(num / den))."""
    tdt = NPT[dt]
    x, r, p, ap = _sdata(dt, n, 21), _sdata(dt, n, 22), _sdata(dt, n, 23), _sdata(dt, n, 24)
    num = torch.tensor([1.7], dtype=tdt, device=DEV)
    den = torch.tensor([3.1], dtype=tdt, device=DEV)
    alpha = dt(dt(1.7) / dt(3.1))
    x_ref = oracle.axpbyz(dt(1), x, alpha, p)
    r_ref = oracle.axpbyz(dt(1), r, -alpha, ap)
    rr_ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, r_ref, return_sumabs=True)
    for offs in (0, 1):
        xd, rd = to_dev(x, offs), to_dev(r, offs)
        got = G.cg_update(xd, rd, to_dev(p, offs), to_dev(ap, offs), alpha=1.0, alpha_num=num, alpha_den=den)
        assert np.array_equal(bits(xd.cpu().numpy()), bits(x_ref))
        assert np.array_equal(bits(rd.cpu().numpy()), bits(r_ref))
        assert abs(float(got.item()) - rr_ref) <= _dot_tol(dt, n, rr_ref, sa)


def test_cg_fused_edge_cases():
    """n == 0 writes 0; a zero numerator gives a zero factor even over 0
    (a converged iteration stays finite); overlapping outputs are rejected."""
    for dt in (torch.float32, torch.float64):
        e = torch.empty(0, dtype=dt, device=DEV)
        assert float(G.cg_direction(e, e, e, e).item()) == 0.0
        assert float(G.cg_update(e, e, e, e).item()) == 0.0
        n = 1000
        z = torch.zeros(1, dtype=dt, device=DEV)
        r, pin = torch.zeros(n, dtype=dt, device=DEV), torch.full((n,), 7.0, dtype=dt, device=DEV)
        pout, ap = torch.empty_like(r), torch.empty_like(r)
        pap = G.cg_direction(r, pin, pout, ap, beta_num=z, beta_den=z)
        assert float(pap.item()) == 0.0 and bool((pout == 0).all()) and bool((ap == 0).all())
        x = torch.ones(n, dtype=dt, device=DEV)
        rr = G.cg_update(x, r, pout, ap, alpha_num=z, alpha_den=pap)
        assert float(rr.item()) == 0.0 and bool((x == 1).all())
        with pytest.raises(ValueError):
            G.cg_direction(r, pin, pin, ap)        # p_out aliases p_in
        with pytest.raises(ValueError):
            G.cg_update(x, x, pout, ap)            # x aliases r


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("with_diag", [False, True])
def test_cg_graph_fused_vs_unfused(dt, with_diag):
    """The fused iteration (2 kernels) and the 6-kernel one converge on the
    same diagonally dominant system to the same tolerance, in about the same
    number of iterations; the fused solution's residual, recomputed by the
    oracle, meets rtol."""
    n = (1 << 20) + 5
    npdt = np.float32 if dt == torch.float32 else np.float64
    bh = _sdata(npdt, n, 5)
    dh = (4.0 + synth.host_fill(synth.F64_U01, 6, n)).astype(npdt) if with_diag else None
    b = torch.from_numpy(bh).to(DEV)
    dd = torch.from_numpy(dh).to(DEV) if with_diag else None
    rtol = 1e-5 if dt == torch.float32 else 1e-12
    fused = gcg.cg_graph(b, offdiag=-1.0, d=4.0, diag=dd, rtol=rtol, maxiter=200, block=8, fused=True)
    plain = gcg.cg_graph(b, offdiag=-1.0, d=4.0, diag=dd, rtol=rtol, maxiter=200, block=8, fused=False)
    assert fused.converged and plain.converged
    assert abs(fused.iterations - plain.iterations) <= 8
    x = fused.x.cpu().numpy().astype(np.float64)
    r = bh.astype(np.float64) - oracle.stencil3(-1.0, 4.0, -1.0, x, diag=None if dh is None else dh.astype(np.float64))
    u = 2.0 ** -24 if dt == torch.float32 else 2.0 ** -53
    bn = np.linalg.norm(bh.astype(np.float64))
    assert np.linalg.norm(r) <= rtol * bn + 50 * u * bn
