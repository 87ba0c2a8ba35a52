"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs.  Bars:
  - elementwise: bit-exact (<= 1 ulp is the stated bound; 0 is the target)
  - integer reductions / scans, float max/min: bit-exact
  - float SUM (sum/dot/norm2): |gpu - oracle| <= max(tol_rel*|oracle|, n*u*sum|t_i|),
    tol_rel = 1e-5 (fp32 accumulation) / 1e-12 (fp64), u = 2^-24 / 2^-53,
    and the flat tol_rel*|oracle| clause is ALSO asserted alone (R10).
Sizes span several tiles plus ragged tails; offsets make unaligned views."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    import paper_1304_5553_b200 as ga
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"
SIZES = [1, 2, 3, 7, 31, 32, 33, 255, 256, 257, 4095, 4096, 4097, 8191, 8193, 65536 + 13,
         (1 << 20) - (1 << 18) + 5]
NPT = {np.float32: torch.float32, np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}


def to_dev(a, offset=0):
    """Copy numpy `a` to the GPU as a contiguous view starting `offset` elements
    into a fresh allocation (offset > 0 makes the view unaligned)."""
    buf = torch.empty(a.size + offset, dtype=NPT[a.dtype.type], device=DEV)
    v = buf[offset:]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


def host_data(dt, n, seed, signed=False, ints=(-1000, 1000)):
    if dt == np.float32:
        return synth.host_fill(synth.F32_S11 if signed else synth.F32_U01, seed, n)
    if dt == np.float64:
        return synth.host_fill(synth.F64_S11 if signed else synth.F64_U01, seed, n)
    if dt == np.int32:
        return synth.host_fill(synth.I32_RANGE, seed, n, lo=ints[0], hi=ints[1])
    return synth.host_fill(synth.I64_RANGE, seed, n, lo=ints[0], hi=ints[1])


def bits(a):
    a = np.asarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def assert_bit_exact(got, ref):
    assert got.dtype == ref.dtype and got.shape == ref.shape
    if got.dtype.kind == "f":
        nan = np.isnan(got) & np.isnan(ref)
        bad = (bits(got) != bits(ref)) & ~nan
    else:
        bad = got != ref
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(f"{int(bad.sum())} mismatches; first at {i}: gpu={got[i]!r} oracle={ref[i]!r}")


# ------------------------------------------------------------------ elementwise
@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32, np.int64])
@pytest.mark.parametrize("n", SIZES)
def test_axpbyz_bit_exact(dt, n):
    x = host_data(dt, n, 1, signed=True)
    y = host_data(dt, n, 2, signed=True)
    a, b = (5.0, -6.0) if np.dtype(dt).kind == "f" else (123457, -98765)
    z = ga.axpbyz(a, to_dev(x), b, to_dev(y)).cpu().numpy()
    assert_bit_exact(z, oracle.axpbyz(dt(a), x, dt(b), y))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_axpbyz_unfused_composition_equals_fused(dt):
    """The temporaries evaluation t = a*x; u = b*y; z = t + u (axpbz with
    b = -0.0, then axpbyz with unit coefficients; tools/fusion_bench.py) is
    bit-identical to the single pass (R1: RN(RN(a x) + RN(b y)))."""
    n = 1_000_003
    x, y = host_data(dt, n, 1, signed=True), host_data(dt, n, 2, signed=True)
    xd, yd = to_dev(x), to_dev(y)
    t = G.axpbz(5.0, xd, -0.0)
    u = G.axpbz(-6.0, yd, -0.0)
    z = G.axpbyz(1.0, t, 1.0, u).cpu().numpy()
    assert_bit_exact(z, oracle.axpbyz(dt(5.0), x, dt(-6.0), y))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("offs", [(1, 1, 1), (3, 3, 3), (7, 7, 7), (1, 2, 3), (0, 5, 0), (2, 0, 0)])
def test_axpbyz_unaligned_views(dt, offs):
    n = 10007
    x = host_data(dt, n, 1)
    y = host_data(dt, n, 2)
    out = torch.empty(n + offs[2], dtype=NPT[dt], device=DEV)[offs[2]:]
    G.axpbyz(5.7, to_dev(x, offs[0]), -1.25, to_dev(y, offs[1]), out=out)
    assert_bit_exact(out.cpu().numpy(), oracle.axpbyz(dt(5.7), x, dt(-1.25), y))


@pytest.mark.parametrize("dt", [np.float32, np.int64])
def test_axpbyz_inplace(dt):
    n = 70001
    x = host_data(dt, n, 1)
    y = host_data(dt, n, 2)
    xd, yd = to_dev(x), to_dev(y)
    ref = oracle.axpbyz(dt(3), x, dt(2), y)
    G.axpbyz(3, xd, 2, yd, out=xd)      # z == x
    assert_bit_exact(xd.cpu().numpy(), ref)
    xd = to_dev(x)
    G.axpbyz(3, xd, 2, yd, out=yd)      # z == y
    assert_bit_exact(yd.cpu().numpy(), ref)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32, np.int64])
@pytest.mark.parametrize("n", [1, 9, 4097, 65536 + 13])
def test_axpbz_bit_exact(dt, n):
    x = host_data(dt, n, 3, signed=True)
    a, b = (5.7, -0.3) if np.dtype(dt).kind == "f" else (-77, 12345)
    z = ga.axpbz(a, to_dev(x, 1), b).cpu().numpy()
    assert_bit_exact(z, oracle.axpbz(dt(a), x, dt(b)))


def test_listing1_doubling(golden):
    """Listing 1/2: 4x4 fp32 times two, incl. -0.0."""
    g = golden("listing1_doubling.json")
    x = np.array(g["input"], np.float32).ravel()
    z = ga.axpbz(2.0, to_dev(x), -0.0).cpu().numpy()
    assert_bit_exact(z, np.array(g["output"], np.float32).ravel())


def test_listing4_vector_add(golden):
    g = golden("listing4_vector_add.json")
    x, y, zr = (np.array(g[k], np.float32) for k in ("x", "y", "z"))
    assert_bit_exact(ga.axpbyz(1.0, to_dev(x), 1.0, to_dev(y)).cpu().numpy(), zr)


def test_elementwise_special_values():
    x = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0, 1e-45, 3.4e38, -3.4e38, 1.0], np.float32)
    y = np.array([1.0, np.inf, 2.0, -0.0, -0.0, 1e-45, 3.4e38, 3.4e38, np.nan], np.float32)
    z = ga.axpbyz(2.0, to_dev(x), 3.0, to_dev(y)).cpu().numpy()
    with np.errstate(all="ignore"):
        assert_bit_exact(z, oracle.axpbyz(np.float32(2), x, np.float32(3), y))


def test_elementwise_empty_and_errors():
    e = torch.empty(0, device=DEV)
    assert ga.axpbyz(1.0, e, 1.0, e).numel() == 0
    with pytest.raises(ValueError):
        ga.axpbyz(1.0, torch.ones(3, device=DEV), 1.0, torch.ones(4, device=DEV))
    with pytest.raises(TypeError):
        ga.axpbyz(1.0, torch.ones(3, device=DEV), 1.0, torch.ones(3, device=DEV, dtype=torch.float64))
    with pytest.raises(ValueError):
        ga.axpbyz(1.0, torch.ones(3), 1.0, torch.ones(3))  # CPU tensors: no CPU path
    buf = torch.ones(10, device=DEV)
    with pytest.raises(ValueError):  # partial overlap of z with x
        G.axpbyz(1.0, buf[0:8], 1.0, torch.ones(8, device=DEV), out=buf[1:9])


# ------------------------------------------------------------------ reductions
def float_tol(dt, n, ref, sumabs):
    rel, u = (1e-5, 2.0 ** -24) if dt == np.float32 else (1e-12, 2.0 ** -53)
    return max(rel * abs(ref), n * u * sumabs), rel * abs(ref)


@pytest.mark.parametrize("dt,odt", [(np.float32, np.float32), (np.float32, np.float64), (np.float64, np.float64)])
@pytest.mark.parametrize("mp", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
@pytest.mark.parametrize("n", [1, 2, 7, 33, 257, 4097, 65536 + 13, (1 << 20) - (1 << 18) + 5, 3_000_017])
@pytest.mark.parametrize("signed", [False, True])
def test_float_sum_within_tolerance(dt, odt, mp, n, signed):
    x = host_data(dt, n, 1, signed=signed)
    y = host_data(dt, n, 2, signed=signed)
    got = float(G.reduce(G.SUM, mp, to_dev(x), to_dev(y) if mp == G.MUL else None, out_dtype=NPT[odt]).item())
    ref, sa = oracle.reduce(oracle.SUM, mp, x, y, return_sumabs=True)
    tol, flat = float_tol(odt, n, ref, sa)
    assert abs(got - ref) <= tol
    if not signed:
        # no cancellation: the flat relative clause must hold on its own (R10)
        assert abs(got - ref) <= flat


@pytest.mark.parametrize("in_dt,out_dt", [(np.int32, np.int32), (np.int32, np.int64), (np.int64, np.int64)])
@pytest.mark.parametrize("mp", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
@pytest.mark.parametrize("n", [0, 1, 2, 255, 256, 257, 4097, 65536, 1_000_003])
def test_int_sum_bit_exact(in_dt, out_dt, mp, n):
    info = np.iinfo(in_dt)
    rng = np.random.default_rng(n)
    x = rng.integers(info.min, info.max, size=n, dtype=in_dt, endpoint=True)
    y = rng.integers(info.min, info.max, size=n, dtype=in_dt, endpoint=True)
    got = int(G.reduce(G.SUM, mp, to_dev(x, 1), to_dev(y, 3) if mp == G.MUL else None, out_dtype=NPT[out_dt]).item())
    assert got == oracle.reduce(oracle.SUM, mp, x, y, out_dtype=out_dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32, np.int64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
@pytest.mark.parametrize("mp", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 4097, 100_000, 1_000_003])
def test_maxmin_bit_exact(dt, op, mp, n):
    if np.dtype(dt).kind == "f":
        x = host_data(dt, n, 4, signed=True)
        y = host_data(dt, n, 5, signed=True)
    else:
        info = np.iinfo(dt)
        rng = np.random.default_rng(n + 7)
        x = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
        y = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    got = G.reduce(op, mp, to_dev(x), to_dev(y, 2) if mp == G.MUL else None).cpu().numpy()
    ref = oracle.reduce(op, mp, x, y)
    if np.dtype(dt).kind == "f":  # bit-exact, the sign of a zero extreme included (R7)
        assert np.array(got, dt).tobytes() == np.array(ref, dt).tobytes(), (got, ref)
    else:
        assert int(got) == ref


def test_maxmin_planted_and_nan():
    n = 1 << 20
    for pos in (0, n - 1, 123457):
        x = synth.host_fill(synth.F32_S11, 4, n)
        x[pos] = 7.0
        assert float(ga.max(to_dev(x)).item()) == 7.0
        x[pos] = -7.0
        assert float(ga.min(to_dev(x)).item()) == -7.0
    x = np.array([1, np.nan, 3, -2], np.float32)
    assert float(ga.max(to_dev(x)).item()) == 3.0
    assert float(ga.min(to_dev(x)).item()) == -2.0
    allnan = np.full(1000, np.nan, np.float32)
    assert float(ga.max(to_dev(allnan)).item()) == oracle.reduce(oracle.MAX, oracle.MAP_ID, allnan) == -np.inf


def test_reduce_spec_examples(golden):
    g = golden("dot_spec_example.json")
    assert float(ga.dot(to_dev(np.array(g["x"], np.float32)), to_dev(np.array(g["y"], np.float32))).item()) == g["dot"]
    g = golden("sum_1_to_8.json")
    assert int(ga.sum(to_dev(np.array(g["input"], np.int32))).item()) == g["sum"]
    g = golden("min_neutral_spec.json")
    assert int(ga.min(torch.empty(0, dtype=torch.int32, device=DEV)).item()) == g["empty_min"]
    x = to_dev(np.array(g["input"], np.int32))
    assert int(ga.min(x).item()) == g["min"] and int(ga.max(x).item()) == g["max"]


def test_reduce_closed_forms():
    n = 1 << 24
    ramp = torch.arange(1, n + 1, dtype=torch.float64, device=DEV)
    assert float(ga.sum(ramp).item()) == n * (n + 1) / 2
    twos = torch.full((1 << 20,), 2.0, device=DEV)
    r0 = torch.arange(0, 1 << 20, dtype=torch.float32, device=DEV)
    m = 1 << 20
    assert float(ga.dot(twos, r0).item()) == pytest.approx(m * (m - 1), rel=1e-6)
    assert float(ga.norm2sq(torch.ones(m, device=DEV)).item()) == m


def test_reduce_empty_is_neutral():
    e32 = torch.empty(0, device=DEV)
    assert float(ga.sum(e32).item()) == 0.0
    assert float(ga.max(e32).item()) == -np.inf
    assert float(ga.min(e32).item()) == np.inf
    assert int(ga.max(torch.empty(0, dtype=torch.int64, device=DEV)).item()) == -(1 << 63)


def test_reduce_deterministic_and_reusable():
    n = (1 << 24) + 11
    x = synth.device_fill(synth.F32_S11, 1, n, device=DEV)
    y = synth.device_fill(synth.F32_S11, 2, n, device=DEV)
    vals = {float(ga.dot(x, y).item()) for _ in range(5)}
    assert len(vals) == 1
    # different sizes back to back reuse the same workspace (epoch-tagged slots)
    for m in (5, 1 << 20, 3, n):
        xs = x[:m]
        xh = synth.host_fill(synth.F32_S11, 1, m)
        ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_ID, xh, None, return_sumabs=True)
        assert abs(float(ga.sum(xs).item()) - ref) <= float_tol(np.float32, m, ref, sa)[0]


def test_reduce_unsupported_combos():
    x = torch.ones(10, device=DEV)
    with pytest.raises(TypeError):
        G.reduce(G.MAX, G.ID, x, out_dtype=torch.float64)
    with pytest.raises(TypeError):
        G.reduce(G.SUM, G.ID, x, out_dtype=torch.int32)
    with pytest.raises(ValueError):
        G.reduce(G.SUM, G.MUL, x)


# ------------------------------------------------------------------ scan
SCAN_SIZES = [1, 2, 31, 32, 33, 2047, 2048, 2049, 4095, 4096, 4097, 3 * 4096 + 1, 65536 + 13, 1_000_003,
              (1 << 20) - (1 << 18) + 5]


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", SCAN_SIZES)
def test_scan_bit_exact(dt, exclusive, n):
    x = synth.host_fill(synth.I32_RANGE if dt == np.int32 else synth.I64_RANGE, 3, n, lo=-(1 << 20), hi=1 << 20)
    got = ga.scan(to_dev(x), exclusive=exclusive).cpu().numpy()
    assert_bit_exact(got, oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x))


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_scan_wraps_unaligned_inplace_carry(dt):
    info = np.iinfo(dt)
    rng = np.random.default_rng(5)
    n = 300_007
    x = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)   # wraps constantly
    for offs in (0, 1, 5):
        got = ga.scan(to_dev(x, offs)).cpu().numpy()
        assert_bit_exact(got, oracle.scan(oracle.INCLUSIVE, x))
    xd = to_dev(x)
    G.scan(xd, exclusive=True, out=xd)  # in place
    assert_bit_exact(xd.cpu().numpy(), oracle.scan(oracle.EXCLUSIVE, x))
    carry = np.array([info.max, 12345, -7], dt)
    with np.errstate(over="ignore"):
        c = dt(np.add.reduce(carry, dtype=dt))
    for ex in (False, True):
        got = G.scan(to_dev(x), exclusive=ex, carry=to_dev(carry)).cpu().numpy()
        assert_bit_exact(got, oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, x, carry=c))


def test_scan_spec_example_and_closed_forms(golden):
    g = golden("scan_spec_example.json")
    x = to_dev(np.array(g["input"], np.int32))
    assert ga.scan(x).cpu().tolist() == g["inclusive"]
    assert ga.scan(x, exclusive=True).cpu().tolist() == g["exclusive"]
    n = 5_000_011
    ones = torch.ones(n, dtype=torch.int32, device=DEV)
    assert torch.equal(ga.scan(ones), torch.arange(1, n + 1, dtype=torch.int32, device=DEV))
    assert torch.equal(ga.scan(ones, exclusive=True), torch.arange(0, n, dtype=torch.int32, device=DEV))


def test_scan_reduce_consistency_and_reuse():
    """Last inclusive element == reduce SUM; many calls of
    different sizes on one workspace (epoch tags, self-resetting counter)."""
    for n in (100_000, 3, 4096 * 50 + 7, 1, 100_000, 2_000_000):
        x = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=DEV)
        s = ga.scan(x)
        assert int(s[-1].item()) == int(ga.sum(x).item())
        xh = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=9)
        assert_bit_exact(s.cpu().numpy(), oracle.scan(oracle.INCLUSIVE, xh))


def test_scan_empty_and_errors():
    e = torch.empty(0, dtype=torch.int32, device=DEV)
    assert ga.scan(e).numel() == 0
    with pytest.raises(TypeError):
        ga.scan(torch.ones(4, device=DEV, dtype=torch.float16))  # dtype not supported
    with pytest.raises(ValueError):
        G.scan(torch.ones(4, device=DEV), op=7)  # bad scan expression


def test_launch_accounting():
    x = torch.ones(1000, device=DEV)
    c0 = ga.launch_count()
    ga.axpbyz(1.0, x, 1.0, x)
    ga.sum(x)
    ga.scan(torch.ones(1000, dtype=torch.int32, device=DEV))
    assert ga.launch_count() - c0 == 3


# ------------------------------------------------------------------ scan breadth (NEXT-2)
SCAN2_SIZES = [1, 33, 4097, 100_003, 1_000_003, (1 << 20) + 12345]


@pytest.mark.parametrize("dt", [np.int32, np.int64, np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", SCAN2_SIZES)
def test_scan_maxmin_bit_exact(dt, op, exclusive, n):
    if np.dtype(dt).kind == "f":
        x = host_data(dt, n, 6, signed=True)
    else:
        info = np.iinfo(dt)
        x = np.random.default_rng(n).integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
    kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
    for offs in (0, 1):  # aligned (super-tile kernel) and unaligned (register kernel)
        got = G.scan(to_dev(x, offs), exclusive=exclusive, op=op).cpu().numpy()
        assert_bit_exact(got, oracle.scan(kind, x, op=op))


def test_scan_maxmin_nan_carry_inplace():
    x = host_data(np.float32, 200_001, 7, signed=True)
    x[[0, 5000, 199_999]] = np.nan
    for op in (oracle.MAX, oracle.MIN):
        for ex in (False, True):
            c = np.array([0.5, -0.25], np.float32)
            cv = np.float32(max(c) if op == oracle.MAX else min(c))
            got = G.scan(to_dev(x), exclusive=ex, op=op, carry=to_dev(c)).cpu().numpy()
            assert_bit_exact(got, oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, x, op=op, carry=cv))
    xd = to_dev(x)
    G.scan(xd, op=oracle.MAX, out=xd)
    assert_bit_exact(xd.cpu().numpy(), oracle.scan(oracle.INCLUSIVE, x, op=oracle.MAX))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("exclusive", [False, True])
def test_scan_float_sum_small_integers_exact(dt, exclusive):
    """Integer-valued floats whose prefix sums stay below 2^24 (fp32) are
    summed exactly in any order: the float SUM scan must equal the integer
    oracle bit for bit (catches a dropped, doubled or misplaced element)."""
    n = 1_500_007  # 9 * n < 2^24
    k = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=9)
    x = k.astype(dt)
    ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, k).astype(dt)
    for offs in (0, 3):
        got = G.scan(to_dev(x, offs), exclusive=exclusive).cpu().numpy()
        assert_bit_exact(got, ref)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", [1, 4097, 1_000_003])
def test_scan_float_sum_within_bound(dt, exclusive, n):
    """Random signed data: |gpu_i - S_i| <= d_i * u * (|c| + sum_{j<=i}|x_j|)
    with S_i the exact prefix sum and d_i = i/2048 + 512 (R22: the look-back
    chains tile prefixes serially, the in-tile tree is shallow)."""
    x = host_data(dt, n, 8, signed=True)
    u = 2.0 ** -24 if dt == np.float32 else 2.0 ** -53
    kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
    ref, sa = oracle.scan(kind, x, return_sumabs=True)
    for offs in (0, 1):
        got = G.scan(to_dev(x, offs), exclusive=exclusive).cpu().numpy().astype(np.float64)
        d = np.arange(n) / 2048.0 + 512
        assert np.all(np.abs(got - ref) <= d * u * sa + 1e-300)


# ------------------------------------------------------------------ scan super-tile shapes
# (scan_impl.cuh: L when it gives >= 256 tiles, else M when >= 64, else S;
# tiles of 24x32 / 32x8 / 8x8 (16x8 for 8-byte T) rows of 512 input bytes)
def _shape_sizes(isz, osz):
    tile = {"S": (16 if osz == 8 else 8) * 8 * 512 // isz, "M": 32 * 8 * 512 // isz, "L": 24 * 32 * 512 // isz}
    return [64 * tile["M"] - 1, 64 * tile["M"] + 77, 256 * tile["L"] - 3, 256 * tile["L"] + 1001]


@pytest.mark.parametrize("pair", [(np.int32, np.int32), (np.int64, np.int64), (np.int32, np.int64)])
@pytest.mark.parametrize("exclusive", [False, True])
def test_scan_shape_boundaries(pair, exclusive):
    """Sizes either side of the S/M and M/L switch points, wrapping data."""
    tin, tout = pair
    kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
    for n in _shape_sizes(np.dtype(tin).itemsize, np.dtype(tout).itemsize):
        info = np.iinfo(tin)
        x = np.random.default_rng(n).integers(info.min, info.max, size=n, dtype=tin, endpoint=True)
        got = G.scan(to_dev(x), exclusive=exclusive, out_dtype=NPT[tout]).cpu().numpy()
        assert_bit_exact(got, oracle.scan(kind, x, out_dtype=tout))


# ------------------------------------------------------------------ widening scans (NEXT-2, R27)
@pytest.mark.parametrize("op", [oracle.SUM, oracle.MAX, oracle.MIN])
@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", SCAN2_SIZES)
def test_scan_widen_i32_i64_bit_exact(op, exclusive, n):
    """int32 -> int64 scans: full-range data whose int32 SUM scan would wrap;
    super-tile kernel (aligned), register kernel (unaligned input, and an
    output that is 16- but not 32-byte aligned)."""
    x = np.random.default_rng(n + 17).integers(-(1 << 31), (1 << 31) - 1, size=n, dtype=np.int32, endpoint=True)
    kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
    ref = oracle.scan(kind, x, op=op, out_dtype=np.int64)
    for offs, out_offs in ((0, 0), (1, 0), (0, 2)):
        out = torch.empty(n + out_offs, dtype=torch.int64, device=DEV)[out_offs:]
        got = G.scan(to_dev(x, offs), exclusive=exclusive, op=op, out=out, out_dtype=torch.int64)
        assert_bit_exact(got.cpu().numpy(), ref)


def test_scan_widen_i32_i64_carry_and_errors():
    n = 1_000_003
    x = np.full(n, np.iinfo(np.int32).max, np.int32)
    carry = np.array([-(1 << 40), 7], np.int64)
    got = G.scan(to_dev(x), exclusive=True, carry=to_dev(carry), out_dtype=torch.int64).cpu().numpy()
    assert_bit_exact(got, oracle.scan(oracle.EXCLUSIVE, x, carry=np.int64(-(1 << 40) + 7), out_dtype=np.int64))
    assert int(got[-1]) == (n - 1) * (2 ** 31 - 1) - (1 << 40) + 7  # closed form, no wrap
    xd = to_dev(x)
    with pytest.raises(TypeError):
        G.scan(xd, carry=to_dev(np.zeros(1, np.int32)), out_dtype=torch.int64)  # carry is out_dtype
    with pytest.raises(TypeError):
        G.scan(to_dev(x.astype(np.int64)), out_dtype=torch.int32)               # narrowing
    with pytest.raises(ValueError):
        G.scan(xd, out=torch.empty(n - 1, dtype=torch.int64, device=DEV), out_dtype=torch.int64)  # length


@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", [1, 4097, 1_000_003])
def test_scan_widen_f32_f64_within_bound(exclusive, n):
    """float32 -> float64 SUM scans: the f64 bound of R22 on the exact prefix
    sums of the fp32 inputs; MAX/MIN bit-exact."""
    x = host_data(np.float32, n, 8, signed=True)
    kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
    ref, sa = oracle.scan(kind, x, return_sumabs=True, out_dtype=np.float64)
    d = np.arange(n) / 2048.0 + 512
    for offs in (0, 1):
        got = G.scan(to_dev(x, offs), exclusive=exclusive, out_dtype=torch.float64).cpu().numpy()
        assert got.dtype == np.float64
        assert np.all(np.abs(got - ref) <= d * 2.0 ** -53 * sa + 1e-300)
        for op in (oracle.MAX, oracle.MIN):
            g2 = G.scan(to_dev(x, offs), exclusive=exclusive, op=op, out_dtype=torch.float64).cpu().numpy()
            assert_bit_exact(g2, oracle.scan(kind, x, op=op, out_dtype=np.float64))


# ------------------------------------------------------------------ complex (NEXT-3)
CPLX = {np.complex64: torch.complex64, np.complex128: torch.complex128}


def cplx_data(dt, n, seed):
    f = synth.F32_S11 if dt == np.complex64 else synth.F64_S11
    return synth.host_fill(f, seed, 2 * n).view(dt)


def to_dev_c(a, offset=0):
    buf = torch.empty(a.size + offset, dtype=CPLX[a.dtype.type], device=DEV)
    v = buf[offset:]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("n", [1, 3, 4097, 100_003])
@pytest.mark.parametrize("offs", [0, 1])
def test_complex_axpbyz_bit_exact(dt, n, offs):
    x = cplx_data(dt, n, 1)
    y = cplx_data(dt, n, 2)
    a, b = 1.5 - 2.25j, -0.75 + 0.5j
    z = ga.axpbyz(a, to_dev_c(x, offs), b, to_dev_c(y, offs)).cpu().numpy()
    ref = oracle.axpbyz_complex(dt(a), x, dt(b), y)
    f = np.float32 if dt == np.complex64 else np.float64
    assert_bit_exact(z.view(f), ref.view(f))
    # axpbz(a, x, b) == axpbyz(a, x, b, 1) on nonzero data
    zb = ga.axpbz(a, to_dev_c(x), b).cpu().numpy()
    assert_bit_exact(zb.view(f), oracle.axpbyz_complex(dt(a), x, dt(b), np.ones_like(x)).view(f))


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("n", [1, 257, 100_003, 2_000_003])
def test_complex_sum_dot_vdot_norm2(dt, n):
    x = cplx_data(dt, n, 3)
    y = cplx_data(dt, n, 4)
    u, rel = (2.0 ** -24, 1e-5) if dt == np.complex64 else (2.0 ** -53, 1e-12)
    xd, yd = to_dev_c(x), to_dev_c(y, 1)
    for name, got, mp in (("sum", G.sum(xd), oracle.MAP_ID), ("dot", G.dot(xd, to_dev_c(y)), oracle.MAP_MUL),
                          ("vdot", G.vdot(xd, to_dev_c(y)), oracle.MAP_CONJ_MUL)):
        ref, sa = oracle.reduce_complex(mp, x, y, return_sumabs=True)
        g = complex(got.item())
        assert abs(g - ref) <= max(rel * abs(ref), 2 * n * u * sa), name
    n2 = G.norm2sq(xd)
    assert n2.dtype == (torch.float32 if dt == np.complex64 else torch.float64)
    ref = oracle.reduce_complex(oracle.MAP_SQUARE, x)
    assert abs(float(n2.item()) - ref) <= rel * ref
    # unaligned y (offset 1 element) takes the scalar path
    g = complex(G.vdot(xd, yd).item())
    ref, sa = oracle.reduce_complex(oracle.MAP_CONJ_MUL, x, y, return_sumabs=True)
    assert abs(g - ref) <= max(rel * abs(ref), 2 * n * u * sa)


def test_complex_closed_forms_and_errors():
    n = 1 << 20
    ones = torch.ones(n, dtype=torch.complex64, device=DEV)
    i_ = torch.full((n,), 1j, dtype=torch.complex64, device=DEV)
    assert complex(G.dot(i_, i_).item()) == -n          # i*i = -1
    assert complex(G.vdot(i_, i_).item()) == n          # conj(i)*i = 1
    assert float(G.norm2sq(i_ + ones).item()) == 2 * n  # |1+i|^2 = 2
    with pytest.raises(TypeError):
        G.max(ones)
    with pytest.raises(TypeError):
        G.scan(ones)


# ------------------------------------------------------------------ operators / cumath maps (NEXT-2)
EW_EXACT = [oracle.EW_MUL, oracle.EW_DIV, oracle.EW_SQRT, oracle.EW_ABS, oracle.EW_NEG, oracle.EW_MAX, oracle.EW_MIN]
EW_LIBM = [oracle.EW_EXP, oracle.EW_LOG, oracle.EW_SIN, oracle.EW_COS]


def ulp_dist(a, b):
    it = np.int32 if a.dtype == np.float32 else np.int64
    ka, kb = a.view(it).astype(np.int64), b.view(it).astype(np.int64)
    ka = np.where(ka < 0, np.iinfo(it).min - ka, ka)  # monotone key for sign-magnitude floats
    kb = np.where(kb < 0, np.iinfo(it).min - kb, kb)
    d = np.abs(ka - kb)
    both_nan = np.isnan(a) & np.isnan(b)
    return np.where(both_nan, 0, d)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 33, 4097, 1_000_003])
def test_ewmap_float(dt, n):
    x = host_data(dt, n, 1, signed=True) * dt(8)
    y = host_data(dt, n, 2, signed=True) + dt(1.5)
    ax = np.abs(x) + dt(1e-3)
    for op in EW_EXACT + EW_LIBM:
        arg = ax if op in (oracle.EW_SQRT, oracle.EW_LOG) else x
        with np.errstate(all="ignore"):
            ref = oracle.ewmap(op, arg, y)
        for offs in (0, 1):
            got = G.elementwise(op, to_dev(arg, offs), to_dev(y, offs) if op in G._BINARY else None).cpu().numpy()
            if op in EW_EXACT:
                assert_bit_exact(got, ref)
            else:  # R26: CUDA accurate functions vs glibc
                assert ulp_dist(got, ref).max() <= 3, (op, int(ulp_dist(got, ref).max()))


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_ewmap_int(dt):
    info = np.iinfo(dt)
    rng = np.random.default_rng(9)
    x = rng.integers(info.min, info.max, size=100_003, dtype=dt, endpoint=True)
    y = rng.integers(info.min, info.max, size=100_003, dtype=dt, endpoint=True)
    x[5] = info.min
    for op in (oracle.EW_MUL, oracle.EW_ABS, oracle.EW_NEG, oracle.EW_MAX, oracle.EW_MIN):
        got = G.elementwise(op, to_dev(x), to_dev(y) if op in G._BINARY else None).cpu().numpy()
        assert_bit_exact(got, oracle.ewmap(op, x, y))
    with pytest.raises(TypeError):
        G.divide(to_dev(x), to_dev(y))   # integer division is not instantiated


def test_ewmap_special_values_and_inplace():
    x = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 1e-40, 4.0], np.float32)
    with np.errstate(all="ignore"):
        for op in (oracle.EW_SQRT, oracle.EW_LOG, oracle.EW_EXP, oracle.EW_ABS, oracle.EW_NEG):
            got = G.elementwise(op, to_dev(x)).cpu().numpy()
            ref = oracle.ewmap(op, x)
            assert ulp_dist(got, ref).max() <= (0 if op in EW_EXACT else 3), op
    xd = to_dev(x[np.isfinite(x)])
    G.sqrt(G.fabs(xd, out=xd), out=xd)
    with np.errstate(all="ignore"):
        assert_bit_exact(xd.cpu().numpy(), np.sqrt(np.abs(x[np.isfinite(x)])))


# ------------------------------------------------------------ signed zeros and NaN in MAX / MIN (R6, R7)
def zeros_heavy(dt, n, seed):
    """Values from {-0, +0, -1, +1, NaN, -tiny, +tiny} with many signed zeros:
    every max/min tie is a +-0 tie, which only R7's -0 < +0 decides."""
    rng = np.random.default_rng(seed)
    tiny = np.finfo(dt).tiny
    pool = np.array([-0.0, 0.0, -0.0, 0.0, -1.0, 1.0, np.nan, -tiny, tiny], dtype=dt)
    return pool[rng.integers(0, pool.size, size=n)]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
@pytest.mark.parametrize("mp", [oracle.MAP_ID, oracle.MAP_MUL])
@pytest.mark.parametrize("n", [3, 4097, 300_001])
@pytest.mark.parametrize("only_zeros", [False, True])
def test_maxmin_signed_zero_bit_exact(dt, op, mp, n, only_zeros):
    """Bit-exact max/min over data whose extreme is a signed zero (only_zeros:
    nothing but -0 and +0, so the result is +0 for MAX and -0 for MIN whenever
    both occur, whatever the tree order)."""
    x = zeros_heavy(dt, n, n + op)
    y = zeros_heavy(dt, n, n + 11)
    if only_zeros:
        x = np.where(np.arange(n) % 3 == 0, dt(0.0), dt(-0.0)).astype(dt)
        y = np.where(np.arange(n) % 5 == 0, dt(-1.0), dt(1.0)).astype(dt)
    got = G.reduce(op, mp, to_dev(x), to_dev(y) if mp == G.MUL else None).cpu().numpy()
    ref = oracle.reduce(op, mp, x, y)
    assert np.array(got, dt).tobytes() == np.array(ref, dt).tobytes(), (got, ref)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
@pytest.mark.parametrize("exclusive", [False, True])
@pytest.mark.parametrize("n", [5, 70_001, 3_000_017])
def test_scan_maxmin_signed_zero_bit_exact(dt, op, exclusive, n):
    x = zeros_heavy(dt, n, 3 * n + op)
    got = G.scan(to_dev(x), exclusive=exclusive, op=op).cpu().numpy()
    ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, op=op)
    assert np.array_equal(bits(got), bits(ref))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_ewmap_maxmin_signed_zero_bit_exact(dt):
    n = 100_003
    x, y = zeros_heavy(dt, n, 21), zeros_heavy(dt, n, 22)
    for ew, op in ((oracle.EW_MAX, G._abi.GA_EW_MAX), (oracle.EW_MIN, G._abi.GA_EW_MIN)):
        got = G.elementwise(op, to_dev(x), to_dev(y)).cpu().numpy()
        ref = oracle.ewmap(ew, x, y)
        # max(NaN, NaN) is NaN on both sides; payloads compare as a class (R8)
        assert np.array_equal(np.isnan(got), np.isnan(ref)), ew
        keep = ~np.isnan(ref)
        assert np.array_equal(bits(got[keep]), bits(ref[keep])), ew


# 8-byte scans reach the L shape above the ring window (2 GiB of input) or,
# from 96 MiB, when the output is 16- but not 32-byte aligned (the ring's
# 1 KiB rows store 32 bytes per lane)
N_L8 = (768 << 20) // 8 + 12345
N_L8A = (2 << 30) // 8 + 12345


@pytest.mark.parametrize("dt", [np.int64, np.float64])
@pytest.mark.parametrize("offset", [0, 2])
def test_scan_8byte_l_shape_both_row_widths(dt, offset):
    """8-byte scans at the L shape take 1 KiB rows (LDG/STG.256) when input and
    output are 32-byte aligned (past 2 GiB here), else 512-byte rows: a view
    2 elements (16 bytes) into an allocation exercises the second path.
    Integer scans are exact; float64 SUM over integer-valued data (prefix
    sums < 2^53) is exact in any order and must equal the integer oracle bit
    for bit."""
    n = N_L8A if offset == 0 else N_L8  # ragged last tile
    if dt == np.int64:
        x = np.random.default_rng(offset + 5).integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    else:
        k = synth.host_fill(synth.I32_RANGE, 9, n, lo=0, hi=9)
        x = k.astype(np.float64)
    for exclusive in (False, True):
        kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
        got = G.scan(to_dev(x, offset), exclusive=exclusive).cpu().numpy()
        if dt == np.int64:
            assert np.array_equal(got, oracle.scan(kind, x))
        else:
            assert_bit_exact(got, oracle.scan(kind, k, out_dtype=np.int64).astype(np.float64))


@pytest.mark.parametrize("offset", [0, 2])
@pytest.mark.parametrize("n", [300 * 24 * 32 * 64 + 4097, N_L8A])
def test_scan_int64_l_shape_in_place(offset, n):
    """In-place int64 scans: 118 MB (offset 0: the ring kernel; offset 2
    elements = 16 bytes: the L shape with 512-byte rows) and past 2 GiB (the
    L shape, 1 KiB rows at offset 0): coherent loads (the output overwrites
    the input) on every path."""
    x = np.random.default_rng(77 + offset).integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    for exclusive in (False, True):
        d = to_dev(x, offset)
        G.scan(d, exclusive=exclusive, out=d)
        ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x)
        assert np.array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("dt", [np.int64, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
def test_scan_maxmin_8byte_l_shape(dt, op):
    """MAX / MIN scans of 8-byte types at the L shape (1 KiB rows), inclusive
    and exclusive, bit-exact — float64 data zero- and NaN-heavy (R6, R7)."""
    n = N_L8A - 12345 + 999  # past the ring window: the L shape, 1 KiB rows
    if dt == np.int64:
        x = np.random.default_rng(op + 3).integers(-(1 << 62), 1 << 62, size=n, dtype=np.int64)
    else:
        x = zeros_heavy(dt, n, op + 4)
        x[np.random.default_rng(op).integers(0, n, size=64)] = np.random.default_rng(1).standard_normal(64)
    for exclusive in (False, True):
        got = G.scan(to_dev(x), exclusive=exclusive, op=op).cpu().numpy()
        ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, op=op)
        assert np.array_equal(bits(got), bits(ref))


# ------------------------------------------------------------------ ring scan (scan_ring.cuh)
# 16-byte aligned scans of 48 MiB .. 4 GiB (4-byte) / 2 GiB (8-byte, with a
# 32-byte aligned output) of input, and widening scans from 48 MiB, take the
# single-touch ring kernel: 64 KiB tiles (16384 / 8192 elements), persistent
# CTAs, TMA stages, non-widening tiles prefetched into L2 one draw ahead,
# 1 KiB rows for 8-byte types, a ragged tail read element by element past
# the last 16-byte multiple.  (The 4-byte upper edge, n = 2^30,
# is C3's size: test_parity_full_gpu compares that scan whole; the L shape
# beyond it is C5's 2^33 scan, also compared whole.)
RING_MIN = 48 << 20
RING_MAX = {4: 4 << 30, 8: 2 << 30}


def _ring_data(dt, op, n, seed):
    if np.dtype(dt).kind == "f":
        if op == oracle.SUM:  # indicator data: every prefix sum is an integer < 2^24, exact in any order
            return (synth.host_fill(synth.I32_RANGE, seed, n, lo=0, hi=7) == 0).astype(dt)
        x = zeros_heavy(dt, n, seed)
        x[np.random.default_rng(seed).integers(0, n, size=256)] = np.nan
        return x
    info = np.iinfo(dt)
    return np.random.default_rng(seed).integers(info.min, info.max, size=n, dtype=dt, endpoint=True)


@pytest.mark.parametrize("dt", [np.int32, np.int64, np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.SUM, oracle.MAX, oracle.MIN])
def test_scan_ring_every_op_and_dtype(dt, op):
    """Every (op, dtype, kind) of the ring kernel against the oracle, bit for
    bit: full-range integers (SUM wraps constantly), 0/1 floats (float SUM
    exact in any order), zero- and NaN-heavy float MAX / MIN (R6, R7);
    ragged last tile."""
    n = (64 << 20) // np.dtype(dt).itemsize + 12345
    x = _ring_data(dt, op, n, 40 + op)
    for exclusive in (False, True):
        kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
        got = G.scan(to_dev(x), exclusive=exclusive, op=op).cpu().numpy()
        if np.dtype(dt).kind == "f" and op == oracle.SUM:
            ref = oracle.scan(kind, x.astype(np.int64)).astype(dt)
        else:
            ref = oracle.scan(kind, x, op=op)
        assert_bit_exact(got, ref)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_scan_ring_float_sum_within_bound(dt):
    """Signed random data in the ring window: R22's bound on the exact
    prefix sums (the ring chains 64 KiB tile prefixes through the look-back;
    inside a tile: lane-serial 16-byte chunks, warp shuffle scans, rows and
    warps in order)."""
    n = RING_MIN // np.dtype(dt).itemsize + 4099
    x = host_data(dt, n, 12, signed=True)
    u = 2.0 ** -24 if dt == np.float32 else 2.0 ** -53
    d = np.arange(n) / 2048.0 + 512
    for exclusive in (False, True):
        ref, sa = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, return_sumabs=True)
        got = G.scan(to_dev(x), exclusive=exclusive).cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= d * u * sa + 1e-300)


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_scan_ring_window_edges(dt):
    """Sizes either side of the ring window (M shape | ring | ring | L shape;
    int32: the lower edge only, its upper edge is C3's full-size scan) and
    tails of 1-3 elements past a 16-byte multiple, inclusive and exclusive,
    wrapping data."""
    isz = np.dtype(dt).itemsize
    te = 65536 // isz
    lo, hi = RING_MIN // isz, RING_MAX[isz] // isz
    info = np.iinfo(dt)
    for n in (lo - 1, lo, lo + 1, 1000 * te + 3) + ((hi, hi + 1) if isz == 8 else ()):
        x = np.random.default_rng(n).integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
        for exclusive in ((False, True) if n < hi else (False,)):
            kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
            got = G.scan(to_dev(x), exclusive=exclusive).cpu().numpy()
            assert_bit_exact(got, oracle.scan(kind, x))


@pytest.mark.parametrize("dt", [np.int32, np.int64, np.float32])
def test_scan_ring_carry_inplace_and_views(dt):
    """Ring-window sizes with a carry-in (tile 0 publishes carry (+) aggregate),
    in place, and as a view 16 bytes into its allocation (4-byte: still the
    ring kernel; 8-byte: the two-touch M/L shapes, the ring's 1 KiB rows
    needing a 32-byte aligned output) or 1 element in (the unaligned
    register kernel)."""
    isz = np.dtype(dt).itemsize
    n = (96 << 20) // isz + 5
    if np.dtype(dt).kind == "f":
        x = synth.host_fill(synth.I32_RANGE, 51, n, lo=-4, hi=4).astype(dt)  # |prefix| stays < 2^24: exact
        carry = np.array([3.0, -1.0], dt)
        c = dt(2.0)
    else:
        info = np.iinfo(dt)
        x = np.random.default_rng(51).integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
        carry = np.array([info.max, 12345, -7], dt)
        with np.errstate(over="ignore"):
            c = dt(np.add.reduce(carry, dtype=dt))
    def same(got, ref):  # the float oracle returns exact float64 sums (integers < 2^24 here)
        if np.dtype(dt).kind == "f":
            assert np.array_equal(got.astype(np.float64), ref)
        else:
            assert_bit_exact(got, ref)

    for ex in (False, True):
        kind = oracle.EXCLUSIVE if ex else oracle.INCLUSIVE
        got = G.scan(to_dev(x), exclusive=ex, carry=to_dev(carry)).cpu().numpy()
        same(got, oracle.scan(kind, x, carry=c))
        xd = to_dev(x)
        G.scan(xd, exclusive=ex, out=xd)
        same(xd.cpu().numpy(), oracle.scan(kind, x))
        for offs in (16 // isz, 1):
            got = G.scan(to_dev(x, offs), exclusive=ex).cpu().numpy()
            same(got, oracle.scan(kind, x))


@pytest.mark.parametrize("op", [oracle.SUM, oracle.MAX, oracle.MIN])
def test_scan_ring_widening(op):
    """Widening scans of >= 48 MiB of input take the ring kernel (8-byte scan
    type, 32-byte stores per lane): int32 -> int64 full-range data bit-exact
    (no int32 wrap), float32 -> float64 MAX / MIN bit-exact and SUM within
    R22 with u = 2^-53; the 32-byte-aligned output rule (a 16-byte output
    offset goes to the register kernel); carry-in."""
    n = RING_MIN // 4 + 4099
    x = np.random.default_rng(60 + op).integers(-(1 << 31), (1 << 31) - 1, size=n, dtype=np.int32, endpoint=True)
    for exclusive in (False, True):
        kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
        ref = oracle.scan(kind, x, op=op, out_dtype=np.int64)
        for out_offs in (0, 2):
            out = torch.empty(n + out_offs, dtype=torch.int64, device=DEV)[out_offs:]
            got = G.scan(to_dev(x), exclusive=exclusive, op=op, out=out, out_dtype=torch.int64)
            assert_bit_exact(got.cpu().numpy(), ref)
    f = host_data(np.float32, n, 61, signed=True)
    d = np.arange(n) / 2048.0 + 512
    for exclusive in (False, True):
        kind = oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE
        got = G.scan(to_dev(f), exclusive=exclusive, op=op, out_dtype=torch.float64).cpu().numpy()
        if op == oracle.SUM:
            ref, sa = oracle.scan(kind, f, return_sumabs=True, out_dtype=np.float64)
            assert np.all(np.abs(got - ref) <= d * 2.0 ** -53 * sa + 1e-300)
        else:
            assert_bit_exact(got, oracle.scan(kind, f, op=op, out_dtype=np.float64))
    if op == oracle.SUM:
        carry = np.array([-(1 << 40), 7], np.int64)
        got = G.scan(to_dev(x), exclusive=True, carry=to_dev(carry), out_dtype=torch.int64).cpu().numpy()
        assert_bit_exact(got, oracle.scan(oracle.EXCLUSIVE, x, carry=np.int64(-(1 << 40) + 7), out_dtype=np.int64))


@pytest.mark.parametrize("dt,out_dt", [(np.int32, np.int32), (np.int64, np.int64), (np.int32, np.int64),
                                       (np.float32, np.float32)])
def test_scan_guard_bands_every_path(dt, out_dt):
    """Out-of-bounds write check (compute-sanitizer being unavailable on the
    GPU pool): the output of every scan path (S, M, ring, L shape, register
    kernel) sits between 4 KiB guard bands filled with a sentinel, at ragged
    sizes and 16-byte-aligned and unaligned views, in place and out of place;
    the bands must come back untouched and the results must match the
    oracle (float: integer-valued data, exact)."""
    isz, osz = np.dtype(dt).itemsize, np.dtype(out_dt).itemsize
    pad = 4096 // osz
    sizes = [4097, 3_000_017, (64 << 20) // isz + 3]           # S / M / ring
    if isz == 8 and osz == 8:
        sizes.append((768 << 20) // 8 + 5)                      # L shape (8-byte)
    for n in sizes:
        if np.dtype(dt).kind == "f":
            x = synth.host_fill(synth.I32_RANGE, n % 97, n, lo=0, hi=1).astype(dt)
        else:
            x = synth.host_fill(synth.I32_RANGE if dt == np.int32 else synth.I64_RANGE, n % 97, n,
                                lo=-(1 << 20), hi=1 << 20)
        ref = oracle.scan(oracle.EXCLUSIVE, x, out_dtype=None if dt == out_dt else out_dt)
        if np.dtype(dt).kind == "f":
            ref = oracle.scan(oracle.EXCLUSIVE, x.astype(np.int64)).astype(out_dt)
        for offs in (0, 16 // osz, 1):
            buf = torch.full((n + 2 * pad + offs,), 0x5A5A5A5A, dtype=NPT[out_dt], device=DEV)
            out = buf[pad + offs:pad + offs + n]
            G.scan(to_dev(x, offs), exclusive=True, out=out, out_dtype=NPT[out_dt])
            b = buf.cpu().numpy()
            assert np.all(b[:pad + offs] == np.array(0x5A5A5A5A).astype(out_dt)), (n, offs, "head band")
            assert np.all(b[pad + offs + n:] == np.array(0x5A5A5A5A).astype(out_dt)), (n, offs, "tail band")
            assert_bit_exact(b[pad + offs:pad + offs + n], ref)
        if dt == out_dt:  # in place, inside guard bands
            buf = torch.full((n + 2 * pad,), 0x5A5A5A5A, dtype=NPT[dt], device=DEV)
            v = buf[pad:pad + n]
            v.copy_(torch.from_numpy(x))
            G.scan(v, exclusive=True, out=v)
            b = buf.cpu().numpy()
            assert np.all(b[:pad] == np.array(0x5A5A5A5A).astype(dt)) and \
                np.all(b[pad + n:] == np.array(0x5A5A5A5A).astype(dt)), (n, "in-place bands")
            assert_bit_exact(b[pad:pad + n], ref)
