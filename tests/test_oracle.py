"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
numpy's uncontracted arithmetic, math.fsum, fractions.Fraction brute force,
Python big-int arithmetic, closed forms and the worked values of SPEC.md /
the paper's listings (tests/golden/).  Each test names the plausible oracle
mistake it would catch.  CPU only (no GPU marker)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

RNG = np.random.default_rng(1304_5553)


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    if a.dtype.kind == "f":
        ia = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
        ib = b.view(ia.dtype)
        both_nan = np.isnan(a) & np.isnan(b)
        return bool(np.all((ia == ib) | both_nan))
    return bool(np.array_equal(a, b))


# ---------------------------------------------------------------- elementwise
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("ab", [(5.0, 6.0), (5.0, -6.0), (5.7, -1.25), (1.0, -1.0)])
def test_axpbyz_float_matches_numpy_uncontracted(dt, ab):
    """R1: RN(RN(a*x)+RN(b*y)).  numpy evaluates (A*x)+(B*y) op by op with no
    FMA contraction; a contracted (fma) or double-rounded oracle differs by up
    to 4.2M ulp under the a=5,b=-6 cancellation (SURVEY PROBE-4)."""
    n = 1 << 16
    kx, ky = (synth.F32_U01, synth.F32_U01) if dt == np.float32 else (synth.F64_U01, synth.F64_U01)
    x = synth.host_fill(kx, 1, n)
    y = synth.host_fill(ky, 2, n)
    a, b = dt(ab[0]), dt(ab[1])
    ref = (a * x) + (b * y)
    assert ref.dtype == dt
    assert bits_equal(oracle.axpbyz(a, x, b, y), ref)


def test_axpbyz_fma_would_be_caught():
    """The cancellation data really separates fma(a,x,RN(b*y)) from R1."""
    n = 1 << 16
    x = synth.host_fill(synth.F32_U01, 1, n).astype(np.float64)
    y = synth.host_fill(synth.F32_U01, 2, n).astype(np.float64)
    # fma(a,x,RN32(b*y)) computed exactly in f64 then rounded once to f32
    by = (np.float32(-6.0) * y.astype(np.float32)).astype(np.float64)
    fused = (5.0 * x + by).astype(np.float32)  # a*x exact in f64, one rounding
    z = oracle.axpbyz(np.float32(5), x.astype(np.float32), np.float32(-6), y.astype(np.float32))
    assert not bits_equal(z, fused)


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_axpbyz_int_wraps_like_numpy(dt):
    """R4: integer overflow wraps mod 2^w (numpy integer arithmetic wraps)."""
    info = np.iinfo(dt)
    x = RNG.integers(info.min, info.max, size=4097, dtype=dt, endpoint=True)
    y = RNG.integers(info.min, info.max, size=4097, dtype=dt, endpoint=True)
    a, b = dt(123457), dt(-98765)
    with np.errstate(over="ignore"):
        ref = (a * x) + (b * y)
    assert bits_equal(oracle.axpbyz(a, x, b, y), ref)
    # big-int check of a few elements (independent of numpy's wrap)
    w = np.dtype(dt).itemsize * 8
    for i in (0, 1, 4096):
        v = (int(a) * int(x[i]) + int(b) * int(y[i])) % (1 << w)
        v = v - (1 << w) if v >= (1 << (w - 1)) else v
        assert int(oracle.axpbyz(a, x[i:i + 1], b, y[i:i + 1])[0]) == v


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_axpbyz_closed_forms(dt):
    x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 7, 1000)
    y = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 8, 1000)
    # a=b=1, y=x -> 2x exactly (catches using y where x is meant and vice versa... with y != x below)
    assert bits_equal(oracle.axpbyz(1, x, 1, x), x * dt(2))
    # a=1, b=0 -> x (+0.0 added; x has no -0.0)
    assert bits_equal(oracle.axpbyz(1, x, 0, y), x)
    # a=0, b=1 -> y  (catches swapped operands)
    assert bits_equal(oracle.axpbyz(0, x, 1, y), y)
    # a=2, b=-1 on y = x -> x exactly
    assert bits_equal(oracle.axpbyz(2, x, -1, x), x)


def test_listing1_doubling(golden):
    """Listing 1 / Listing 2: a 4x4 fp32 array times two (PAPER.md:245-249,
    364-368).  `a *= 2` is axpbz with b = -0.0, the IEEE additive identity
    (R21), so -0.0 doubles to -0.0."""
    g = golden("listing1_doubling.json")
    x = np.array(g["input"], dtype=np.float32).ravel()
    ref = np.array(g["output"], dtype=np.float32).ravel()
    assert bits_equal(oracle.axpbz(2, x, -0.0), ref)
    assert bits_equal(oracle.axpbyz(2, x, 0, np.zeros_like(x))[x != 0], ref[x != 0])


def test_listing4_vector_add(golden):
    g = golden("listing4_vector_add.json")
    x, y, z = (np.array(g[k], dtype=np.float32) for k in ("x", "y", "z"))
    assert bits_equal(oracle.axpbyz(1, x, 1, y), z)


@pytest.mark.parametrize("dt", [np.float32, np.float64, np.int32, np.int64])
def test_axpbz_matches_numpy(dt):
    if np.dtype(dt).kind == "f":
        x = RNG.standard_normal(3001).astype(dt)
        a, b = dt(5.7), dt(-0.3)
    else:
        x = RNG.integers(-(1 << 20), 1 << 20, size=3001).astype(dt)
        a, b = dt(-77), dt(12345)
    with np.errstate(over="ignore"):
        ref = (a * x) + b
    assert bits_equal(oracle.axpbz(a, x, b), ref)


def test_elementwise_empty():
    z = oracle.axpbyz(np.float32(1), np.zeros(0, np.float32), np.float32(1), np.zeros(0, np.float32))
    assert z.size == 0


# ------------------------------------------------------------ float reduce SUM
def _terms_f64(map_, x, y):
    x = x.astype(np.float64)
    if map_ == oracle.MAP_ID:
        return x
    if map_ == oracle.MAP_MUL:
        return x * y.astype(np.float64)
    return x * x


@pytest.mark.parametrize("map_", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
@pytest.mark.parametrize("kind", [synth.F32_U01, synth.F32_S11])
def test_sum_f32_equals_fsum(map_, kind):
    """fp32 terms are exact in float64; math.fsum is exactly rounded.  The
    Neumaier oracle must agree to ~1 ulp (catches a dropped compensation term,
    a wrong branch, or a map that squares y instead of x)."""
    n = (1 << 18) + 3
    x = synth.host_fill(kind, 1, n)
    y = synth.host_fill(kind, 2, n)
    t = _terms_f64(map_, x, y)
    ref = math.fsum(t.tolist())
    got, sa = oracle.reduce(oracle.SUM, map_, x, y, return_sumabs=True)
    assert abs(got - ref) <= 2 * np.spacing(abs(ref))
    assert abs(sa - math.fsum(np.abs(t).tolist())) <= 2 * np.spacing(sa)


def test_neumaier_catastrophic_cancellation():
    """[1, 1e30, 1, -1e30] sums to exactly 2 (plain and Kahan summation give 0)."""
    x = np.array([1.0, 1e30, 1.0, -1e30], dtype=np.float32)
    assert float(np.float32(1e30)) + 1.0 == float(np.float32(1e30))  # naive f64 loses the 1s
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, x) == 2.0
    x64 = np.array([1.0, 1e100, 1.0, -1e100])
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, x64) == 2.0


def test_sum_f64_mul_includes_product_error():
    """For fp64 inputs the oracle adds RN(x*y) and fma's exact error term:
    dot([1+2^-30, -1], [1-2^-30, 1]) = -2^-60 exactly (0 without the term)."""
    x = np.array([1 + 2.0 ** -30, -1.0])
    y = np.array([1 - 2.0 ** -30, 1.0])
    assert oracle.reduce(oracle.SUM, oracle.MAP_MUL, x, y) == -(2.0 ** -60)
    assert oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, np.array([1 + 2.0 ** -30]), None) == 1.0 + 2.0 ** -29


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("map_", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
def test_sum_brute_force_fraction(n, map_):
    """Exact rational brute force on tiny inputs: the fp64-rounded exact sum."""
    for dt in (np.float32, np.float64):
        x = (RNG.standard_normal(n) * 10.0 ** RNG.integers(-5, 5, n)).astype(dt)
        y = (RNG.standard_normal(n) * 10.0 ** RNG.integers(-5, 5, n)).astype(dt)
        fx = [Fraction(float(v)) for v in x]
        fy = [Fraction(float(v)) for v in y]
        if map_ == oracle.MAP_ID:
            exact = sum(fx, Fraction(0))
        elif map_ == oracle.MAP_MUL:
            exact = sum((a * b for a, b in zip(fx, fy)), Fraction(0))
        else:
            exact = sum((a * a for a in fx), Fraction(0))
        got = oracle.reduce(oracle.SUM, map_, x, y)
        # Neumaier bound: eps*|S| + O(n eps^2) sum|t| (tiny here); a dropped term is far outside
        sumabs = sum(abs(a * b) if map_ == oracle.MAP_MUL else abs(a * a if map_ == oracle.MAP_SQUARE else a)
                     for a, b in zip(fx, fy))
        tol = Fraction(abs(float(exact))) * Fraction(1, 1 << 51) + sumabs * Fraction(4 * n, 1 << 104)
        assert abs(Fraction(got) - exact) <= tol


def test_sum_closed_forms():
    n = 1 << 20
    ramp1 = synth.host_fill(synth.F32_RAMP, 0, n, lo=1)          # 1..n
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, ramp1) == n * (n + 1) / 2
    ramp0 = synth.host_fill(synth.F32_RAMP, 0, n, lo=0)          # 0..n-1
    twos = np.full(n, 2.0, np.float32)
    assert oracle.reduce(oracle.SUM, oracle.MAP_MUL, twos, ramp0) == n * (n - 1)     # BJ: constant . ramp
    assert oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, np.ones(n, np.float32)) == n
    m = 1 << 17
    r = synth.host_fill(synth.F64_RAMP, 0, m)
    assert oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, r) == (m - 1) * m * (2 * m - 1) / 6


def test_dot_spec_example(golden):
    g = golden("dot_spec_example.json")
    x = np.array(g["x"], dtype=np.float32)
    y = np.array(g["y"], dtype=np.float32)
    assert oracle.reduce(oracle.SUM, oracle.MAP_MUL, x, y) == g["dot"]


def test_float_sum_empty_is_neutral():
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, np.zeros(0, np.float32)) == 0.0
    assert oracle.reduce(oracle.SUM, oracle.MAP_MUL, np.zeros(0), np.zeros(0)) == 0.0


# ------------------------------------------------------------ integer reduce SUM
@pytest.mark.parametrize("in_dt,out_dt", [(np.int32, np.int32), (np.int32, np.int64), (np.int64, np.int64)])
@pytest.mark.parametrize("map_", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
def test_int_sum_matches_bigint(in_dt, out_dt, map_):
    """Python big ints, then mod 2^w_out: catches a missing widen-before-multiply
    or summing in the wrong width."""
    info = np.iinfo(in_dt)
    x = RNG.integers(info.min, info.max, size=2000, dtype=in_dt, endpoint=True)
    y = RNG.integers(info.min, info.max, size=2000, dtype=in_dt, endpoint=True)
    w = np.dtype(out_dt).itemsize * 8
    if map_ == oracle.MAP_ID:
        terms = [int(v) for v in x]
    elif map_ == oracle.MAP_MUL:
        terms = [int(a) * int(b) for a, b in zip(x, y)]
    else:
        terms = [int(a) * int(a) for a in x]
    v = sum(terms) % (1 << w)
    v = v - (1 << w) if v >= (1 << (w - 1)) else v
    assert oracle.reduce(oracle.SUM, map_, x, y, out_dtype=out_dt) == v


def test_int_sum_spec_and_closed_form(golden):
    g = golden("sum_1_to_8.json")
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, np.array(g["input"], np.int32)) == g["sum"]
    n = 1 << 20
    r = synth.host_fill(synth.I32_RAMP, 0, n, lo=1)
    v = (n * (n + 1) // 2) % (1 << 32)
    v = v - (1 << 32) if v >= (1 << 31) else v
    assert oracle.reduce(oracle.SUM, oracle.MAP_ID, r) == v  # wraps (5.5e11 > 2^31)
    with np.errstate(over="ignore"):
        assert oracle.reduce(oracle.SUM, oracle.MAP_ID, r) == int(np.add.reduce(r, dtype=np.int32))


# ------------------------------------------------------------ MAX / MIN
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("map_", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
def test_float_maxmin_match_numpy(dt, map_):
    """map in the input dtype (R3), fold with maxNum/minNum (R6)."""
    x = RNG.standard_normal(5003).astype(dt)
    y = RNG.standard_normal(5003).astype(dt)
    t = x if map_ == oracle.MAP_ID else (x * y if map_ == oracle.MAP_MUL else x * x)
    assert oracle.reduce(oracle.MAX, map_, x, y) == np.max(t)
    assert oracle.reduce(oracle.MIN, map_, x, y) == np.min(t)


def test_float_maxmin_planted_and_nan():
    for pos in (0, 4095, 1234):
        x = synth.host_fill(synth.F32_S11, 4, 4096)
        x[pos] = 3.0
        assert oracle.reduce(oracle.MAX, oracle.MAP_ID, x) == 3.0
        x[pos] = -3.0
        assert oracle.reduce(oracle.MIN, oracle.MAP_ID, x) == -3.0
    x = np.array([1, np.nan, 3, -2], np.float32)
    assert oracle.reduce(oracle.MAX, oracle.MAP_ID, x) == np.fmax.reduce(x) == 3
    assert oracle.reduce(oracle.MIN, oracle.MAP_ID, x) == np.fmin.reduce(x) == -2
    # all-NaN: maxNum folding from the neutral element keeps the neutral (R6);
    # numpy.fmax.reduce starts from x[0] instead and returns nan.
    assert oracle.reduce(oracle.MAX, oracle.MAP_ID, np.array([np.nan, np.nan], np.float32)) == -np.inf
    assert np.fmax(np.float32(-np.inf), np.fmax(np.float32(-np.inf), np.float32(np.nan))) == -np.inf


# MAX / MIN with signed zeros (R7): IEEE 754-2019 maximumNumber /
# minimumNumber — NaN loses, -0 < +0.  Pinned against a brute force that
# knows nothing of the C code: Python's max/min over the non-NaN values keyed
# by (value, copysign(1, value)), so +0 ranks above -0.
def _key(v):
    return (float(v), math.copysign(1.0, float(v)))


def _brute_max(vals, neutral):
    vals = [v for v in vals if not math.isnan(float(v))]
    return max(vals, key=_key) if vals else neutral


def _brute_min(vals, neutral):
    vals = [v for v in vals if not math.isnan(float(v))]
    return min(vals, key=_key) if vals else neutral


def _zeros_heavy(dt, n, seed):
    rng = np.random.default_rng(seed)
    tiny = np.finfo(dt).tiny
    pool = np.array([-0.0, 0.0, -0.0, 0.0, -1.0, 1.0, np.nan, -tiny, tiny], dtype=dt)
    return pool[rng.integers(0, pool.size, size=n)]


def _same_bits(a, b, dt):
    return np.array(a, dt).tobytes() == np.array(b, dt).tobytes()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_maxmin_signed_zero_pairs(dt):
    """The four +-0 pairs in both operand orders, elementwise and folded."""
    p, m = dt(0.0), dt(-0.0)
    for a, b in ((p, m), (m, p), (p, p), (m, m)):
        x, y = np.array([a], dt), np.array([b], dt)
        want_max = p if (not np.signbit(a) or not np.signbit(b)) else m
        want_min = m if (np.signbit(a) or np.signbit(b)) else p
        assert _same_bits(oracle.ewmap(oracle.EW_MAX, x, y)[0], want_max, dt)
        assert _same_bits(oracle.ewmap(oracle.EW_MIN, x, y)[0], want_min, dt)
        xy = np.array([a, b], dt)
        assert _same_bits(oracle.reduce(oracle.MAX, oracle.MAP_ID, xy), want_max, dt)
        assert _same_bits(oracle.reduce(oracle.MIN, oracle.MAP_ID, xy), want_min, dt)
    # (+0) * (-1) = -0 under the x*y map: the product's sign counts too
    x, y = np.array([0.0, 0.0], dt), np.array([-1.0, 1.0], dt)
    assert _same_bits(oracle.reduce(oracle.MAX, oracle.MAP_MUL, x, y), p, dt)
    assert _same_bits(oracle.reduce(oracle.MIN, oracle.MAP_MUL, x, y), m, dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("mp", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
def test_maxmin_signed_zero_brute_force(dt, mp):
    for seed in range(6):
        x, y = _zeros_heavy(dt, 501, seed), _zeros_heavy(dt, 501, seed + 100)
        with np.errstate(all="ignore"):
            t = x if mp == oracle.MAP_ID else (x * y if mp == oracle.MAP_MUL else x * x)
        assert _same_bits(oracle.reduce(oracle.MAX, mp, x, y), _brute_max(t, dt(-np.inf)), dt)
        assert _same_bits(oracle.reduce(oracle.MIN, mp, x, y), _brute_min(t, dt(np.inf)), dt)
        # any order of the same values gives the same bits (a total order)
        perm = np.random.default_rng(seed).permutation(x.size)
        assert _same_bits(oracle.reduce(oracle.MAX, mp, x[perm], y[perm]), oracle.reduce(oracle.MAX, mp, x, y), dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
def test_scan_and_ewmap_maxmin_signed_zero_brute_force(dt, op):
    x, y = _zeros_heavy(dt, 700, 7 + op), _zeros_heavy(dt, 700, 8 + op)
    brute = _brute_max if op == oracle.MAX else _brute_min
    neutral = dt(-np.inf) if op == oracle.MAX else dt(np.inf)
    inc = oracle.scan(oracle.INCLUSIVE, x, op=op)
    exc = oracle.scan(oracle.EXCLUSIVE, x, op=op)
    for i in range(x.size):
        assert _same_bits(inc[i], brute(list(x[:i + 1]), neutral), dt), i
        assert _same_bits(exc[i], brute(list(x[:i]), neutral), dt), i
    ew = oracle.ewmap(oracle.EW_MAX if op == oracle.MAX else oracle.EW_MIN, x, y)
    for i in range(x.size):
        assert _same_bits(ew[i], brute([x[i], y[i]], dt(np.nan)), dt), i


def test_float_maxmin_empty_is_neutral():
    assert oracle.reduce(oracle.MAX, oracle.MAP_ID, np.zeros(0, np.float32)) == -np.inf
    assert oracle.reduce(oracle.MIN, oracle.MAP_ID, np.zeros(0)) == np.inf


@pytest.mark.parametrize("dt", [np.int32, np.int64])
@pytest.mark.parametrize("map_", [oracle.MAP_ID, oracle.MAP_MUL, oracle.MAP_SQUARE])
def test_int_maxmin(dt, map_):
    info = np.iinfo(dt)
    x = RNG.integers(info.min, info.max, size=3000, dtype=dt, endpoint=True)
    y = RNG.integers(info.min, info.max, size=3000, dtype=dt, endpoint=True)
    with np.errstate(over="ignore"):
        t = x if map_ == oracle.MAP_ID else (x * y if map_ == oracle.MAP_MUL else x * x)
    assert oracle.reduce(oracle.MAX, map_, x, y) == max(int(v) for v in t)
    assert oracle.reduce(oracle.MIN, map_, x, y) == min(int(v) for v in t)


def test_int_min_spec(golden):
    g = golden("min_neutral_spec.json")
    assert oracle.reduce(oracle.MIN, oracle.MAP_ID, np.zeros(0, np.int32)) == g["empty_min"]
    x = np.array(g["input"], np.int32)
    assert oracle.reduce(oracle.MIN, oracle.MAP_ID, x) == g["min"]
    assert oracle.reduce(oracle.MAX, oracle.MAP_ID, x) == g["max"]
    for n in (1, 255, 256, 257, 100000):  # SPEC.md:555 sizes
        v = RNG.integers(-(1 << 31), (1 << 31) - 1, size=n, dtype=np.int32)
        assert oracle.reduce(oracle.MIN, oracle.MAP_ID, v) == min(int(a) for a in v)
    assert oracle.reduce(oracle.MAX, oracle.MAP_ID, np.zeros(0, np.int64)) == -(1 << 63)


# ------------------------------------------------------------ scan
def test_scan_spec_example(golden):
    g = golden("scan_spec_example.json")
    x = np.array(g["input"], np.int32)
    assert oracle.scan(oracle.INCLUSIVE, x).tolist() == g["inclusive"]
    assert oracle.scan(oracle.EXCLUSIVE, x).tolist() == g["exclusive"]


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_scan_closed_forms(dt):
    n = 100003
    ones = np.ones(n, dt)
    assert bits_equal(oracle.scan(oracle.INCLUSIVE, ones), np.arange(1, n + 1, dtype=dt))   # BJ: i+1
    assert bits_equal(oracle.scan(oracle.EXCLUSIVE, ones), np.arange(0, n, dtype=dt))       # i
    r = np.arange(n, dtype=np.int64)
    tri = (r * (r + 1) // 2)
    with np.errstate(over="ignore"):
        assert bits_equal(oracle.scan(oracle.INCLUSIVE, r.astype(dt)), tri.astype(dt))


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_scan_matches_numpy_cumsum_wrap(dt):
    info = np.iinfo(dt)
    x = RNG.integers(info.min // 4, info.max // 4, size=70001, dtype=dt)
    with np.errstate(over="ignore"):
        inc = np.cumsum(x, dtype=dt)
    assert bits_equal(oracle.scan(oracle.INCLUSIVE, x), inc)
    exc = np.concatenate([np.zeros(1, dt), inc[:-1]])
    assert bits_equal(oracle.scan(oracle.EXCLUSIVE, x), exc)
    # carry-in shifts everything (sharded offset)
    c = dt(1234567)
    with np.errstate(over="ignore"):
        assert bits_equal(oracle.scan(oracle.INCLUSIVE, x, carry=c), (inc + c).astype(dt))
        assert bits_equal(oracle.scan(oracle.EXCLUSIVE, x, carry=c), (exc + c).astype(dt))


def test_scan_reduce_consistency_and_inplace():
    """Last inclusive element == reduce SUM; in-place allowed (R13)."""
    x = synth.host_fill(synth.I32_RANGE, 3, 1 << 20, lo=0, hi=9)
    inc = oracle.scan(oracle.INCLUSIVE, x)
    assert int(inc[-1]) == oracle.reduce(oracle.SUM, oracle.MAP_ID, x)
    y = x.copy()
    oracle.scan(oracle.INCLUSIVE, y, out=y)
    assert bits_equal(y, inc)


def test_scan_empty():
    assert oracle.scan(oracle.INCLUSIVE, np.zeros(0, np.int32)).size == 0


# ------------------------------------------------------------ scans with MAX/MIN and float SUM (NEXT-2)
@pytest.mark.parametrize("dt", [np.int32, np.int64, np.float32, np.float64])
@pytest.mark.parametrize("op", [oracle.MAX, oracle.MIN])
def test_scan_maxmin_match_numpy_accumulate(dt, op):
    """Running max/min = numpy.fmax/fmin.accumulate (NaN-ignoring, R6);
    exclusive = the same shifted right with the neutral element at the head."""
    if np.dtype(dt).kind == "f":
        x = RNG.standard_normal(10007).astype(dt)
        x[[5, 77, 4000]] = np.nan
        acc = np.fmax.accumulate if op == oracle.MAX else np.fmin.accumulate
        neutral = -np.inf if op == oracle.MAX else np.inf
    else:
        info = np.iinfo(dt)
        x = RNG.integers(info.min, info.max, size=10007, dtype=dt, endpoint=True)
        acc = np.maximum.accumulate if op == oracle.MAX else np.minimum.accumulate
        neutral = info.min if op == oracle.MAX else info.max
    inc = acc(np.concatenate([np.array([neutral], dt), x]))[1:].astype(dt)  # fold from the neutral
    assert bits_equal(oracle.scan(oracle.INCLUSIVE, x, op=op), inc)
    exc = np.concatenate([np.array([neutral], dt), inc[:-1]])
    assert bits_equal(oracle.scan(oracle.EXCLUSIVE, x, op=op), exc)


def test_scan_max_spec_like_example():
    x = np.array([3, 1, 4, 1, 5, 9, 2, 6], np.int32)
    assert oracle.scan(oracle.INCLUSIVE, x, op=oracle.MAX).tolist() == [3, 3, 4, 4, 5, 9, 9, 9]
    assert oracle.scan(oracle.EXCLUSIVE, x, op=oracle.MIN).tolist() == [2147483647, 3, 1, 1, 1, 1, 1, 1]
    assert oracle.scan(oracle.INCLUSIVE, x, op=oracle.MAX, carry=7).tolist() == [7, 7, 7, 7, 7, 9, 9, 9]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_scan_float_sum_exact_prefixes(dt):
    """Float SUM scan returns the exact prefix sums (as float64): equal to
    math.fsum of every prefix at sampled points (catches an uncompensated
    running sum, an off-by-one head, a dropped carry)."""
    x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 9, 50_001)
    x[100] = 1e20
    x[101] = -1e20  # cancellation a plain running double sum would get wrong
    inc, sa = oracle.scan(oracle.INCLUSIVE, x, return_sumabs=True)
    exc = oracle.scan(oracle.EXCLUSIVE, x, carry=0.25)
    u = 2.0 ** -53
    for i in (0, 1, 99, 100, 101, 102, 4095, 50_000):
        pref = math.fsum(float(v) for v in x[:i + 1])
        sabs = math.fsum(abs(float(v)) for v in x[:i + 1])
        # Neumaier's bound: 2u|S| + 2 i u^2 sum|x| (the 1e20 terms make the second visible)
        assert abs(inc[i] - pref) <= 2 * u * abs(pref) + 2 * (i + 1) * u * u * sabs + 1e-300
        assert sa[i] == pytest.approx(sabs, rel=1e-15)
        pe = math.fsum([0.25] + [float(v) for v in x[:i]])
        assert abs(exc[i] - pe) <= 2 * u * abs(pe) + 2 * (i + 1) * u * u * (sabs + 0.25) + 1e-300
    # a plain running float64 sum is visibly worse right after the cancellation
    plain = np.cumsum(x.astype(np.float64))
    exact = math.fsum(float(v) for v in x[:102])
    assert abs(plain[101] - exact) > abs(inc[101] - exact)


def test_scan_float_sum_closed_forms():
    n = 1 << 20
    ones = np.ones(n, np.float32)
    assert np.array_equal(oracle.scan(oracle.INCLUSIVE, ones), np.arange(1, n + 1, dtype=np.float64))
    r = synth.host_fill(synth.F64_RAMP, 0, n)
    i = np.arange(n, dtype=np.float64)
    assert np.array_equal(oracle.scan(oracle.EXCLUSIVE, r), i * (i - 1) / 2)


def test_scan_widening_closed_forms():
    """Widened scans (R27): int32 -> int64 does not wrap where the int32 scan
    does (closed form k*(2^31-1)); MAX/MIN are unchanged by widening; float32
    -> float64 keeps prefixes an fp32 running sum loses (1 + k*2^-30)."""
    n = 70_001
    big = np.full(n, np.iinfo(np.int32).max, np.int32)
    k = np.arange(1, n + 1, dtype=np.int64)
    w = oracle.scan(oracle.INCLUSIVE, big, out_dtype=np.int64)
    assert w.dtype == np.int64 and bits_equal(w, k * (2 ** 31 - 1))
    we = oracle.scan(oracle.EXCLUSIVE, big, out_dtype=np.int64, carry=-5)
    assert bits_equal(we, (k - 1) * (2 ** 31 - 1) - 5)
    assert oracle.scan(oracle.INCLUSIVE, big)[1] == -2  # the narrow scan wraps: 2(2^31-1) mod 2^32
    x = RNG.integers(-(1 << 31), (1 << 31) - 1, size=n, dtype=np.int32)
    for op in (oracle.MAX, oracle.MIN):
        assert bits_equal(oracle.scan(oracle.INCLUSIVE, x, op=op, out_dtype=np.int64),
                          oracle.scan(oracle.INCLUSIVE, x, op=op).astype(np.int64))
    f = np.full(1 << 16, 2.0 ** -30, np.float32)
    f[0] = 1.0
    pf = oracle.scan(oracle.INCLUSIVE, f, out_dtype=np.float64)
    assert np.array_equal(pf, 1.0 + np.arange(1 << 16) * 2.0 ** -30)
    with pytest.raises(TypeError):
        oracle.scan(oracle.INCLUSIVE, np.zeros(3, np.int64), out_dtype=np.int32)


# ------------------------------------------------------------ complex (NEXT-3)
def _cplx(dt, n, seed):
    f = np.float32 if dt == np.complex64 else np.float64
    r = synth.host_fill(synth.F32_S11 if f == np.float32 else synth.F64_S11, seed, 2 * n)
    return r.view(dt)


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
def test_complex_axpbyz_matches_componentwise_numpy(dt):
    """R24: re = RN(RN(ar xr) - RN(ai xi)) etc., re-derived here with numpy
    real arithmetic (independent twin); a swapped sign or component fails."""
    x = _cplx(dt, 5003, 1)
    y = _cplx(dt, 5003, 2)
    a, b = dt(1.5 - 2.25j), dt(-0.75 + 0.5j)
    f = np.float32 if dt == np.complex64 else np.float64
    ar, ai, br, bi = f(a.real), f(a.imag), f(b.real), f(b.imag)
    xr, xi, yr, yi = x.real, x.imag, y.real, y.imag
    zr = ((ar * xr) - (ai * xi)) + ((br * yr) - (bi * yi))
    zi = ((ar * xi) + (ai * xr)) + ((br * yi) + (bi * yr))
    z = oracle.axpbyz_complex(a, x, b, y)
    assert bits_equal(z.real.copy(), zr) and bits_equal(z.imag.copy(), zi)
    # closed forms: a=1, b=0 -> x; a=i, b=0 -> i*x = (-xi, xr)
    assert bits_equal(oracle.axpbyz_complex(1, x, 0, y).view(f), (x + 0 * y).view(f))
    iz = oracle.axpbyz_complex(1j, x, 0, y)
    assert bits_equal(iz.real.copy(), -xi + f(0)) and bits_equal(iz.imag.copy(), xr + f(0))


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
def test_complex_sums_against_fraction_and_fsum(dt):
    x = _cplx(dt, 20001, 3)
    y = _cplx(dt, 20001, 4)
    xc, yc = x.astype(np.complex128), y.astype(np.complex128)
    # sum: fsum per component
    s = oracle.reduce_complex(oracle.MAP_ID, x)
    assert s.real == math.fsum(xc.real.tolist()) and s.imag == math.fsum(xc.imag.tolist())
    # dot / vdot / norm2 on a small prefix with exact rational arithmetic
    m = 50
    fx = [(Fraction(float(v.real)), Fraction(float(v.imag))) for v in xc[:m]]
    fy = [(Fraction(float(v.real)), Fraction(float(v.imag))) for v in yc[:m]]
    dre = sum(a[0] * b[0] - a[1] * b[1] for a, b in zip(fx, fy))
    dim = sum(a[0] * b[1] + a[1] * b[0] for a, b in zip(fx, fy))
    vre = sum(a[0] * b[0] + a[1] * b[1] for a, b in zip(fx, fy))
    vim = sum(a[0] * b[1] - a[1] * b[0] for a, b in zip(fx, fy))
    n2 = sum(a[0] * a[0] + a[1] * a[1] for a in fx)
    d = oracle.reduce_complex(oracle.MAP_MUL, x[:m], y[:m])
    v = oracle.reduce_complex(oracle.MAP_CONJ_MUL, x[:m], y[:m])
    assert d.real == float(dre) and d.imag == float(dim)
    assert v.real == float(vre) and v.imag == float(vim)
    assert oracle.reduce_complex(oracle.MAP_SQUARE, x[:m]) == float(n2)
    # vdot(x, x) = |x|^2 (imaginary part exactly 0)
    vv = oracle.reduce_complex(oracle.MAP_CONJ_MUL, x, x)
    assert vv.imag == 0.0 and vv.real == pytest.approx(oracle.reduce_complex(oracle.MAP_SQUARE, x), rel=1e-15)


# ------------------------------------------------------------ stencil / tridiagonal matvec (NEXT-4)
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_stencil3_matches_dense_and_numpy(dt):
    """Against numpy's uncontracted (l*x[:-2] + d*x[1:-1]) + u*x[2:] with the
    boundary terms omitted, and against a dense tridiagonal matrix product
    (float64, tolerance) — catches swapped l/u, a shifted neighbour, a
    boundary term that should be omitted."""
    n = 1001
    x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 1, n)
    l, d, u = dt(-1.25), dt(2.5), dt(-0.75)
    y = oracle.stencil3(l, d, u, x)
    ref = np.empty_like(x)
    ref[1:-1] = ((l * x[:-2]) + (d * x[1:-1])) + (u * x[2:])
    ref[0] = (d * x[0]) + (u * x[1])
    ref[-1] = (l * x[-2]) + (d * x[-1])
    assert bits_equal(y, ref)
    A = np.diag(np.full(n, float(d))) + np.diag(np.full(n - 1, float(l)), -1) + np.diag(np.full(n - 1, float(u)), 1)
    assert np.allclose(A @ x.astype(np.float64), y, rtol=0, atol=1e-5 if dt == np.float32 else 1e-13)
    diag = synth.host_fill(synth.F32_U01 if dt == np.float32 else synth.F64_U01, 2, n)
    yd = oracle.stencil3(l, d, u, x, diag=diag)
    A = np.diag(diag.astype(np.float64)) + np.diag(np.full(n - 1, float(l)), -1) + np.diag(np.full(n - 1, float(u)), 1)
    assert np.allclose(A @ x.astype(np.float64), yd, rtol=0, atol=1e-5 if dt == np.float32 else 1e-13)


def test_stencil3_poisson_closed_forms():
    """1-D Poisson (l = u = -1, d = 2): a constant vector maps to zero inside
    and to the constant at the two ends; a linear ramp maps to zero inside."""
    n = 100
    c = np.full(n, 3.0)
    y = oracle.stencil3(-1, 2, -1, c)
    assert np.all(y[1:-1] == 0) and y[0] == 3.0 and y[-1] == 3.0
    r = np.arange(n, dtype=np.float64)
    y = oracle.stencil3(-1, 2, -1, r)
    assert np.all(y[1:-1] == 0) and y[0] == -1.0 and y[-1] == n


# ------------------------------------------------------------ other operators / cumath maps (NEXT-2)
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_ewmap_float_against_numpy(dt):
    """IEEE-exact ops equal numpy bit for bit; libm maps are within 1 ulp of
    numpy's (both are faithful implementations)."""
    x = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 1, 4099) * dt(3)
    y = synth.host_fill(synth.F32_S11 if dt == np.float32 else synth.F64_S11, 2, 4099) + dt(1.5)
    ax = np.abs(x) + dt(1e-3)
    with np.errstate(all="ignore"):
        assert bits_equal(oracle.ewmap(oracle.EW_MUL, x, y), x * y)
        assert bits_equal(oracle.ewmap(oracle.EW_DIV, x, y), x / y)
        assert bits_equal(oracle.ewmap(oracle.EW_SQRT, ax), np.sqrt(ax))
        assert bits_equal(oracle.ewmap(oracle.EW_ABS, x), np.abs(x))
        assert bits_equal(oracle.ewmap(oracle.EW_NEG, x), -x)
        assert bits_equal(oracle.ewmap(oracle.EW_MAX, x, y), np.fmax(x, y))
        assert bits_equal(oracle.ewmap(oracle.EW_MIN, x, y), np.fmin(x, y))
        for op, f, arg in ((oracle.EW_EXP, np.exp, x), (oracle.EW_LOG, np.log, ax), (oracle.EW_SIN, np.sin, x),
                           (oracle.EW_COS, np.cos, x)):
            got = oracle.ewmap(op, arg)
            # reference: float64 evaluation rounded once (fp32 inputs: the
            # correctly rounded value in all but rare cases); glibc is faithful
            ref = f(arg.astype(np.float64)).astype(dt)
            ulps = np.abs(got.view(np.int32 if dt == np.float32 else np.int64).astype(np.int64)
                          - ref.view(np.int32 if dt == np.float32 else np.int64).astype(np.int64))
            assert ulps.max() <= (1 if dt == np.float32 else 2), (op, ulps.max())
    # special cases: sqrt(-1) = nan, log(0) = -inf, exp(0) = 1
    with np.errstate(all="ignore"):
        assert np.isnan(oracle.ewmap(oracle.EW_SQRT, np.array([-1.0], dt))[0])
        assert oracle.ewmap(oracle.EW_LOG, np.array([0.0], dt))[0] == -np.inf
        assert oracle.ewmap(oracle.EW_EXP, np.array([0.0], dt))[0] == 1.0


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_ewmap_int_wraps(dt):
    info = np.iinfo(dt)
    x = RNG.integers(info.min, info.max, size=3001, dtype=dt, endpoint=True)
    y = RNG.integers(info.min, info.max, size=3001, dtype=dt, endpoint=True)
    x[0] = info.min
    with np.errstate(over="ignore"):
        assert bits_equal(oracle.ewmap(oracle.EW_MUL, x, y), x * y)
        assert bits_equal(oracle.ewmap(oracle.EW_NEG, x), -x)
        assert bits_equal(oracle.ewmap(oracle.EW_ABS, x), np.abs(x))   # abs(INT_MIN) wraps to INT_MIN
    assert bits_equal(oracle.ewmap(oracle.EW_MAX, x, y), np.maximum(x, y))
    assert bits_equal(oracle.ewmap(oracle.EW_MIN, x, y), np.minimum(x, y))
