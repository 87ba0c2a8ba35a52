"""Parity at BASELINE.json's full sizes, through the same calls (and hence the
same launch configurations) bench.py times.  The oracle cannot hold or scan
2^33 elements in one go, so it runs chunk-wise over regenerated inputs
(tests/bigcheck.py); outputs too large to compare whole are checked on
sampled windows whose exact expected values the chunked oracle provides,
plus properties that hold at any size; integer scans are compared whole,
element by element, against the chunked oracle (bigcheck.chunked_scan_compare).

  C2  fp32/fp64 axpbyz (full, bit-exact) and norm2 (tolerance) on n = 2^28
  C3  int32/int64 sum (exact), max (exact, planted), inclusive scan on n = 2^30
  C4  fp32 dot + norm2 on n = 2^33 (one GPU holds both 32 GiB inputs)
  C5  int32 exclusive scan on n = 2^33 (every element, chunked oracle), also
      as 8 contiguous shards with the sharded path's totals -> carry-in
  float32 SUM scan at 2^28: every element within R22's bound
  bench step: axpbyz(5, x, 6, y) + dot + sum + norm2 + exclusive scan at 2^28."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import bigcheck  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"


def free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def need_bytes(nbytes):
    freeb, _ = torch.cuda.mem_get_info()
    if freeb < nbytes * 1.05:
        pytest.skip(f"needs {nbytes / 2**30:.0f} GiB of free device memory, {freeb / 2**30:.0f} available")


def float_tol(odt, n, ref, sumabs):
    rel, u = (1e-5, 2.0 ** -24) if odt == np.float32 else (1e-12, 2.0 ** -53)
    return max(rel * abs(ref), n * u * sumabs), rel * abs(ref)


def bits(a):
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_c2_axpbyz_full_bit_exact(dt):
    n = 1 << 28
    kind, npdt = (synth.F32_S11, np.float32) if dt == "f32" else (synth.F64_S11, np.float64)
    need_bytes(3 * n * np.dtype(npdt).itemsize)
    x = synth.device_fill(kind, 1, n, device=DEV)
    y = synth.device_fill(kind, 2, n, device=DEV)
    z = G.axpbyz(5.0, x, -6.0, y).cpu().numpy()
    del x, y
    free()
    xh = synth.host_fill(kind, 1, n)
    yh = synth.host_fill(kind, 2, n)
    ref = oracle.axpbyz(npdt(5.0), xh, npdt(-6.0), yh)
    bad = np.count_nonzero(bits(z) != bits(ref))
    assert bad == 0, f"{bad} of {n} elements differ"


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("signed", [False, True])
def test_c2_norm2_full(dt, signed):
    n = 1 << 28
    if dt == "f32":
        kind, npdt = (synth.F32_S11 if signed else synth.F32_U01), np.float32
    else:
        kind, npdt = (synth.F64_S11 if signed else synth.F64_U01), np.float64
    x = synth.device_fill(kind, 1, n, device=DEV)
    got = float(G.norm2sq(x).item())
    del x
    free()
    ref, sa = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_SQUARE, n, kind, 1)
    tol, flat = float_tol(npdt, n, ref, sa)
    assert abs(got - ref) <= tol and abs(got - ref) <= flat  # squares never cancel


@pytest.mark.parametrize("dt", ["i32", "i64"])
def test_c3_int_sum_max_scan_2p30(dt):
    n = 1 << 30
    kind = synth.I32_RANGE if dt == "i32" else synth.I64_RANGE
    npdt = np.int32 if dt == "i32" else np.int64
    esz = np.dtype(npdt).itemsize
    need_bytes(2 * n * esz)
    # sum over U[-2^15, 2^15): exact (wrapping) integer arithmetic on both sides
    x = synth.device_fill(kind, 3, n, lo=-(1 << 15), hi=(1 << 15) - 1, device=DEV)
    got_sum = int(G.sum(x).item())
    ref_sum, _ = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_ID, n, kind, 3, lo=-(1 << 15), hi=(1 << 15) - 1,
                                         out_dtype=npdt)
    assert got_sum == ref_sum
    # max over full-range data with a unique planted maximum
    del x
    free()
    lo, hi = -(1 << 31), (1 << 31) - 2
    x = synth.device_fill(kind, 4, n, lo=lo, hi=hi, device=DEV)
    pos = 987_654_321
    orig = int(x[pos].item())
    planted = int(np.iinfo(npdt).max)   # above every generated value: a unique maximum
    x[pos] = planted
    assert int(G.max(x).item()) == planted
    x[pos] = orig
    ref_max, _ = bigcheck.chunked_reduce(oracle.MAX, oracle.MAP_ID, n, kind, 4, lo=lo, hi=hi)
    ref_min, _ = bigcheck.chunked_reduce(oracle.MIN, oracle.MAP_ID, n, kind, 4, lo=lo, hi=hi)
    assert int(G.max(x).item()) == ref_max
    assert int(G.min(x).item()) == ref_min
    del x
    free()
    # inclusive scan of U{0..9}: exact windows at every chunk boundary + last element
    k = synth.device_fill(kind, 3, n, lo=0, hi=9, device=DEV)
    out = G.scan(k)
    del k
    free()
    _check_scan_full(out, n, kind, 3, 0, 9, npdt, exclusive=False)


@pytest.mark.parametrize("n,exclusive", [((1 << 30), True), ((1 << 30) + 5, False)])
def test_int32_scan_at_the_ring_windows_upper_edge(n, exclusive):
    """4 GiB of int32 input is the last size the ring kernel takes (with its
    one-tile L2 prefetch); 5 elements more go to the two-touch L shape.  Both
    sides of the edge, every element against the chunked oracle."""
    need_bytes(2 * n * 4)
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=DEV)
    out = G.scan(k, exclusive=exclusive)
    del k
    free()
    _check_scan_full(out, n, synth.I32_RANGE, 3, 0, 9, np.int32, exclusive=exclusive)


def _check_scan_full(out, n, kind, seed, lo, hi, npdt, exclusive):
    """Every element of the device scan output against the chunked oracle."""
    def fetch(start, m, dest):
        torch.from_numpy(dest).copy_(out[start:start + m])
    compared, bad, first = bigcheck.chunked_scan_compare(fetch, n, kind, seed, lo, hi, npdt, exclusive)
    assert compared == n
    assert bad == 0, f"{bad} of {n} elements differ, first at {first}"


def _check_scan_windows(out, n, kind, seed, lo, hi, npdt, exclusive, window=1 << 16, widen=False):
    chunk = bigcheck.CHUNK
    sums = bigcheck.chunk_sums_int(n, kind, seed, lo, hi, chunk)
    w = 1 << (np.dtype(npdt).itemsize * 8)
    prefix = 0
    checked = 0
    for c, s in enumerate(sums):
        start = c * chunk
        m = min(window, n - start)
        xin = synth.host_fill(kind, seed, m, start=start, lo=lo, hi=hi)
        carry = npdt(((prefix + w // 2) % w) - w // 2)
        ref = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, xin, carry=carry,
                          out_dtype=npdt if widen else None)
        got = out[start:start + m].cpu().numpy()
        assert np.array_equal(got, ref), f"window at {start}"
        checked += m
        prefix += s
    # the last element against the whole-array oracle total
    xlast = synth.host_fill(kind, seed, 1, start=n - 1, lo=lo, hi=hi)
    total = (prefix + w // 2) % w - w // 2
    last = int(out[n - 1].item())
    expect = total - int(xlast[0]) if exclusive else total
    expect = (expect + w // 2) % w - w // 2
    assert last == expect
    assert checked >= min(n, len(sums) * window)


def test_c3_widening_scan_2p30():
    """int32 -> int64 inclusive scan at C3's size (NEXT-2, R27): the U{0..9}
    prefix sums reach ~4.8e9, past int32's range, and must not wrap."""
    n = 1 << 30
    need_bytes(12 * n)
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=DEV)
    out = G.scan(k, out_dtype=torch.int64)
    del k
    free()
    assert int(out[-1].item()) > (1 << 31)
    _check_scan_full(out, n, synth.I32_RANGE, 3, 0, 9, np.int64, exclusive=False)


def test_c4_dot_norm2_2p33():
    n = 1 << 33
    need_bytes(2 * n * 4)
    x = synth.device_fill(synth.F32_U01, 1, n, device=DEV)
    y = synth.device_fill(synth.F32_U01, 2, n, device=DEV)
    got_dot = float(G.dot(x, y).item())
    got_n2 = float(G.norm2sq(x).item())
    del x, y
    free()
    ref, sa = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_MUL, n, synth.F32_U01, 1, kind_y=synth.F32_U01, seed_y=2)
    tol, flat = float_tol(np.float32, n, ref, sa)
    assert abs(got_dot - ref) <= flat, (got_dot, ref, abs(got_dot - ref) / ref)
    ref2, sa2 = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_SQUARE, n, synth.F32_U01, 1)
    assert abs(got_n2 - ref2) <= float_tol(np.float32, n, ref2, sa2)[1]


def test_c5_exclusive_scan_2p33():
    n = 1 << 33
    need_bytes(2 * n * 4)
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=DEV)
    out = G.scan(k, exclusive=True)
    del k
    free()
    _check_scan_full(out, n, synth.I32_RANGE, 3, 0, 9, np.int32, exclusive=True)
    del out
    free()


def test_bench_step_full_size():
    """The exact calls of one bench.py step at n = 2^28, each checked."""
    n = 1 << 28
    x = synth.device_fill(synth.F32_U01, synth.SEED_X, n, device=DEV)
    y = synth.device_fill(synth.F32_U01, synth.SEED_Y, n, device=DEV)
    k = synth.device_fill(synth.I32_RANGE, synth.SEED_INT, n, lo=0, hi=9, device=DEV)
    z = torch.empty_like(x)
    s = torch.empty_like(k)
    red = torch.empty(3, dtype=torch.float32, device=DEV)
    G.axpbyz(5.0, x, 6.0, y, out=z)
    G.reduce(G.SUM, G.MUL, x, y, out=red[0:1])
    G.reduce(G.SUM, G.ID, x, out=red[1:2])
    G.reduce(G.SUM, G.SQUARE, x, out=red[2:3])
    G.scan(k, exclusive=True, out=s)
    zh = z.cpu().numpy()
    r = red.cpu().numpy()
    del x, y, z, k
    free()
    xh = synth.host_fill(synth.F32_U01, synth.SEED_X, n)
    yh = synth.host_fill(synth.F32_U01, synth.SEED_Y, n)
    assert np.array_equal(bits(zh), bits(oracle.axpbyz(np.float32(5), xh, np.float32(6), yh)))
    for got, mp in zip(r, (oracle.MAP_MUL, oracle.MAP_ID, oracle.MAP_SQUARE)):
        ref = oracle.reduce(oracle.SUM, mp, xh, yh)
        assert abs(float(got) - ref) <= 1e-5 * abs(ref)
    del xh, yh
    _check_scan_windows(s, n, synth.I32_RANGE, synth.SEED_INT, 0, 9, np.int32, exclusive=True)
    kh = synth.host_fill(synth.I32_RANGE, synth.SEED_INT, n, lo=0, hi=9)
    assert np.array_equal(s.cpu().numpy(), oracle.scan(oracle.EXCLUSIVE, kh))   # and the whole vector
    assert math.isfinite(float(r[0]))


@pytest.mark.parametrize("exclusive", [False, True])
def test_float_sum_scan_2p28_every_element_within_r22(exclusive):
    """float32 SUM scan of 2^28 signed U[-1, 1) elements (the bench size):
    every element within R22's bound of the exact prefix sum, chunk by chunk
    (bigcheck.chunked_float_scan_compare)."""
    n = 1 << 28
    x = synth.device_fill(synth.F32_S11, 6, n, device=DEV)
    out = G.scan(x, exclusive=exclusive)
    del x
    free()

    def fetch(start, m, dest):
        torch.from_numpy(dest).copy_(out[start:start + m])
    compared, bad, first, worst = bigcheck.chunked_float_scan_compare(fetch, n, synth.F32_S11, 6, np.float32,
                                                                      exclusive)
    assert compared == n
    assert bad == 0, f"{bad} elements outside R22, first at {first}"
    assert worst < 1.0
    del out
    free()


def test_c5_sharded_decomposition_8_shards_2p33():
    """C5 as the 8-GPU run computes it, on one GPU: 8 contiguous shards of
    2^30 (R16), each rank's total T_g by the reduction kernel, then each
    shard scanned with carry-in T_0 + ... + T_{g-1} (R18, the kernels
    gpuarray_scan_sharded runs around its allgather); the concatenated output
    is compared whole against the unsharded chunked oracle."""
    n, world = 1 << 33, 8
    need_bytes(2 * n * 4)
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=DEV)
    out = torch.empty_like(k)
    totals = torch.empty(world, dtype=torch.int32, device=DEV)
    bounds = [(g * n) // world for g in range(world + 1)]
    for g in range(world):
        G.sum(k[bounds[g]:bounds[g + 1]], out=totals[g:g + 1])
    for g in range(world):  # rank g's carry: the totals of ranks < g (empty for rank 0)
        G.scan(k[bounds[g]:bounds[g + 1]], exclusive=True, out=out[bounds[g]:bounds[g + 1]],
               carry=totals[:g] if g else None)
    del k
    free()
    _check_scan_full(out, n, synth.I32_RANGE, 3, 0, 9, np.int32, exclusive=True)
    del out
    free()
