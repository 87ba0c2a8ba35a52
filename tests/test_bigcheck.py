"""The chunked full-size checker itself (CPU, -m "not gpu"): it must find
every kind of wrong element it is meant to catch, and accept a correct
output.  The "device output" here is a host array built from numpy's own
cumsum of the regenerated stream (independent of the oracle's scan), so a
harness that only ever compared the oracle with itself would not pass."""
import numpy as np
import pytest

import bigcheck
import synth


def _numpy_scan(n, kind, seed, lo, hi, dt, exclusive):
    x = synth.host_fill(kind, seed, n, lo=lo, hi=hi).astype(dt)
    inc = np.cumsum(x, dtype=dt)  # wraps modulo 2^w like the method (R4)
    if not exclusive:
        return inc
    out = np.empty_like(inc)
    out[0] = 0
    out[1:] = inc[:-1]
    return out


def _fetch(arr):
    def fetch(start, m, dest):
        dest[:] = arr[start:start + m]
    return fetch


@pytest.mark.parametrize("dt,exclusive", [(np.int32, True), (np.int32, False), (np.int64, False)])
def test_chunked_scan_compare_accepts_a_correct_scan(dt, exclusive):
    kind = synth.I32_RANGE if dt == np.int32 else synth.I64_RANGE
    n = 5 * 4096 + 77  # ragged last chunk
    ref = _numpy_scan(n, kind, 3, 0, 9, dt, exclusive)
    compared, bad, first = bigcheck.chunked_scan_compare(_fetch(ref), n, kind, 3, 0, 9, dt, exclusive, chunk=4096,
                                                         batch=2, procs=2)
    assert (compared, bad, first) == (n, 0, -1)


def test_chunked_scan_compare_wraps_like_int32():
    # U[-2^15, 2^15) data in int32 past 2^31 in magnitude is not needed: a
    # large constant carry makes every chunk carry wrap
    n = 6 * 2048
    x = synth.host_fill(synth.I32_RANGE, 9, n, lo=(1 << 30), hi=(1 << 30) + 9)
    ref = np.cumsum(x, dtype=np.int32)
    compared, bad, _ = bigcheck.chunked_scan_compare(_fetch(ref), n, synth.I32_RANGE, 9, 1 << 30, (1 << 30) + 9,
                                                     np.int32, False, chunk=2048, batch=4, procs=2)
    assert compared == n and bad == 0


@pytest.mark.parametrize("where", ["first", "chunk_edge", "interior", "last"])
def test_chunked_scan_compare_finds_one_wrong_element(where):
    n = 4 * 4096 + 13
    ref = _numpy_scan(n, synth.I32_RANGE, 3, 0, 9, np.int32, True)
    i = {"first": 0, "chunk_edge": 2 * 4096, "interior": 3 * 4096 + 1234, "last": n - 1}[where]
    bad_out = ref.copy()
    bad_out[i] += 1
    compared, bad, first = bigcheck.chunked_scan_compare(_fetch(bad_out), n, synth.I32_RANGE, 3, 0, 9, np.int32,
                                                         True, chunk=4096, batch=3, procs=2)
    assert compared == n and bad == 1 and first == i


def test_chunked_scan_compare_finds_a_shifted_tile():
    # a store error confined to one tile: a block of outputs off by the tile's sum
    n = 8 * 1024
    ref = _numpy_scan(n, synth.I32_RANGE, 3, 0, 9, np.int32, False)
    bad_out = ref.copy()
    bad_out[5000:5512] -= 7
    _, bad, first = bigcheck.chunked_scan_compare(_fetch(bad_out), n, synth.I32_RANGE, 3, 0, 9, np.int32, False,
                                                  chunk=1024, batch=8, procs=2)
    assert bad == 512 and first == 5000


@pytest.mark.parametrize("exclusive", [False, True])
def test_chunked_float_scan_compare(exclusive):
    """A float32 scan computed in float64 and rounded once (far inside R22's
    bound) passes; the same with one element off by 1% of its prefix fails
    exactly there."""
    n, chunk = 3 * 2048 + 91, 2048
    x = synth.host_fill(synth.F32_S11, 5, n).astype(np.float64)
    inc = np.cumsum(x)
    ref = (np.concatenate([[0.0], inc[:-1]]) if exclusive else inc).astype(np.float32)
    res = bigcheck.chunked_float_scan_compare(_fetch(ref), n, synth.F32_S11, 5, np.float32, exclusive, chunk=chunk,
                                              batch=2, procs=2)
    assert res[:3] == (n, 0, -1) and res[3] <= 1.0 / 512  # one rounding: <= u|S_i| <= u sum|x|
    bad = ref.copy()
    i = 2 * 2048 + 17
    bad[i] += np.float32(0.01 * np.sum(np.abs(x[:i + 1])) + 1.0)
    res = bigcheck.chunked_float_scan_compare(_fetch(bad), n, synth.F32_S11, 5, np.float32, exclusive, chunk=chunk,
                                              batch=2, procs=2)
    assert res[1] == 1 and res[2] == i
