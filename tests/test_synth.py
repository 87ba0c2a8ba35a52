"""The shared synthetic generator (synth/): host twin pinned against an
independent pure-Python splitmix64, range and distribution sanity.  CPU only."""
import numpy as np
import pytest

import synth

M64 = (1 << 64) - 1


def py_mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def py_hash(seed, i):
    return py_mix64(((seed << 40) + i) & M64)


def test_splitmix_reference_value():
    # splitmix64 with state 0: first output is 0xe220a8397b1dcdaf (published test vector)
    assert py_mix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("start", [0, 12345, (1 << 33) - 7])
def test_host_twin_matches_python(start):
    n = 64
    f = synth.host_fill(synth.F32_U01, 1, n, start=start)
    d = synth.host_fill(synth.F64_U01, 2, n, start=start)
    s = synth.host_fill(synth.F32_S11, 5, n, start=start)
    s64 = synth.host_fill(synth.F64_S11, 6, n, start=start)
    r = synth.host_fill(synth.I32_RANGE, 3, n, start=start, lo=-5, hi=9)
    full = synth.host_fill(synth.I64_FULL, 4, n, start=start)
    for k in range(n):
        i = start + k
        assert f[k] == np.float32((py_hash(1, i) >> 40) * 2.0 ** -24)
        assert d[k] == (py_hash(2, i) >> 11) * 2.0 ** -53
        assert s[k] == np.float32(((py_hash(5, i) >> 39) - (1 << 24)) * 2.0 ** -24)
        assert s64[k] == ((py_hash(6, i) >> 10) - (1 << 53)) * 2.0 ** -53
        assert r[k] == -5 + (((py_hash(3, i) >> 32) * 15) >> 32)
        h = py_hash(4, i)
        assert full[k] == (h - (1 << 64) if h >= (1 << 63) else h)


def test_shard_consistency():
    whole = synth.host_fill(synth.F32_U01, 1, 1000)
    parts = [synth.host_fill(synth.F32_U01, 1, 250, start=s) for s in (0, 250, 500, 750)]
    assert np.array_equal(whole, np.concatenate(parts))


def test_ranges_and_distribution():
    n = 1 << 20
    u = synth.host_fill(synth.F32_U01, 1, n)
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 2e-3
    s = synth.host_fill(synth.F64_S11, 1, n)
    assert s.min() >= -1 and s.max() < 1 and abs(s.mean()) < 4e-3
    r = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=9)
    assert r.min() == 0 and r.max() == 9
    full = synth.host_fill(synth.I32_RANGE, 3, n, lo=-(1 << 31), hi=(1 << 31) - 1)
    assert full.min() < -(1 << 30) and full.max() > (1 << 30)
    ramp = synth.host_fill(synth.I64_RAMP, 0, 10, start=5, lo=1)
    assert ramp.tolist() == list(range(6, 16))


def test_rejects_bad_range():
    with pytest.raises(ValueError):
        synth.host_fill(synth.I32_RANGE, 3, 10, lo=5, hi=4)
