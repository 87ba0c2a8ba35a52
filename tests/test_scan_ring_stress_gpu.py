"""Stress test of the ring scan (scan_ring.cuh): its roles (producer,
fold, look-back, data warps) meet through mbarriers, per-use rings of
slots and the workspace ticket, so an ordering bug would show up as a
rare wrong tile, not a systematic one.  compute-sanitizer's racecheck /
synccheck are closed on the GPU pool, so instead every configuration is run
hundreds of times back to back (no host sync in between) and every result
is compared bit for bit on the device with the first one, which itself is
checked against the CPU oracle.  Configurations: int32 / int64 / widening,
inclusive and exclusive, carry-in, in place, ragged tails, sizes at both
ends of the window, PDL chains of different kernels in between."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"
REPS = 1000


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("case", ["i32_excl", "i32_incl_carry", "i64_incl", "i32_to_i64", "f32_max_tail"])
def test_ring_repeated_bit_identical(case):
    if case.startswith("i64"):
        n = (64 << 20) // 8 + 1
        x = np.random.default_rng(81).integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    elif case.startswith("f32"):
        n = (48 << 20) // 4 + 3                               # lower edge, 3-element tail past a 16-byte multiple
        x = synth.host_fill(synth.F32_S11, 82, n)
    else:
        n = (96 << 20) // 4 + 2
        x = synth.host_fill(synth.I32_RANGE, 83, n, lo=-(1 << 30), hi=1 << 30)
    xd = _dev(x)
    carry = _dev(np.array([7, -3], x.dtype)) if case == "i32_incl_carry" else None
    kw = dict(exclusive=case.endswith("excl"), carry=carry,
              op=G.MAX if case.startswith("f32") else G.SUM,
              out_dtype=torch.int64 if case == "i32_to_i64" else None)
    first = G.scan(xd, **kw)
    kind = oracle.EXCLUSIVE if kw["exclusive"] else oracle.INCLUSIVE
    if case == "i32_incl_carry":
        with np.errstate(over="ignore"):
            ref = oracle.scan(kind, x, carry=np.int32(4))
    elif case == "i32_to_i64":
        ref = oracle.scan(kind, x, out_dtype=np.int64)
    elif case.startswith("f32"):
        ref = oracle.scan(kind, x, op=oracle.MAX)
    else:
        ref = oracle.scan(kind, x)
    assert np.array_equal(first.cpu().numpy(), ref)
    bad = torch.zeros((), dtype=torch.int64, device=DEV)
    out = torch.empty_like(first)
    y = torch.empty(n, dtype=torch.float32, device=DEV)
    for r in range(REPS):
        G.scan(xd, out=out, **kw)
        bad += (out != first).sum()
        if r % 10 == 0:  # other kernels in the PDL chain between ring launches
            G.sum(xd if xd.dtype != torch.int64 else xd[: n // 2])
            G.axpbz(2.0, y, 1.0, out=y)
    assert int(bad.item()) == 0, f"{case}: {int(bad.item())} elements differed over {REPS} runs"


def test_ring_in_place_repeated():
    """In place: the output overwrites the input tile by tile while other
    CTAs' bulk copies read later tiles; each run re-copies the input."""
    n = (128 << 20) // 4 + 5
    x = synth.host_fill(synth.I32_RANGE, 84, n, lo=0, hi=9)
    ref = _dev(oracle.scan(oracle.EXCLUSIVE, x))
    src = _dev(x)
    buf = torch.empty_like(src)
    bad = torch.zeros((), dtype=torch.int64, device=DEV)
    for _ in range(300):
        buf.copy_(src)
        G.scan(buf, exclusive=True, out=buf)
        bad += (buf != ref).sum()
    assert int(bad.item()) == 0
