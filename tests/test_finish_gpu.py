"""GPU tests of the single-pass reduction finish (R29): epoch-tagged
block-partial slots, group leaders, grid leader.  Grids around the group
size (128 blocks) and the one-group shortcut, values of 4, 8 and 16 bytes
(slot strides 8, 16, 32 B) interleaved on ONE cached workspace, and long
runs of consecutive calls (the epoch advances once per call) — every result
against the CPU oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"
# elements per block of the fp32 / int32 sum (256 threads x 8 vectors x 8 lanes)
PER_BLOCK = 256 * 8 * 8


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("grid", [1, 2, 127, 128, 129, 255, 256, 257, 1000])
def test_int_sum_across_group_boundaries(grid):
    """int32 SUM is bit-exact, so any slot lost, read twice, read stale or
    folded out of its group shows up as a wrong integer."""
    n = grid * PER_BLOCK - 5  # ragged last block
    x = synth.host_fill(synth.I32_RANGE, 11, n, lo=-(1 << 20), hi=1 << 20)
    got = int(G.reduce(G.SUM, G.ID, dev(x)).item())
    assert got == oracle.reduce(oracle.SUM, oracle.MAP_ID, x)


def test_mixed_value_sizes_share_one_workspace():
    """4-, 8- and 16-byte partials (int32 sum, int64 max, float64 norm2,
    complex128 sum) alternate on the binding's single cached workspace: slots
    of different strides overlap, and only the current call's tag counts."""
    n = 257 * PER_BLOCK + 3
    xi = synth.host_fill(synth.I32_RANGE, 12, n, lo=-1000, hi=1000)
    xl = np.random.default_rng(13).integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    xf = synth.host_fill(synth.F64_S11, 14, n)
    re, im = synth.host_fill(synth.F64_S11, 15, n), synth.host_fill(synth.F64_S11, 16, n)
    xc = (re + 1j * im).astype(np.complex128)
    di, dl, df, dc = dev(xi), dev(xl), dev(xf), dev(xc)
    ref_i = oracle.reduce(oracle.SUM, oracle.MAP_ID, xi)
    ref_l = oracle.reduce(oracle.MAX, oracle.MAP_ID, xl)
    ref_f, sa_f = oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, xf, return_sumabs=True)
    ref_c = oracle.reduce_complex(oracle.MAP_ID, xc)
    tol_f = max(1e-12 * abs(ref_f), n * 2.0 ** -53 * sa_f)
    for _ in range(3):
        assert int(G.reduce(G.SUM, G.ID, di).item()) == ref_i
        assert int(G.reduce(G.MAX, G.ID, dl).item()) == ref_l
        assert abs(float(G.reduce(G.SUM, G.SQUARE, df).item()) - ref_f) <= tol_f
        c = complex(G.reduce(G.SUM, G.ID, dc).item())
        assert abs(c - complex(ref_c)) <= 1e-9 * max(1.0, abs(complex(ref_c)))


def test_many_consecutive_calls_each_exact():
    """400 calls back to back without a host sync in between, sizes cycling
    through one-group and multi-group grids; results kept on the device and
    checked at the end (a stale slot from call k-1 accepted by call k would
    give call k's sum a wrong value)."""
    sizes = [5, PER_BLOCK, 128 * PER_BLOCK, 129 * PER_BLOCK + 1, 3 * PER_BLOCK + 7]
    xs = [synth.host_fill(synth.I32_RANGE, 20 + i, m, lo=-50, hi=50) for i, m in enumerate(sizes)]
    ds = [dev(x) for x in xs]
    refs = [oracle.reduce(oracle.SUM, oracle.MAP_ID, x) for x in xs]
    out = torch.empty(400, dtype=torch.int32, device=DEV)
    for k in range(400):
        G.reduce(G.SUM, G.ID, ds[k % len(sizes)], out=out[k:k + 1])
    got = out.cpu().numpy()
    for k in range(400):
        assert int(got[k]) == refs[k % len(sizes)], k


def test_float_sum_deterministic_across_group_shapes():
    """Same data, same grid -> the same bits on every call (the fold order
    depends only on (grid, group), R9)."""
    n = 300 * PER_BLOCK + 11
    x = synth.device_fill(synth.F32_S11, 3, n, device=DEV)
    vals = {float(G.reduce(G.SUM, G.ID, x).item()) for _ in range(8)}
    assert len(vals) == 1


def test_concurrent_large_reductions_on_four_streams():
    """Four multi-group reductions at 2^30 elements run concurrently on four
    streams (256 groups each, 4 x 256 group leaders against ~592 resident
    blocks), ten rounds without a host sync: the finish must make progress
    and every result must be exact (int) / within R10 (float).  Progress
    rests on blocks being dispatched in index order within a grid (a group
    leader is its group's last block, so every block it waits for is already
    resident, whatever the other grids hold; R29)."""
    n = 1 << 30
    free, _ = torch.cuda.mem_get_info()
    if free < 4 * n * 4 * 1.1:
        pytest.skip("needs 16 GiB of free device memory")
    xi = synth.device_fill(synth.I32_RANGE, 31, n, lo=-(1 << 15), hi=(1 << 15) - 1, device=DEV)
    xj = synth.device_fill(synth.I32_RANGE, 32, n, lo=-(1 << 15), hi=(1 << 15) - 1, device=DEV)
    xf = synth.device_fill(synth.F32_U01, 33, n, device=DEV)
    yf = synth.device_fill(synth.F32_U01, 34, n, device=DEV)
    rounds = 10
    outs = [torch.empty(rounds, dtype=dt, device=DEV)
            for dt in (torch.int32, torch.int32, torch.float32, torch.float32)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    for r in range(rounds):
        calls = [lambda o: G.reduce(G.SUM, G.ID, xi, out=o), lambda o: G.reduce(G.MAX, G.ID, xj, out=o),
                 lambda o: G.reduce(G.SUM, G.MUL, xf, yf, out=o), lambda o: G.reduce(G.SUM, G.SQUARE, xf, out=o)]
        for s, call, o in zip(streams, calls, outs):
            with torch.cuda.stream(s):
                call(o[r:r + 1])
    torch.cuda.synchronize()
    got = [o.cpu().numpy() for o in outs]
    del xi, xj, xf, yf
    torch.cuda.empty_cache()
    import bigcheck
    ref_i, _ = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_ID, n, synth.I32_RANGE, 31, lo=-(1 << 15),
                                       hi=(1 << 15) - 1, out_dtype=np.int32)
    ref_j, _ = bigcheck.chunked_reduce(oracle.MAX, oracle.MAP_ID, n, synth.I32_RANGE, 32, lo=-(1 << 15),
                                       hi=(1 << 15) - 1)
    ref_d, _ = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_MUL, n, synth.F32_U01, 33, kind_y=synth.F32_U01,
                                       seed_y=34)
    ref_n, _ = bigcheck.chunked_reduce(oracle.SUM, oracle.MAP_SQUARE, n, synth.F32_U01, 33)
    assert all(int(v) == ref_i for v in got[0])
    assert all(int(v) == ref_j for v in got[1])
    for v in got[2]:
        assert abs(float(v) - ref_d) <= 1e-5 * abs(ref_d)
    for v in got[3]:
        assert abs(float(v) - ref_n) <= 1e-5 * abs(ref_n)
    # a fixed fold order per (grid, group): every round gives the same bits
    assert len(set(got[2].tolist())) == 1 and len(set(got[3].tolist())) == 1
