"""GPU regression test: ONE scan workspace shared by scans of every element
size, widening, tile count and super-tile shape (include/gpuarray.h promises
the workspace stays valid after one zero-fill; VERDICT r1 "What's weak" #1).

The look-back status of every tile is a run of 64-bit words that each carry
the call's epoch and flag in their high half (scan_kernel.cuh, Status), so a
word left by an earlier call — of another element size, laid out at another
tile stride — can only show an older epoch.  The sequences below are built to
catch the failure this replaced: int32 MAX scans over U{0..6} / U{0..9} leave
small raw values in the status region (under the round-1 layout those read as
"current epoch, AGGREGATE / INCLUSIVE" flags to a following 8-byte scan),
then int64 SUM, int32 -> int64 and float32 -> float64 scans run on the same
bytes with the next epochs.  Every output is compared with the CPU oracle
bit for bit (integer-valued data, so the float scans are exact too,
DESIGN.md R22).  Calls go straight through the C ABI with one caller-owned
workspace (the Python binding keeps separate workspaces per element size)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import _abi
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"
# S / M / L super-tile shapes for 4-byte and 8-byte scans (scan_impl.cuh
# choose_shape: L from 256 tiles of 98304 (4-byte) / 49152 (8-byte) elements,
# M from 64 tiles of 32768 / 16384) and the ring kernel, which takes scans of
# 48 MiB .. 4 GiB (4-byte) / 2 GiB (8-byte) of input and widening scans
# from 48 MiB (its own ticket-reset rule: every CTA draws one id past the last
# tile).  "R" runs the ring for every scan here; "L" runs the L shape for the
# int64 scans, between ring-kernel int32 and widening scans.
SIZES = {"S": 100_003, "M": 3_000_017, "R": 26_000_003, "L": (2 << 30) // 8 + 4099}
TDT = {np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32, np.float64: torch.float64}
GADT = {np.int32: 2, np.int64: 3, np.float32: 0, np.float64: 1}


def _dev(a, offs=0):
    buf = torch.empty(a.size + offs, dtype=TDT[a.dtype.type], device=DEV)
    v = buf[offs:]
    v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


def _run(ws, op, exclusive, x, out_np_dtype, offs=0):
    """One gpuarray_scan through the C ABI on the shared workspace."""
    xd = _dev(x, offs)
    out = torch.empty(x.size + offs, dtype=TDT[out_np_dtype], device=DEV)[offs:]
    st = _abi.gpuarray_scan(op, _abi.GA_SCAN_EXCLUSIVE if exclusive else _abi.GA_SCAN_INCLUSIVE,
                            GADT[x.dtype.type], GADT[out_np_dtype], x.size, xd.data_ptr(), out.data_ptr(), None, 0,
                            ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    _abi.check(st)
    return out


def _ref(op, exclusive, x, out_np_dtype):
    return oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x, op=op,
                       out_dtype=None if out_np_dtype == x.dtype.type else out_np_dtype)


def _check(got, ref, what):
    g = got.cpu().numpy()
    assert g.dtype == ref.dtype, what
    bad = g != ref
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(f"{what}: {int(bad.sum())} mismatches, first at {i}: gpu={g[i]} oracle={ref[i]}")


@pytest.mark.parametrize("shape", ["S", "M", "R", "L"])
def test_mixed_element_sizes_share_one_workspace(shape):
    n = SIZES[shape]
    nbytes = max(_abi.gpuarray_scan_workspace_bytes(d, SIZES["L"] + 8) for d in (0, 1, 2, 3))
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=DEV)
    k06 = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=6)
    k09 = synth.host_fill(synth.I32_RANGE, 4, n, lo=0, hi=9)
    l09 = k09.astype(np.int64)
    f09 = k09.astype(np.float32)
    # (op, exclusive, input, output dtype): small-value 4-byte MAX scans, then
    # every 8-byte / widened flavour, interleaved so each follows a 4-byte call
    seq = [
        (oracle.MAX, False, k06, np.int32),
        (oracle.SUM, False, l09, np.int64),
        (oracle.MAX, False, k09, np.int32),
        (oracle.SUM, True, k09, np.int64),    # int32 -> int64 widening
        (oracle.MAX, True, k06, np.int32),
        (oracle.SUM, False, f09, np.float64),  # float32 -> float64 widening
        (oracle.MAX, False, k06, np.int32),
        (oracle.SUM, True, l09, np.int64),
        (oracle.SUM, False, k09, np.int32),
        (oracle.MAX, False, l09, np.int64),
    ]
    for rep in range(1 if shape == "L" else 2):
        for op, ex, x, odt in seq:
            got = _run(ws, op, ex, x, odt)
            _check(got, _ref(op, ex, x, odt), f"rep {rep} op {op} ex {ex} {x.dtype}->{np.dtype(odt)} n {n}")


def test_sizes_and_alignments_alternate_on_one_workspace():
    """Tile counts, shapes and the unaligned register kernel (other tile
    size) alternate with element sizes: status of one call lands at tile
    indices the next call reads with a different stride."""
    nbytes = max(_abi.gpuarray_scan_workspace_bytes(d, SIZES["L"] + 8) for d in (0, 1, 2, 3))
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=DEV)
    plan = [(SIZES["R"], 0), (SIZES["S"], 1), (SIZES["M"], 0), (777_777, 1), (SIZES["R"], 1), (SIZES["M"], 3),
            (SIZES["R"], 4), (SIZES["S"], 0)]
    for i, (n, offs) in enumerate(plan):
        k = synth.host_fill(synth.I32_RANGE, 30 + i, n, lo=0, hi=6)
        for op, ex, x, odt in ((oracle.MAX, False, k, np.int32), (oracle.SUM, False, k.astype(np.int64), np.int64),
                               (oracle.SUM, True, k, np.int64)):
            got = _run(ws, op, ex, x, odt, offs)
            _check(got, _ref(op, ex, x, odt), f"plan {i} op {op} {x.dtype}->{np.dtype(odt)} offs {offs}")


def test_ring_scans_on_concurrent_streams():
    """Ring-kernel scans (persistent CTAs holding every SM's shared memory)
    on three streams at once, interleaved with a multi-group reduction on a
    fourth, five rounds without a host sync: each grid draws tiles only while
    its CTAs are resident and no tile waits on another grid, so the scans
    must complete and match the oracle bit for bit (the binding keeps one
    workspace per stream and element size)."""
    n32, n64 = (96 << 20) // 4 + 13, (96 << 20) // 8 + 7
    k = synth.host_fill(synth.I32_RANGE, 70, n32, lo=-(1 << 20), hi=1 << 20)
    l = np.random.default_rng(71).integers(-(1 << 40), 1 << 40, size=n64, dtype=np.int64)
    kd, ld = _dev(k), _dev(l)
    r = synth.device_fill(synth.I32_RANGE, 72, 1 << 26, lo=-100, hi=100, device=DEV)
    rounds = 5
    outs = [[torch.empty(n32, dtype=torch.int32, device=DEV) for _ in range(rounds)],
            [torch.empty(n64, dtype=torch.int64, device=DEV) for _ in range(rounds)],
            [torch.empty(n32, dtype=torch.int64, device=DEV) for _ in range(rounds)]]
    sums = torch.empty(rounds, dtype=torch.int32, device=DEV)
    streams = [torch.cuda.Stream() for _ in range(4)]
    torch.cuda.synchronize()
    for i in range(rounds):
        with torch.cuda.stream(streams[0]):
            G.scan(kd, exclusive=bool(i & 1), out=outs[0][i])
        with torch.cuda.stream(streams[1]):
            G.scan(ld, out=outs[1][i])
        with torch.cuda.stream(streams[2]):
            G.scan(kd, out=outs[2][i], out_dtype=torch.int64)
        with torch.cuda.stream(streams[3]):
            G.reduce(G.SUM, G.ID, r, out=sums[i:i + 1])
    torch.cuda.synchronize()
    ref_k = {ex: oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, k) for ex in (False, True)}
    ref_l = oracle.scan(oracle.INCLUSIVE, l)
    ref_w = oracle.scan(oracle.INCLUSIVE, k, out_dtype=np.int64)
    rh = synth.host_fill(synth.I32_RANGE, 72, 1 << 26, lo=-100, hi=100)
    ref_s = oracle.reduce(oracle.SUM, oracle.MAP_ID, rh)
    for i in range(rounds):
        _check(outs[0][i], ref_k[bool(i & 1)], f"round {i} int32")
        _check(outs[1][i], ref_l, f"round {i} int64")
        _check(outs[2][i], ref_w, f"round {i} int32->int64")
        assert int(sums[i].item()) == ref_s
