"""Fused cross-GPU finish (NEXT-1), exercised on one GPU: `world` virtual
ranks, each on its own CUDA stream with its own exchange buffer, launch
gpuarray_reduce_xgpu concurrently; every rank's last block stores its local
result into every buffer and folds all slots in rank order.  The results
must be identical on all ranks and equal to the unsharded oracle — over
repeated calls (sequence parity / slot reuse), all ops and maps, and an
empty shard."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402

if torch.cuda.is_available():
    from paper_1304_5553_b200 import _abi
    from paper_1304_5553_b200 import dist as gdist
    from paper_1304_5553_b200 import gpuarray as G

DEV = "cuda:0"

# NOTE on the single-GPU emulation: the virtual ranks' kernels wait for each
# other, so the host must be able to launch every rank's kernels without
# blocking in between — all buffers (outputs, workspaces) are allocated before
# the launches, because a cudaMalloc inside the launch loop may synchronise
# the device while rank 0's kernel is waiting for rank 1's launch; likewise
# every kernel is launched once beforehand, because CUDA's lazy module
# loading synchronises on a function's first launch.  (Real ranks live in
# separate processes on separate GPUs and do not block each other this way.)


def prealloc(streams, dtype, n):
    for st in streams:
        G.workspace("reduce", torch.device(DEV), st.cuda_stream, _abi.gpuarray_reduce_workspace_bytes(0, 0))
        G.workspace("scan", torch.device(DEV), st.cuda_stream, _abi.gpuarray_scan_workspace_bytes(G.ga_dtype(dtype), n))


def make_ranks(world):
    nbytes = _abi.gpuarray_xgpu_buffer_bytes()
    bufs = [torch.zeros(nbytes, dtype=torch.uint8, device=DEV) for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    return [gdist.Exchange(peers, r, world, keepalive=bufs) for r in range(world)]


def run_all(exchs, shards, op, map_, out_dtype, streams):
    outs = [torch.empty((), dtype=out_dtype or x.dtype, device=DEV) for x, _ in shards]
    prealloc(streams, shards[0][0].dtype, 0)
    torch.cuda.synchronize()  # inputs were produced on the default stream
    for ex, (x, y), st, o in zip(exchs, shards, streams, outs):
        with torch.cuda.stream(st):
            gdist.reduce_fused(op, map_, x, y, out_dtype=out_dtype, exchange=ex, out=o)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_fused_reduce_matches_oracle(world):
    n = 2_000_003
    exchs = make_ranks(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    xh = synth.host_fill(synth.F32_S11, 1, n)
    yh = synth.host_fill(synth.F32_S11, 2, n)
    kh = synth.host_fill(synth.I32_RANGE, 3, n, lo=-1000, hi=1000)
    spans = [gdist.shard_range(n, world, r) for r in range(world)]
    fx = [torch.from_numpy(xh[s:s + c]).to(DEV) for s, c in spans]
    fy = [torch.from_numpy(yh[s:s + c]).to(DEV) for s, c in spans]
    ik = [torch.from_numpy(kh[s:s + c]).to(DEV) for s, c in spans]
    for rep in range(3):  # repeated calls: both slot parities, reuse
        outs = run_all(exchs, list(zip(fx, fy)), G.SUM, G.MUL, torch.float64, streams)
        ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_MUL, xh, yh, return_sumabs=True)
        assert all(o.tobytes() == outs[0].tobytes() for o in outs)
        assert abs(float(outs[0]) - ref) <= max(1e-12 * abs(ref), n * 2.0 ** -53 * sa)
        outs = run_all(exchs, list(zip(fx, fy)), G.MAX, G.ID, None, streams)
        assert all(float(o) == oracle.reduce(oracle.MAX, oracle.MAP_ID, xh) for o in outs)
        outs = run_all(exchs, [(k, None) for k in ik], G.SUM, G.SQUARE, torch.int64, streams)
        assert all(int(o) == oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, kh, out_dtype=np.int64) for o in outs)
        outs = run_all(exchs, [(k, None) for k in ik], G.MIN, G.ID, None, streams)
        assert all(int(o) == oracle.reduce(oracle.MIN, oracle.MAP_ID, kh) for o in outs)
    assert all(e.seq == 12 for e in exchs)


def test_fused_reduce_empty_shard():
    world = 3
    exchs = make_ranks(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    xh = synth.host_fill(synth.F64_U01, 5, 1000)
    shards = [torch.from_numpy(xh[:600]).to(DEV), torch.zeros(0, dtype=torch.float64, device=DEV),
              torch.from_numpy(xh[600:]).to(DEV)]
    outs = run_all(exchs, [(s, None) for s in shards], G.SUM, G.ID, None, streams)
    ref = oracle.reduce(oracle.SUM, oracle.MAP_ID, xh)
    assert all(abs(float(o) - ref) <= 1e-12 * ref for o in outs)
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()


def test_fused_reduce_argument_errors():
    ex = make_ranks(2)[0]
    x = torch.ones(10, device=DEV)
    bad = gdist.Exchange(ex.peers, 2, 2)
    with pytest.raises(ValueError):
        gdist.reduce_fused(G.SUM, G.ID, x, exchange=bad)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exclusive", [False, True])
def test_fused_sharded_scan(world, exclusive):
    """Sharded scan with the offset from the fused finish (no collective)."""
    n = 3_000_017
    exchs = make_ranks(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    kh = synth.host_fill(synth.I32_RANGE, 3, n, lo=-(1 << 20), hi=1 << 20)
    spans = [gdist.shard_range(n, world, r) for r in range(world)]
    ks = [torch.from_numpy(kh[s:s + c]).to(DEV) for s, c in spans]
    prealloc(streams, torch.int32, n)
    warm = torch.ones(1 << 20, dtype=torch.int32, device=DEV)
    G.scan(warm, exclusive=exclusive)
    G.reduce(G.SUM, G.ID, warm)
    outs = [torch.empty_like(k) for k in ks]
    offs = [torch.empty(1, dtype=torch.int32, device=DEV) for _ in ks]
    torch.cuda.synchronize()
    for rep in range(2):
        for ex, k, st, o, off in zip(exchs, ks, streams, outs, offs):
            with torch.cuda.stream(st):
                gdist.scan_fused(k, exclusive=exclusive, exchange=ex, out=o, offset=off)
        torch.cuda.synchronize()
        got = np.concatenate([o.cpu().numpy() for o in outs])
        assert np.array_equal(got, oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, kh))


def test_fused_complex_vdot():
    """16-byte (complex128) values through the exchange slots."""
    world = 3
    exchs = make_ranks(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    n = 300_001
    xh = synth.host_fill(synth.F64_S11, 11, 2 * n).view(np.complex128)
    yh = synth.host_fill(synth.F64_S11, 12, 2 * n).view(np.complex128)
    spans = [gdist.shard_range(n, world, r) for r in range(world)]
    shards = [(torch.from_numpy(xh[s:s + c]).to(DEV), torch.from_numpy(yh[s:s + c]).to(DEV)) for s, c in spans]
    warm = torch.ones(64, dtype=torch.complex128, device=DEV)
    G.vdot(warm, warm)
    for rep in range(2):
        outs = run_all(exchs, shards, G.SUM, G.CONJ_MUL, None, streams)
        ref, sa = oracle.reduce_complex(oracle.MAP_CONJ_MUL, xh, yh, return_sumabs=True)
        assert all(o.tobytes() == outs[0].tobytes() for o in outs)
        assert abs(complex(outs[0]) - ref) <= max(1e-12 * abs(ref), 2 * n * 2.0 ** -53 * sa)
