"""The sharded path with the REAL CUDA kernels: two processes share cuda:0
(this environment has one GPU) and talk over gloo, which moves CUDA tensors
through the host.  Checks dist.reduce / reduce_many / scan (local reduce ->
allgather of totals -> scan with carry-in) against the unsharded oracle."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist
    from paper_1304_5553_b200 import dist as gdist
    from paper_1304_5553_b200 import gpuarray as G
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, cnt = gdist.shard_range(n, world, rank)
        dev = torch.device("cuda:0")
        x = synth.device_fill(synth.F32_S11, 1, cnt, start=start, device=dev)
        y = synth.device_fill(synth.F32_S11, 2, cnt, start=start, device=dev)
        k = synth.device_fill(synth.I32_RANGE, 3, cnt, start=start, lo=-(1 << 30), hi=1 << 30, device=dev)
        res = {}
        res["dot"] = float(gdist.reduce(G.SUM, G.MUL, x, y, out_dtype=torch.float64).item())
        res["max"] = float(gdist.reduce(G.MAX, G.ID, x).item())
        red = torch.empty(3, dtype=torch.float32, device=dev)
        gdist.reduce_many([(G.MUL, x, y), (G.ID, x, None), (G.SQUARE, x, None)], red)
        res["many"] = red.cpu().tolist()
        for ex in (False, True):
            res[f"scan{int(ex)}"] = (start, gdist.scan(k, exclusive=ex).cpu().numpy())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 3_000_017), (3, 1_000_003)])
def test_sharded_cuda_equals_oracle(world, n):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = synth.host_fill(synth.F32_S11, 1, n)
    y = synth.host_fill(synth.F32_S11, 2, n)
    k = synth.host_fill(synth.I32_RANGE, 3, n, lo=-(1 << 30), hi=1 << 30)
    dot, sa = oracle.reduce(oracle.SUM, oracle.MAP_MUL, x, y, return_sumabs=True)
    s1, sa1 = oracle.reduce(oracle.SUM, oracle.MAP_ID, x, return_sumabs=True)
    n2 = oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, x)
    for r in range(world):
        res = out[r]
        assert abs(res["dot"] - dot) <= max(1e-12 * abs(dot), n * 2.0 ** -53 * sa)
        assert res["max"] == oracle.reduce(oracle.MAX, oracle.MAP_ID, x)
        assert abs(res["many"][0] - dot) <= max(1e-5 * abs(dot), n * 2.0 ** -24 * sa)
        assert abs(res["many"][1] - s1) <= max(1e-5 * abs(s1), n * 2.0 ** -24 * sa1)
        assert abs(res["many"][2] - n2) <= 1e-5 * n2
        assert res["many"] == out[0]["many"] and res["dot"] == out[0]["dot"]
    for ex in (0, 1):
        parts = sorted((out[r][f"scan{ex}"] for r in range(world)), key=lambda sp: sp[0])
        got = np.concatenate([p for _, p in parts])
        assert np.array_equal(got, oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, k))
