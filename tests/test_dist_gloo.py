"""Host logic of the sharded path (paper_1304_5553_b200/dist.py) under a real
world_size-2 process group on CPU (gloo).  The local GPU operations are
replaced by a CPU stand-in built on the oracle (this is a test), so what is
checked here is the sharding arithmetic, the collective choreography
(scalar allreduce; allgather of shard totals -> carry-in) and that every
rank ends with the global result of the unsharded oracle."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1304_5553_b200 import dist as gdist

_NP = {torch.float32: np.float32, torch.float64: np.float64, torch.int32: np.int32, torch.int64: np.int64}


class OracleOps:
    """CPU stand-in for CudaOps with the same call signatures."""

    def reduce(self, op, map_, x, y=None, out_dtype=None, out=None):
        xn = x.numpy()
        yn = y.numpy() if y is not None else None
        out_dtype = out_dtype or x.dtype
        r = oracle.reduce(op, map_, xn, yn, out_dtype=_NP[out_dtype])
        if out is None:
            out = torch.empty((), dtype=out_dtype)
        out.view(-1)[0] = float(r) if out_dtype.is_floating_point else int(r)
        return out

    def scan(self, x, exclusive=False, out=None, carry=None):
        c = 0
        if carry is not None and carry.numel():
            with np.errstate(over="ignore"):
                c = np.add.reduce(carry.numpy(), dtype=carry.numpy().dtype)
        r = oracle.scan(oracle.EXCLUSIVE if exclusive else oracle.INCLUSIVE, x.numpy(), carry=c)
        if out is None:
            return torch.from_numpy(r)
        out.copy_(torch.from_numpy(r))
        return out


def test_shard_range():
    for n in (0, 1, 7, 100, 2 ** 33 + 3):
        for world in (1, 2, 3, 8):
            spans = [gdist.shard_range(n, world, g) for g in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        gdist.shard_range(10, 2, 2)


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OracleOps()
        start, cnt = gdist.shard_range(n, world, rank)
        x = torch.from_numpy(synth.host_fill(synth.F64_S11, 1, cnt, start=start))
        y = torch.from_numpy(synth.host_fill(synth.F64_S11, 2, cnt, start=start))
        k = torch.from_numpy(synth.host_fill(synth.I32_RANGE, 3, cnt, start=start, lo=-(1 << 30), hi=1 << 30))
        res = {}
        res["dot"] = float(gdist.reduce(0, 1, x, y, ops=ops))
        res["max"] = float(gdist.reduce(1, 0, x, ops=ops))
        res["min"] = float(gdist.reduce(2, 0, x, ops=ops))
        red = torch.empty(3, dtype=torch.float64)
        gdist.reduce_many([(1, x, y), (0, x, None), (2, x, None)], red, ops=ops)
        res["many"] = red.tolist()
        res["isum"] = int(gdist.reduce(0, 0, k, ops=ops, out_dtype=torch.int64))
        for ex in (False, True):
            s = gdist.scan(k, exclusive=ex, ops=ops)
            res[f"scan{int(ex)}"] = (start, s.numpy().copy())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 100_003), (3, 5), (2, 1)])
def test_sharded_equals_unsharded_oracle(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = synth.host_fill(synth.F64_S11, 1, n)
    y = synth.host_fill(synth.F64_S11, 2, n)
    k = synth.host_fill(synth.I32_RANGE, 3, n, lo=-(1 << 30), hi=1 << 30)
    dot = oracle.reduce(oracle.SUM, oracle.MAP_MUL, x, y)
    for r in range(world):
        res = out[r]
        assert res["dot"] == pytest.approx(dot, rel=1e-12, abs=1e-9)
        assert res["max"] == oracle.reduce(oracle.MAX, oracle.MAP_ID, x)
        assert res["min"] == oracle.reduce(oracle.MIN, oracle.MAP_ID, x)
        assert res["many"][0] == pytest.approx(dot, rel=1e-12, abs=1e-9)
        assert res["many"][1] == pytest.approx(oracle.reduce(oracle.SUM, oracle.MAP_ID, x), rel=1e-12, abs=1e-9)
        assert res["isum"] == oracle.reduce(oracle.SUM, oracle.MAP_ID, k, out_dtype=np.int64)
        # all ranks hold identical bits for the reductions
        assert res["dot"] == out[0]["dot"] and res["many"] == out[0]["many"]
    for ex in (0, 1):
        glob = oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, k)
        parts = sorted((out[r][f"scan{ex}"] for r in range(world)), key=lambda sp: sp[0])
        got = np.concatenate([p for _, p in parts]) if parts else np.zeros(0, np.int32)
        assert np.array_equal(got, glob)
