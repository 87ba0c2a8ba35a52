"""GPU tests of the sharded C entry points (include/gpuarray.h:
gpuarray_reduce_sharded / gpuarray_scan_sharded; SURVEY.md §8(a) a6/a7,
§8(b)) with a real NCCL communicator: torch's ProcessGroupNCCL at world size
1 on cuda:0 (one GPU per rank is all NCCL allows; the multi-rank run is
tests/test_multigpu_torchrun.py, which needs >= 2 GPUs).  At world 1 the
global array is the shard, so every result is compared with the CPU oracle
on the whole array: bit-exact for integers and max/min, R10/R11 tolerance
for float sums.  The process group is created in a child process so that no
NCCL state leaks into the other tests of the session."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    try:
        import torch.distributed as dist

        from paper_1304_5553_b200 import _abi
        from paper_1304_5553_b200 import dist as gdist
        from paper_1304_5553_b200 import gpuarray as G
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        comm = gdist.nccl_comm()
        res = {"comm": bool(comm)}
        n = 1_000_003
        x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
        y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
        k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
        kw = synth.device_fill(synth.I32_RANGE, 4, n, lo=-(1 << 31), hi=(1 << 31) - 1, device=dev)
        d = synth.device_fill(synth.F64_S11, 5, n, device=dev)
        res["dot"] = float(G.reduce(G.SUM, G.MUL, x, y, nccl_comm=comm).item())
        res["sum"] = float(gdist.reduce(G.SUM, G.ID, x).item())                     # dist -> C entry
        res["norm2_f64"] = float(G.reduce(G.SUM, G.SQUARE, x, out_dtype=torch.float64, nccl_comm=comm).item())
        res["isum"] = int(G.reduce(G.SUM, G.ID, kw, nccl_comm=comm).item())
        res["isum64"] = int(G.reduce(G.SUM, G.ID, kw, out_dtype=torch.int64, nccl_comm=comm).item())
        res["dmax"] = float(G.reduce(G.MAX, G.ID, d, nccl_comm=comm).item())
        res["imin"] = int(G.reduce(G.MIN, G.ID, kw, nccl_comm=comm).item())
        res["empty"] = float(G.reduce(G.MAX, G.ID, x[:0], nccl_comm=comm).item())
        for ex in (False, True):
            res[f"scan{int(ex)}"] = gdist.scan(k, exclusive=ex).cpu().numpy()
            res[f"wscan{int(ex)}"] = G.scan(kw, exclusive=ex, out_dtype=torch.int64, nccl_comm=comm).cpu().numpy()
        res["maxscan"] = G.scan(kw, op=G.MAX, nccl_comm=comm).cpu().numpy()
        carry = torch.tensor([7, -3, 1 << 30], dtype=torch.int32, device=dev)
        res["carryscan"] = G.scan(k, exclusive=True, carry=carry, nccl_comm=comm).cpu().numpy()
        res["scan_empty"] = G.scan(k[:0], nccl_comm=comm).numel()
        # bad communicator pointer is caught by NCCL, not by a crash
        res["null_comm"] = _abi.gpuarray_reduce_sharded(0, 0, 0, 0, 4, x.data_ptr(), None, y.data_ptr(),
                                                        G.workspace("reduce", dev, G._stream(x), 1).data_ptr(),
                                                        _abi.gpuarray_reduce_workspace_bytes(0, 4), None,
                                                        G._stream(x))
        torch.cuda.synchronize()
        dist.destroy_process_group()
        q.put(("ok", res))
    except Exception as e:  # report to the parent
        import traceback
        q.put(("err", traceback.format_exc() + repr(e)))


@pytest.fixture(scope="module")
def results():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_port(), q))
    p.start()
    status, res = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", res
    return res


def _tol_ok(got, ref, sa, n, rel, u):
    return abs(got - ref) <= max(rel * abs(ref), n * u * sa)


def test_reduce_sharded_world1(results):
    n = 1_000_003
    xh = synth.host_fill(synth.F32_U01, 1, n)
    yh = synth.host_fill(synth.F32_U01, 2, n)
    kw = synth.host_fill(synth.I32_RANGE, 4, n, lo=-(1 << 31), hi=(1 << 31) - 1)
    dh = synth.host_fill(synth.F64_S11, 5, n)
    assert results["comm"]
    ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_MUL, xh, yh, return_sumabs=True)
    assert abs(results["dot"] - ref) <= 1e-5 * abs(ref)
    ref = oracle.reduce(oracle.SUM, oracle.MAP_ID, xh)
    assert abs(results["sum"] - ref) <= 1e-5 * abs(ref)
    ref, sa = oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, xh, out_dtype=np.float64, return_sumabs=True)
    assert _tol_ok(results["norm2_f64"], ref, sa, n, 1e-12, 2.0 ** -53)
    assert results["isum"] == oracle.reduce(oracle.SUM, oracle.MAP_ID, kw)
    assert results["isum64"] == oracle.reduce(oracle.SUM, oracle.MAP_ID, kw, out_dtype=np.int64)
    assert results["dmax"] == oracle.reduce(oracle.MAX, oracle.MAP_ID, dh)
    assert results["imin"] == oracle.reduce(oracle.MIN, oracle.MAP_ID, kw)
    assert results["empty"] == -np.inf  # n == 0 on a rank: the neutral, still allreduced


def test_scan_sharded_world1(results):
    n = 1_000_003
    k = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=9)
    kw = synth.host_fill(synth.I32_RANGE, 4, n, lo=-(1 << 31), hi=(1 << 31) - 1)
    for ex in (False, True):
        kind = oracle.EXCLUSIVE if ex else oracle.INCLUSIVE
        np.testing.assert_array_equal(results[f"scan{int(ex)}"], oracle.scan(kind, k))
        np.testing.assert_array_equal(results[f"wscan{int(ex)}"], oracle.scan(kind, kw, out_dtype=np.int64))
    np.testing.assert_array_equal(results["maxscan"], oracle.scan(oracle.INCLUSIVE, kw, op=oracle.MAX))
    with np.errstate(over="ignore"):
        c = np.add.reduce(np.array([7, -3, 1 << 30], np.int32), dtype=np.int32)
    np.testing.assert_array_equal(results["carryscan"], oracle.scan(oracle.EXCLUSIVE, k, carry=c))
    assert results["scan_empty"] == 0


def test_null_comm_is_an_argument_error(results):
    assert results["null_comm"] == 1  # GA_ERR_INVALID_ARGUMENT


def _symm_worker(port, q):
    """dist.Exchange.symmetric (torch symmetric memory + rendezvous) at world
    size 1, then the fused in-kernel finish (gpuarray_reduce_xgpu) through it."""
    try:
        import torch.distributed as dist

        from paper_1304_5553_b200 import dist as gdist
        from paper_1304_5553_b200 import gpuarray as G
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        xch = gdist.Exchange.symmetric(device=dev)
        n = 777_777
        x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
        k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
        res = {"rank": xch.rank, "world": xch.world}
        res["sum"] = float(gdist.reduce_fused(G.SUM, G.ID, x, exchange=xch).item())
        res["isum"] = int(gdist.reduce_fused(G.SUM, G.ID, k, exchange=xch).item())
        res["scan"] = gdist.scan_fused(k, exclusive=True, exchange=xch).cpu().numpy()
        res["seq"] = xch.seq
        torch.cuda.synchronize()
        dist.destroy_process_group()
        q.put(("ok", res))
    except Exception as e:
        import traceback
        q.put(("err", traceback.format_exc() + repr(e)))


def test_symmetric_exchange_world1():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_worker, args=(_port(), q))
    p.start()
    status, res = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", res
    n = 777_777
    xh = synth.host_fill(synth.F32_U01, 1, n)
    k = synth.host_fill(synth.I32_RANGE, 3, n, lo=0, hi=9)
    assert (res["rank"], res["world"]) == (0, 1)
    ref = oracle.reduce(oracle.SUM, oracle.MAP_ID, xh)
    assert abs(res["sum"] - ref) <= 1e-5 * abs(ref)
    assert res["isum"] == oracle.reduce(oracle.SUM, oracle.MAP_ID, k)
    np.testing.assert_array_equal(res["scan"], oracle.scan(oracle.EXCLUSIVE, k))
    assert res["seq"] == 3
