"""Worker for tests/test_multigpu_torchrun.py (run under torchrun, one rank
per GPU, NCCL): the sharded reductions and scans of a global array split
contiguously over the ranks (ragged shards), through BOTH cross-GPU paths —
the C entries with NCCL (gpuarray_reduce_sharded / gpuarray_scan_sharded via
paper_1304_5553_b200.dist) and the fused in-kernel NVLink finish
(gpuarray_reduce_xgpu over torch symmetric memory) — each rank checking its
results against the CPU oracle of the UNSHARDED global array: integers and
max/min bit-exact, float sums within R10.  Writes one JSON verdict per rank
to $MGPU_OUT/rank<r>.json."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1304_5553_b200 import dist as gdist  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = (1 << 24) + 12_345 + world  # ragged shards
    start, cnt = gdist.shard_range(n, world, rank)
    x = synth.device_fill(synth.F32_U01, synth.SEED_X, cnt, start=start, device=dev)
    y = synth.device_fill(synth.F32_U01, synth.SEED_Y, cnt, start=start, device=dev)
    k = synth.device_fill(synth.I32_RANGE, synth.SEED_INT, cnt, start=start, lo=0, hi=9, device=dev)
    xh = synth.host_fill(synth.F32_U01, synth.SEED_X, n)
    yh = synth.host_fill(synth.F32_U01, synth.SEED_Y, n)
    kh = synth.host_fill(synth.I32_RANGE, synth.SEED_INT, n, lo=0, hi=9)
    ref = {"dot": oracle.reduce(oracle.SUM, oracle.MAP_MUL, xh, yh),
           "sum": oracle.reduce(oracle.SUM, oracle.MAP_ID, xh),
           "norm2": oracle.reduce(oracle.SUM, oracle.MAP_SQUARE, xh),
           "max": float(oracle.reduce(oracle.MAX, oracle.MAP_ID, xh)),
           "isum": int(oracle.reduce(oracle.SUM, oracle.MAP_ID, kh))}
    sref = {ex: oracle.scan(oracle.EXCLUSIVE if ex else oracle.INCLUSIVE, kh)[start:start + cnt] for ex in (0, 1)}
    z = G.axpbyz(5.0, x, 6.0, y)
    zref = oracle.axpbyz(np.float32(5), xh[start:start + cnt], np.float32(6), yh[start:start + cnt])

    fails = []

    def close(name, got, want):
        if not abs(got - want) <= 1e-5 * abs(want):
            fails.append(f"{name}: {got} vs {want}")

    def exact(name, got, want):
        if not np.array_equal(got, want):
            fails.append(f"{name}: mismatch")

    exact("axpbyz", z.cpu().numpy().view(np.uint32), zref.view(np.uint32))
    results = {}
    for path in ("nccl", "fused"):
        xch = gdist.Exchange.symmetric(device=dev) if path == "fused" else None

        def red(op, map_, a, b=None):
            if xch is None:
                return gdist.reduce(op, map_, a, b)
            return gdist.reduce_fused(op, map_, a, b, exchange=xch)

        got = {"dot": float(red(G.SUM, G.MUL, x, y).item()), "sum": float(red(G.SUM, G.ID, x).item()),
               "norm2": float(red(G.SUM, G.SQUARE, x).item()), "max": float(red(G.MAX, G.ID, x).item()),
               "isum": int(red(G.SUM, G.ID, k).item())}
        for key in ("dot", "sum", "norm2"):
            close(f"{path}/{key}", got[key], ref[key])
        if got["max"] != ref["max"]:
            fails.append(f"{path}/max")
        if got["isum"] != ref["isum"]:
            fails.append(f"{path}/isum")
        for ex in (0, 1):
            s = gdist.scan(k, exclusive=bool(ex)) if xch is None else gdist.scan_fused(k, exclusive=bool(ex),
                                                                                       exchange=xch)
            exact(f"{path}/scan{ex}", s.cpu().numpy(), sref[ex])
        # every rank must hold identical bits of the float results
        t = torch.tensor([got["dot"], got["sum"], got["norm2"]], dtype=torch.float64, device=dev)
        lo, hi = t.clone(), t.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        if not torch.equal(lo, hi):
            fails.append(f"{path}: ranks disagree")
        results[path] = got
    torch.cuda.synchronize()
    out = os.environ.get("MGPU_OUT", ".")
    with open(os.path.join(out, f"rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "world": world, "n": n, "fails": fails, "results": results}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
