"""CG workload timing (NEXT-4): host-scalar iteration vs the CUDA-graph
iteration with device-resident scalars (GraphCG: graph captured once,
solve() timed), unfused (6 kernels) and fused (2 kernels:
gpuarray_cg_direction + gpuarray_cg_update).  Fixed 64 iterations
(rtol = 0) of a diagonally dominant tridiagonal system, fp32 and fp64.
Algorithmic bytes per iteration and element: unfused stencil 2, dot 2, three
axpbyz 3 each, norm2 1 -> 14 element-sizes; fused 4 + 6 = 10.  "gbs" is each
variant's own algorithmic bytes / time (its roofline fraction); compare
variants by us_per_iter.

    python tools/cg_bench.py [--out gpurun_out/cg_bench.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import cg as gcg  # noqa: E402

rows = []
for dt in (torch.float32, torch.float64):
    for lg in (14, 16, 18, 20, 22, 24, 26):
        n = 1 << lg
        kind = synth.F32_S11 if dt == torch.float32 else synth.F64_S11
        b = synth.device_fill(kind, 7, n, device="cuda:0")
        out = {"dtype": str(dt).replace("torch.", ""), "log2n": lg}
        solver = gcg.GraphCG(n, dt, d=4.0, block=16, fused=False)
        fsolver = gcg.GraphCG(n, dt, d=4.0, block=16, fused=True)
        for name, fn, elts in (("host", lambda: gcg.cg(b, d=4.0, rtol=0.0, maxiter=64), 14),
                               ("graph", lambda: solver.solve(b, rtol=0.0, maxiter=64), 14),
                               ("graph_fused", lambda: fsolver.solve(b, rtol=0.0, maxiter=64), 10)):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 3
            for _ in range(reps):
                res = fn()
            torch.cuda.synchronize()
            dt_s = (time.perf_counter() - t0) / reps
            it_us = dt_s / res.iterations * 1e6
            esz = 4 if dt == torch.float32 else 8
            out[name] = {"us_per_iter": round(it_us, 2), "gbs": round(elts * esz * n / (it_us * 1e-6) / 1e9, 1),
                         "elt_sizes": elts, "iterations": res.iterations}
        rows.append(out)
        print(json.dumps(out), flush=True)
path = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "gpurun_out", "cg_bench.json")
json.dump(rows, open(path, "w"), indent=0)
