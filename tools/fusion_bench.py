"""The paper's one "where the time goes" claim for this path (SURVEY §8(d),
optional fusion evidence): evaluating z = a*x + b*y with temporaries,
"a new temporary ... for each intermediate result",
against ElementwiseKernel's "single pass".

  fused     gpuarray_axpbyz                         12 B/elt fp32 (read x, y; write z)
  unfused   t = a*x; u = b*y; z = t + u              28 B/elt (8 + 8 + 12), our kernels:
            axpbz(a, x, -0) -> t, axpbz(b, y, -0) -> u, axpbyz(1, t, 1, u) -> z
            (adding -0.0 and scaling by 1 are exact: the bits equal the fused result)
  torch     a * x + b * y in eager PyTorch (three kernels, two temporaries)

Back-to-back calls (working sets >> L2 at the sizes timed), CUDA events,
median of 20.  python tools/fusion_bench.py [--out gpurun_out/fusion.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402


def med(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


rows = []
dev = torch.device("cuda:0")
for dt in (torch.float32, torch.float64):
    for lg in (24, 26, 28):
        n = 1 << lg
        kind = synth.F32_U01 if dt == torch.float32 else synth.F64_U01
        x = synth.device_fill(kind, 1, n, device=dev)
        y = synth.device_fill(kind, 2, n, device=dev)
        z, t, u = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        a, b = 5.0, -6.0

        def unfused():
            G.axpbz(a, x, -0.0, out=t)
            G.axpbz(b, y, -0.0, out=u)
            G.axpbyz(1.0, t, 1.0, u, out=z)

        fused_ms = med(lambda: G.axpbyz(a, x, b, y, out=z))
        zf = z.clone()
        unfused_ms = med(unfused)
        assert torch.equal(z.view(torch.int32 if dt == torch.float32 else torch.int64),
                           zf.view(torch.int32 if dt == torch.float32 else torch.int64))
        torch_ms = med(lambda: a * x + b * y)
        esz = x.element_size()
        row = {"dtype": str(dt).replace("torch.", ""), "log2n": lg, "fused_ms": round(fused_ms, 4),
               "unfused_ms": round(unfused_ms, 4), "torch_eager_ms": round(torch_ms, 4),
               "unfused_over_fused": round(unfused_ms / fused_ms, 3), "torch_over_fused": round(torch_ms / fused_ms, 3),
               "bytes_ratio": 28 / 12, "fused_gbs": round(3 * esz * n / (fused_ms * 1e-3) / 1e9, 1),
               "unfused_gbs": round(7 * esz * n / (unfused_ms * 1e-3) / 1e9, 1), "bits_equal": True}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del x, y, z, t, u, zf
        torch.cuda.empty_cache()
path = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "gpurun_out", "fusion.json")
json.dump(rows, open(path, "w"), indent=0)
