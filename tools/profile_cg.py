"""Drive the fused CG kernels (and their unfused equivalents) a few times at
one size, for ncu captures:  python tools/profile_cg.py [log2n] [f32|f64]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dt = torch.float64 if len(sys.argv) > 2 and sys.argv[2] == "f64" else torch.float32
n = 1 << lg
kind = synth.F32_S11 if dt == torch.float32 else synth.F64_S11
r, p, x, ap = (synth.device_fill(kind, s, n, device="cuda:0") for s in (1, 2, 3, 4))
p2 = torch.empty_like(p)
num = torch.tensor([0.5], dtype=dt, device="cuda:0")
den = torch.tensor([2.0], dtype=dt, device="cuda:0")
for _ in range(3):
    pap = G.cg_direction(r, p, p2, ap, beta_num=num, beta_den=den, d=4.0)
    rr = G.cg_update(x, r, p2, ap, alpha_num=num, alpha_den=den)
    G.stencil3(-1.0, 4.0, -1.0, p2, out=ap)
    G.dot(p2, ap)
    G.axpbyz(1.0, x, 0.5, p2, out=x)
torch.cuda.synchronize()
print("ok", float(pap.item()), float(rr.item()))
