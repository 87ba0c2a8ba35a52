"""Run each hot-path op a few times at n = 2^log2n (for ncu captures).
    python tools/profile_ops.py [log2n] [ops...]   ops: axpbyz dot sum norm2 scan scan64 axpbyz64 norm2_64 max"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_1304_5553_b200 import gpuarray as G

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ops = sys.argv[2:] or ["axpbyz", "dot", "sum", "norm2", "scan"]
n = 1 << lg
dev = torch.device("cuda:0")
x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
z = torch.empty_like(x)
s = torch.empty_like(k)
need64 = any(o.endswith("64") for o in ops)
if need64:
    x64 = synth.device_fill(synth.F64_U01, 1, n, device=dev)
    y64 = synth.device_fill(synth.F64_U01, 2, n, device=dev)
    k64 = synth.device_fill(synth.I64_RANGE, 3, n, lo=0, hi=9, device=dev)
    z64 = torch.empty_like(x64)
    s64 = torch.empty_like(k64)
r = torch.empty(1, device=dev)
r64 = torch.empty(1, dtype=torch.float64, device=dev)
for rep in range(3):
    for op in ops:
        if op == "axpbyz":
            G.axpbyz(5.0, x, 6.0, y, out=z)
        elif op == "dot":
            G.reduce(G.SUM, G.MUL, x, y, out=r)
        elif op == "sum":
            G.reduce(G.SUM, G.ID, x, out=r)
        elif op == "norm2":
            G.reduce(G.SUM, G.SQUARE, x, out=r)
        elif op == "max":
            G.reduce(G.MAX, G.ID, x, out=r)
        elif op == "scan":
            G.scan(k, exclusive=True, out=s)
        elif op == "scan64":
            G.scan(k64, exclusive=False, out=s64)
        elif op == "axpbyz64":
            G.axpbyz(5.0, x64, 6.0, y64, out=z64)
        elif op == "norm2_64":
            G.reduce(G.SUM, G.SQUARE, x64, out=r64)
torch.cuda.synchronize()
print("done", lg, ops)
