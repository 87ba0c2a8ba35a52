import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_1304_5553_b200 import gpuarray as G
dev = torch.device("cuda:0")
flush = torch.empty(512 * 2 ** 20 // 4, device=dev); clean = torch.ones(512 * 2 ** 20 // 4, device=dev)
sink = torch.empty((), device=dev)
def t(fn, reps=15, flushit=True):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        if flushit:
            flush.fill_(1.0); G.sum(clean, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort(); return ts[len(ts) // 2]
for lg in (20, 22, 24, 25, 26, 27, 28):
    n = 1 << lg
    x = torch.rand(n, device=dev); y = torch.rand(n, device=dev); z = torch.empty_like(x)
    r = torch.empty((), device=dev)
    a = t(lambda: G.sum(x, out=r)); b = t(lambda: torch.sum(x, dim=0, out=r))
    c = t(lambda: G.axpbyz(1.0, x, 1.0, y, out=z)); d = t(lambda: torch.add(x, y, out=z))
    e = t(lambda: G.sum(x, out=r), flushit=False)
    print(f"2^{lg}: sum ours {a:.1f}us ({4*n/a/1e3:.0f} GB/s) torch {b:.1f}us ({4*n/b/1e3:.0f})  | add ours {c:.1f} ({12*n/c/1e3:.0f}) torch {d:.1f} ({12*n/d/1e3:.0f}) | sum hot {e:.1f}", flush=True)
