"""Our exclusive/inclusive scan vs torch.cumsum (CUB DeviceScan) at one-call
granularity with the L2 flushed before each call (tools/sweep.py protocol)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1304_5553_b200 import gpuarray as G  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(512 * 2 ** 20 // 4, device=dev)
clean = torch.ones(512 * 2 ** 20 // 4, device=dev)
sink = torch.empty((), device=dev)


def t(fn, reps=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        G.sum(clean, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for dt in (torch.int32, torch.int64):
    for lg in (20, 22, 24, 26, 28, 30):
        n = 1 << lg
        x = torch.randint(0, 10, (n,), dtype=dt, device=dev)
        out = torch.empty_like(x)
        esz = x.element_size()
        a = t(lambda: G.scan(x, out=out))
        b = t(lambda: torch.cumsum(x, 0, out=out))
        assert torch.equal(G.scan(x), torch.cumsum(x, 0, dtype=x.dtype))
        print(f"{dt} 2^{lg}: ours {a:.1f}us ({2*esz*n/a/1e3:.0f} GB/s)  torch.cumsum {b:.1f}us ({2*esz*n/b/1e3:.0f} GB/s)",
              flush=True)
        del x, out
        torch.cuda.empty_cache()
