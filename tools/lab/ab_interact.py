"""Does the reduction that runs before a scan change the scan's time?
(tuning lab, GPU only).  norm2 (fp32, 2^28) from library X, then the int32
exclusive scan (2^28) from library A, 120 back-to-back pairs per (X, A) as in
bench.py's step (no host sync inside); the scan alone is timed with events.
    python tools/lab/ab_interact.py LIB_NEW LIB_HEAD [norm2|none|sleep]
    python tools/lab/ab_interact.py LIB [mode]       (one library: no mixing)"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tools/lab")
from ab_reduce import load as load_red  # noqa: E402
from ab_scan import load as load_scan  # noqa: E402

GA_F32, GA_I32 = 0, 2


def main():
    paths = sys.argv[1:3] if len(sys.argv) > 2 and sys.argv[2].endswith(".so") else [sys.argv[1]] * 2
    reds = [load_red(p) for p in paths]
    scans = [load_scan(p) for p in paths]
    dev = torch.device("cuda:0")
    n = 1 << 28
    x = torch.rand(n, device=dev)
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    rws = [torch.zeros(lib.gpuarray_reduce_workspace_bytes(GA_F32, n), dtype=torch.uint8, device=dev) for lib in reds]
    sws = [torch.zeros(lib.gpuarray_scan_workspace_bytes(GA_I32, n), dtype=torch.uint8, device=dev) for lib in scans]
    s = torch.cuda.current_stream().cuda_stream
    mode = sys.argv[-1] if sys.argv[-1] in ("norm2", "none", "sleep") else "norm2"

    def pre(i):
        if mode == "none":
            return
        if mode == "sleep":
            torch.cuda._sleep(200000)
            return
        assert reds[i].gpuarray_reduce(0, 2, GA_F32, GA_F32, n, x.data_ptr(), None, out.data_ptr(),
                                       rws[i].data_ptr(), rws[i].numel(), s) == 0

    def scan(j):
        assert scans[j].gpuarray_scan(0, 1, GA_I32, GA_I32, n, k.data_ptr(), o.data_ptr(), None, 0,
                                      sws[j].data_ptr(), sws[j].numel(), s) == 0
    res = {}
    for rnd in range(2):
        for i in (0, 1):
            for j in (0, 1):
                evs = []
                for it in range(120):
                    pre(i)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    scan(j)
                    e1.record()
                    if it >= 20:
                        evs.append((e0, e1))
                torch.cuda.synchronize()
                res.setdefault((i, j), []).extend(a.elapsed_time(b) * 1e3 for a, b in evs)
    names = ["new", "head"]
    for (i, j), v in sorted(res.items()):
        print(f"pre={mode}:{names[i]:4s} scan={names[j]:4s}  {statistics.median(v):8.1f} us  (min {min(v):.1f})")


if __name__ == "__main__":
    main()
