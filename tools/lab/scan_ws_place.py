"""Does the scan's time depend on where its workspace (ticket + look-back
status words) sits in memory?  (tuning lab, GPU only)  One library, the int32
exclusive scan at 2^28, the workspace at several offsets inside one buffer,
offsets interleaved per rep, events around each call, median of reps.
    python tools/lab/scan_ws_place.py [LIB]"""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tools/lab")
from ab_scan import load  # noqa: E402

GA_I32 = 2


def main():
    lib = load(sys.argv[1] if len(sys.argv) > 1 else "paper_1304_5553_b200/libgpuarray.so")
    dev = torch.device("cuda:0")
    n = 1 << 28
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    need = lib.gpuarray_scan_workspace_bytes(GA_I32, n)
    buf = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    # disjoint regions (each zeroed once, never shared)
    offs = [0, (3 << 20) + 4096, (6 << 20) + 65536, 9 << 20, (12 << 20) + 512, 15 << 20, (18 << 20) + 2048, (21 << 20) + 8192]
    s = torch.cuda.current_stream().cuda_stream
    res = {o_: [] for o_ in offs}
    for rep in range(31):
        for off in (offs if rep % 2 == 0 else offs[::-1]):
            ws = buf[off:off + need]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert lib.gpuarray_scan(0, 1, GA_I32, GA_I32, n, k.data_ptr(), o.data_ptr(), None, 0, ws.data_ptr(),
                                     need, s) == 0
            e1.record()
            torch.cuda.synchronize()
            if rep:
                res[off].append(e0.elapsed_time(e1) * 1e3)
    base = buf.data_ptr()
    for off in offs:
        v = res[off]
        print(f"ws at base+{off:>10d} (addr %#x): median {statistics.median(v):7.1f} us  min {min(v):7.1f}"
              % (base + off), flush=True)


if __name__ == "__main__":
    main()
