"""Per-super-tile timeline of the product scan (tuning lab, GPU only): the
L-shape int32 exclusive kernel compiled with TRACE (tile_lab.cu
lab_scan_trace), one traced call at 2^28 after warm-up, with (0) and
without (1) the L2 prefetch.  Results: profiles/r2_scan.md.
    [TRACE_LOG2N=k] python tools/lab/trace_l2.py run | analyze"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
CASES = {0: "prefetch 42 ids ahead (product)", 1: "no prefetch"}


def run():
    import torch
    L = ctypes.CDLL(os.environ.get("TILE_LAB_LIB", os.path.join(HERE, "libtile_lab.so")))
    L.lab_scan_trace.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5
    dev = torch.device("cuda:0")
    n = 1 << int(os.environ.get("TRACE_LOG2N", "28"))
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
    tiles = -(-n // (24 * 32 * 128))
    tr = torch.zeros(8 * tiles, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for v in CASES:
        for _ in range(4):
            assert L.lab_scan_trace(v, n, k.data_ptr(), o.data_ptr(), ws.data_ptr(), tr.data_ptr(), s) == 0
        torch.cuda.synchronize()
        np.save(os.path.join(ROOT, "gpurun_out", f"trace_l2_{v}.npy"), tr.view(-1, 8).cpu().numpy())


def analyze():
    for v, label in CASES.items():
        a = np.load(os.path.join(ROOT, "gpurun_out", f"trace_l2_{v}.npy")).astype(np.int64)
        t0 = a[:, 0].min()
        st, p1, lb, en = [(a[:, i] - t0) / 1e3 for i in range(4)]
        lb = np.where(a[:, 2] > 0, lb, p1)  # tile 0 has no look-back
        print(f"{label}: {len(a)} tiles, span {en.max():.1f} us")
        for name, x in (("phase 1", p1 - st), ("look-back", lb - p1), ("phase 3", en - lb), ("life", en - st)):
            q = np.percentile(x[1:], [10, 50, 90, 99, 100])
            print(f"  {name:10s} mean {x[1:].mean():6.2f}  p10/50/90/99/max " + " ".join(f"{y:6.2f}" for y in q))
        lag = np.maximum.accumulate(p1) - p1
        print(f"  latest predecessor's phase-1 end after this tile's: mean {lag.mean():.2f} "
              f"p90 {np.percentile(lag, 90):.2f} us")
        gaps = []
        for sm in np.unique(a[:, 7]):
            m = a[:, 7] == sm
            o = np.argsort(st[m])
            gaps.extend((st[m][o][1:] - en[m][o][:-1]).tolist())
        g = np.array(gaps)
        print(f"  same-SM gap, tile end -> next tile start: mean {g.mean():.2f} p50 {np.median(g):.2f} us")
        ts = np.linspace(0, en.max(), 200)
        ph = ([((st <= t) & (p1 > t)).sum() for t in ts], [((p1 <= t) & (lb > t)).sum() for t in ts],
              [((lb <= t) & (en > t)).sum() for t in ts])
        mid = slice(20, 180)
        print("  CTAs in phase 1 / look-back / phase 3 (mid-run mean): "
              + " / ".join(f"{np.mean(x[mid]):.1f}" for x in ph))


if __name__ == "__main__":
    run() if sys.argv[1:] == ["run"] else analyze()
