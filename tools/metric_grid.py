"""BASELINE.json's metric grid ("dot/sum/axpbyz/scan at 1/2/4/8 B200",
SURVEY §8(d): n_global = 2^33 for every op) at G = 1: each op over the whole
2^33-element problem on one GPU (the C4/C5 generators keyed on the global
index; fp32 for dot/sum/axpbyz, int32 exclusive scan), 3 warm-up calls then
10 timed back-to-back calls with CUDA events (working sets 32-96 GiB >> L2).

    python tools/metric_grid.py [--log2n 33] [--out gpurun_out/metric_grid.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402


def timed(fn, reps=10):
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
    return ts[len(ts) // 2], ts[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=33)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "metric_grid.json"))
    a = ap.parse_args()
    n = 1 << a.log2n
    dev = torch.device("cuda:0")
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    rows = []

    def report(op, dtype, nbytes, ms):
        med, best = ms
        gbs = nbytes / (med * 1e-3) / 1e9
        r = {"op": op, "dtype": dtype, "n": n, "G": 1, "ms_median": round(med, 3), "ms_min": round(best, 3),
             "gbs": round(gbs, 1), "frac_of_measured": round(gbs / peak, 4), "frac_of_8tbs": round(gbs / 8000, 4),
             "algorithmic_bytes": nbytes}
        rows.append(r)
        print(json.dumps(r), flush=True)

    x = synth.device_fill(synth.F32_U01, synth.SEED_X, n, device=dev)
    y = synth.device_fill(synth.F32_U01, synth.SEED_Y, n, device=dev)
    r = torch.empty((), dtype=torch.float32, device=dev)
    report("dot", "float32", 8 * n, timed(lambda: G.dot(x, y, out=r)))
    report("sum", "float32", 4 * n, timed(lambda: G.sum(x, out=r)))
    z = torch.empty_like(x)
    report("axpbyz", "float32", 12 * n, timed(lambda: G.axpbyz(5.0, x, 6.0, y, out=z)))
    del x, y, z
    torch.cuda.empty_cache()
    k = synth.device_fill(synth.I32_RANGE, synth.SEED_INT, n, lo=0, hi=9, device=dev)
    o = torch.empty_like(k)
    report("scan", "int32", 8 * n, timed(lambda: G.scan(k, exclusive=True, out=o)))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=0)


if __name__ == "__main__":
    main()
