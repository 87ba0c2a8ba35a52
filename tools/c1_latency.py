"""configs[0] (C1: fp32 n = 2^20, 4 MiB per array, L2-resident; SURVEY §8(d):
"launch-latency-bound, report us/call"): per-op time three ways
  cold   one call after an L2 flush (tools/sweep.py protocol), CUDA events;
  warm   back-to-back eager calls, L2-warm (events around 200 calls);
  graph  the same 200 calls captured once in a CUDA graph and replayed
         (no per-call launch overhead: the kernels' own duration + gaps).
    python tools/c1_latency.py [--log2n 20] [--out gpurun_out/c1.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c1.json"))
    a = ap.parse_args()
    n = 1 << a.log2n
    dev = torch.device("cuda:0")
    x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
    y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
    z, s = torch.empty_like(x), torch.empty_like(k)
    r = torch.empty(3, device=dev)
    flush = torch.empty(512 * 2 ** 20 // 4, device=dev)
    clean = torch.ones(512 * 2 ** 20 // 4, device=dev)
    sink = torch.empty((), device=dev)
    ops = {
        "axpbyz": (12, lambda: G.axpbyz(5.0, x, 6.0, y, out=z)),
        "dot": (8, lambda: G.dot(x, y, out=r[0])),
        "sum": (4, lambda: G.sum(x, out=r[1])),
        "norm2": (4, lambda: G.norm2sq(x, out=r[2])),
        "scan": (8, lambda: G.scan(k, exclusive=True, out=s)),
    }
    stream = torch.cuda.Stream(dev)
    rows = []
    reps = 200
    for name, (bpe, fn) in ops.items():
        with torch.cuda.stream(stream):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            cold = []
            for _ in range(20):
                flush.fill_(1.0)
                G.sum(clean, out=sink)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                cold.append(e0.elapsed_time(e1) * 1e3)
            cold.sort()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            warm = e0.elapsed_time(e1) * 1e3 / reps
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(reps):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            graph = e0.elapsed_time(e1) * 1e3 / reps
        row = {"op": name, "n": n, "cold_us": round(cold[len(cold) // 2], 2), "warm_us": round(warm, 2),
               "graph_us": round(graph, 2), "graph_gbs": round(bpe * n / (graph * 1e-6) / 1e9, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=0)


if __name__ == "__main__":
    main()
