"""bench.py's step with a configurable op order (tuning lab, GPU only): which
neighbour makes a kernel slower inside the step?  Same data, binding and
workspaces as bench.py; per-op CUDA events, 200 timed steps.
    STEP_ORDER=axpbyz,dot,sum,norm2,scan python tools/lab/step_lab.py"""
import os
import statistics
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1304_5553_b200 import gpuarray as G  # noqa: E402


def main():
    order = os.environ.get("STEP_ORDER", "axpbyz,dot,sum,norm2,scan").split(",")
    dev = torch.device("cuda:0")
    n = 1 << 28
    x = synth.device_fill(synth.F32_U01, synth.SEED_X, n, device=dev)
    y = synth.device_fill(synth.F32_U01, synth.SEED_Y, n, device=dev)
    k = synth.device_fill(synth.I32_RANGE, synth.SEED_INT, n, lo=0, hi=9, device=dev)
    z = torch.empty_like(x)
    s = torch.empty_like(k)
    red = torch.empty(3, dtype=torch.float32, device=dev)
    # STEP_PAD_BYTES: a small-pool allocation made before the workspaces, to
    # move where the lazily allocated scan workspace lands
    pad = torch.empty(int(os.environ.get("STEP_PAD_BYTES", "0")), dtype=torch.uint8, device=dev)  # noqa: F841
    # STEP_SCAN_WS_OFFSET: place the scan workspace at this byte offset from
    # a 2 MiB boundary (a pre-seeded binding workspace)
    if "STEP_SCAN_WS_OFFSET" in os.environ:
        off = int(os.environ["STEP_SCAN_WS_OFFSET"], 0)
        arena = torch.zeros(8 << 20, dtype=torch.uint8, device=dev)
        base = (-arena.data_ptr()) % (2 << 20)
        G._ws[("scan4", dev.index, torch.cuda.current_stream(dev).cuda_stream)] = [arena[base + off:base + off + (1 << 20)], 0]
    # STEP_WS_LAYOUT=same|apart: the reduce and scan workspaces in one 2 MiB
    # page (reduce at +0x200, scan at +0x100200) or in two different pages
    lay = os.environ.get("STEP_WS_LAYOUT")
    if lay:
        arena = torch.zeros(16 << 20, dtype=torch.uint8, device=dev)
        base = (-arena.data_ptr()) % (2 << 20)
        st = torch.cuda.current_stream(dev).cuda_stream
        r_off = base + 0x200
        s_off = base + (0x100200 if lay == "same" else (6 << 20) + 0x200)
        G._ws[("reduce", dev.index, st)] = [arena[r_off:r_off + (1 << 20) + 65536], 0]
        G._ws[("scan4", dev.index, st)] = [arena[s_off:s_off + (1 << 20) - 0x400], 0]
    ops = {
        "axpbyz": lambda: G.axpbyz(5.0, x, 6.0, y, out=z),
        "dot": lambda: G.reduce(G.SUM, G.MUL, x, y, out=red[0:1]),
        "sum": lambda: G.reduce(G.SUM, G.ID, x, out=red[1:2]),
        "norm2": lambda: G.reduce(G.SUM, G.SQUARE, x, out=red[2:3]),
        "scan": lambda: G.scan(k, exclusive=True, out=s),
        "sleep": lambda: torch.cuda._sleep(100000),
    }
    ev = {o: [] for o in order}
    for it in range(210):
        for o in order:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops[o]()
            e1.record()
            if it >= 10:
                ev[o].append((e0, e1))
    torch.cuda.synchronize()
    wsp = {kk[0]: "%#x" % w[0].data_ptr() for kk, w in G._ws.items()}
    print(wsp, " ".join(f"{o}:{statistics.mean(a.elapsed_time(b) for a, b in ev[o]) * 1e3:.1f}" for o in order),
          flush=True)


if __name__ == "__main__":
    main()
