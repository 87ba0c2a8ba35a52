"""Is the scan's per-element slowdown from 2^30 to 2^33 a size effect or the
power cap?  Times the int32 exclusive scan (product dispatch: ring at 2^30,
L shape at 2^33) and a copy in short and long back-to-back bursts while a
thread samples SM clock / power / throttle reasons through NVML.
    python tools/lab/power_probe.py"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1304_5553_b200 import gpuarray as G  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.002)


def burst(fn, reps):
    torch.cuda.synchronize()
    samples.clear()
    stop.clear()
    th = threading.Thread(target=sampler)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    clk = sorted(s[0] for s in samples)
    pw = max(s[1] for s in samples) if samples else 0
    capped = sum(1 for s in samples if s[2] & 0x4) if samples else 0  # SW power cap bit
    return ms, clk[len(clk) // 2] if clk else 0, pw, capped, len(samples)


dev = torch.device("cuda:0")
for lg in (30, 33):
    n = 1 << lg
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    for reps in ((3, 30, 150) if lg == 30 else (2, 12)):
        G.scan(k, exclusive=True, out=o)
        time.sleep(3)  # cool down between bursts
        ms, clk, pw, capped, ns = burst(lambda: G.scan(k, exclusive=True, out=o), reps)
        print(f"scan 2^{lg} x{reps}: {ms * 1e3:.1f} us/call = {8 * n / ms / 1e6:.0f} GB/s per-element "
              f"{ms * 1e6 / n * 1e3:.3f} ps | SM clock median {clk} MHz, max power {pw:.0f} W, "
              f"power-capped samples {capped}/{ns}", flush=True)
        time.sleep(3)
        ms, clk, pw, capped, ns = burst(lambda: o.copy_(k), reps)
        print(f"copy 2^{lg} x{reps}: {ms * 1e3:.1f} us/call = {8 * n / ms / 1e6:.0f} GB/s | SM clock median {clk} MHz, "
              f"max power {pw:.0f} W, power-capped samples {capped}/{ns}", flush=True)
    del k, o
    torch.cuda.empty_cache()
