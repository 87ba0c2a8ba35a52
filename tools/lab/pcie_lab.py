"""Host link ceilings for bench.py's e2e leg (tuning lab, GPU only): pinned
H2D alone, D2H alone, and both at once on two streams, 1 GiB per direction,
CUDA events.    python tools/lab/pcie_lab.py"""
import torch


def main():
    dev = torch.device("cuda:0")
    n = 1 << 28
    h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.float32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    gb = 4 * n / 1e9

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    def h2d():
        d1.copy_(h1, non_blocking=True)

    def d2h():
        h2.copy_(d2, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream(dev)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    t = timed(h2d)
    print(f"H2D alone  {gb / t:6.1f} GB/s")
    t = timed(d2h)
    print(f"D2H alone  {gb / t:6.1f} GB/s")
    t = timed(both)
    print(f"both       {2 * gb / t:6.1f} GB/s total ({gb / t:.1f} per direction)")


if __name__ == "__main__":
    main()
