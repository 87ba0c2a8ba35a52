"""Per-super-tile timeline of the two-touch scan (tuning lab)."""
import ctypes, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np, torch, synth
L = ctypes.CDLL(os.path.join(HERE, "libscan_lab.so"))
L.lab_scan.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
L.lab_scan_tile.restype = ctypes.c_int64
n = 1 << 28
dev = torch.device("cuda:0")
k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
out = torch.empty_like(k)
ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream().cuda_stream
for v in [int(a) for a in sys.argv[1:]] or [142]:
    tiles = n // L.lab_scan_tile(v)
    tr = torch.zeros(tiles * 8, dtype=torch.int64, device=dev)
    L.lab_set_trace(None)
    for _ in range(3):
        L.lab_scan(v, n, k.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
    L.lab_set_trace(ctypes.c_void_p(tr.data_ptr()))
    L.lab_scan(v, n, k.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
    torch.cuda.synchronize()
    L.lab_set_trace(None)
    t = tr.view(tiles, 8).cpu().numpy().astype(np.float64)[:, :4]
    t = (t - t[:, 0].min()) / 1000.0
    print(f"variant {v} tiles {tiles} span {t[:, 3].max():.1f} us  tile {L.lab_scan_tile(v)}")
    for a, b, nm in [(0, 1, "phase1"), (1, 2, "lookback"), (2, 3, "phase3"), (0, 3, "total")]:
        d = t[:, b] - t[:, a]
        print(f"  {nm:9s} mean {d.mean():7.2f} p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f} max {d.max():7.2f}")
    st = np.sort(t[:, 0])
    print(f"  start rate (tiles/us, middle half): {tiles / 2 / (st[3 * tiles // 4] - st[tiles // 4]):.2f}")
