"""Per-tile timeline of the warp-specialized scan (tuning lab)."""
import ctypes, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np, torch, synth
L = ctypes.CDLL(os.path.join(HERE, "libscan_lab.so"))
L.lab_scan.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
L.lab_scan_tile.restype = ctypes.c_int64
v = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = 1 << 28
dev = torch.device("cuda:0")
k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
out = torch.empty_like(k)
ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
tiles = n // L.lab_scan_tile(v)
tr = torch.zeros(tiles * 8, dtype=torch.int64, device=dev)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    L.lab_scan(v, n, k.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
L.lab_set_trace(ctypes.c_void_p(tr.data_ptr()))
L.lab_scan(v, n, k.data_ptr(), out.data_ptr(), ws.data_ptr(), s)
torch.cuda.synchronize()
t = tr.view(tiles, 8).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
t = (t - t0) / 1000.0  # us
names = ["claim", "land", "agg", "lb_start", "lb_end", "cons_ready", "stored"]
print("variant", v, "tiles", tiles, "span us", t[:, 6].max())
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 6), (5, 4), (0, 6)]:
    d = t[:, b] - t[:, a]
    print(f"{names[a]:>10} -> {names[b]:<10} mean {d.mean():7.2f} p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f} max {d.max():7.2f}")
# claim rate over time
order = np.argsort(t[:, 0])
print("claims per us (middle half):", tiles / 2 / (t[order[3 * tiles // 4], 0] - t[order[tiles // 4], 0]))
print("sample tiles:", [list(np.round(t[i, :7], 1)) for i in (1000, 1001, 1002, 20000)])
