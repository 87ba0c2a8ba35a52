import sys, time, faulthandler
sys.path.insert(0, '.')
faulthandler.dump_traceback_later(100, exit=True)
import torch, synth, paper_1304_5553_b200 as ga
from paper_1304_5553_b200 import gpuarray as G
dev = torch.device('cuda:0')
for lg in (20, 24, 26, 28):
    n = 1 << lg
    t0 = time.time()
    k = synth.device_fill(synth.I32_RANGE, 3, n, lo=0, hi=9, device=dev)
    torch.cuda.synchronize(); print('fill', lg, time.time()-t0, flush=True)
    s = G.scan(k, exclusive=True); torch.cuda.synchronize(); print('scan', lg, time.time()-t0, flush=True)
    x = synth.device_fill(synth.F32_U01, 1, n, device=dev)
    y = synth.device_fill(synth.F32_U01, 2, n, device=dev)
    z = G.axpbyz(5.0, x, 6.0, y); torch.cuda.synchronize(); print('axpbyz', lg, time.time()-t0, flush=True)
    r = G.dot(x, y); torch.cuda.synchronize(); print('dot', lg, r.item(), time.time()-t0, flush=True)
