import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import torch, numpy as np, synth, oracle
from paper_1304_5553_b200 import _abi, dist as gdist, gpuarray as G
DEV = "cuda:0"
world = 2
nbytes = _abi.gpuarray_xgpu_buffer_bytes()
bufs = [torch.zeros(nbytes, dtype=torch.uint8, device=DEV) for _ in range(world)]
peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
exchs = [gdist.Exchange(peers, r, world, keepalive=bufs) for r in range(world)]
streams = [torch.cuda.Stream() for _ in range(world)]
n = 3_000_017
kh = synth.host_fill(synth.I32_RANGE, 3, n, lo=-(1 << 20), hi=1 << 20)
spans = [gdist.shard_range(n, world, r) for r in range(world)]
ks = [torch.from_numpy(kh[s:s + c]).to(DEV) for s, c in spans]
for st in streams:
    G.workspace("reduce", torch.device(DEV), st.cuda_stream, _abi.gpuarray_reduce_workspace_bytes(0, 0))
    G.workspace("scan", torch.device(DEV), st.cuda_stream, _abi.gpuarray_scan_workspace_bytes(2, n))
offs = [torch.empty(1, dtype=torch.int32, device=DEV) for _ in ks]
torch.cuda.synchronize()
print("step A: prefix-only reduce", flush=True)
for ex, k, st, off in zip(exchs, ks, streams, offs):
    with torch.cuda.stream(st):
        gdist.reduce_fused(G.SUM, G.ID, k, out_dtype=torch.int32, out=off, exchange=ex, prefix_only=True)
torch.cuda.synchronize()
print("offs", [int(o.item()) for o in offs], "expect", [0, int(np.add.reduce(kh[:spans[1][0]], dtype=np.int64))], flush=True)
print("step B: all-fold reduce", flush=True)
for ex, k, st, off in zip(exchs, ks, streams, offs):
    with torch.cuda.stream(st):
        gdist.reduce_fused(G.SUM, G.ID, k, out_dtype=torch.int32, out=off, exchange=ex)
torch.cuda.synchronize()
print("offs", [int(o.item()) for o in offs], flush=True)
print("step C: scans with carry, sequential", flush=True)
for k, off in zip(ks, offs):
    r = G.scan(k, carry=off)
    torch.cuda.synchronize()
print("ok C", flush=True)
