"""Sharded GPUArray operations across GPUs (one process per GPU).

Arrays are sharded contiguously: rank g of G owns global indices
[start_g, start_{g+1}) with start_g = floor(g*n/G) (R16).

  elementwise   shard-local, no communication
  reductions    local single-pass reduce -> ONE scalar NCCL allreduce
                
  scan          local reduce -> NCCL allgather of the G shard totals -> local
                single-pass scan whose carry-in is the fold of the totals of
                ranks < g: 3 element-sizes of HBM
                traffic per element instead of the 4 of scan-then-add.

With an NCCL process group, reduce() and scan() are ONE call each into the C
ABI (gpuarray_reduce_sharded / gpuarray_scan_sharded), which runs the local
kernels and the NCCL collective on the caller's stream with the group's own
communicator (ProcessGroupNCCL._comm_ptr()): torch supplies the process
group, nothing else.  With another backend (gloo: the CPU tests of this host
logic, or ranks sharing one GPU) the same choreography runs with the local
operations from `ops` and the collectives from torch.distributed; `ops`
defaults to the CUDA kernels (tests pass a CPU stand-in).
"""
import torch
import torch.distributed as dist

_COMMS = {}


def nccl_comm(group=None, device=None):
    """The ncclComm_t (as an int) of `group`'s NCCL backend on `device`
    (default: the current CUDA device), or None when the group is not NCCL.
    A lazily created communicator is created by one tiny collective."""
    if not dist.is_initialized():
        return None
    pg = group or dist.group.WORLD
    if dist.get_backend(pg) != "nccl":
        return None
    device = device or torch.device("cuda", torch.cuda.current_device())
    key = (id(pg), device.index)
    ptr = _COMMS.get(key)
    if ptr:
        return ptr
    be = pg._get_backend(device)
    ptr = be._comm_ptr()
    if not ptr:
        dist.all_reduce(torch.zeros(1, device=device), group=pg)
        torch.cuda.synchronize(device)
        ptr = be._comm_ptr()
    if not ptr:
        raise RuntimeError("NCCL process group has no communicator on this device")
    _COMMS[key] = ptr
    return ptr


def shard_range(n, world, rank):
    """(start, count) of rank's contiguous shard of a length-n array."""
    if not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard request")
    start = (rank * n) // world
    stop = ((rank + 1) * n) // world
    return start, stop - start


class CudaOps:
    """The local operations, all through libgpuarray.so."""

    def __init__(self):
        from . import gpuarray as G
        self.G = G

    def reduce(self, op, map_, x, y=None, out_dtype=None, out=None):
        return self.G.reduce(op, map_, x, y, out_dtype=out_dtype, out=out)

    def scan(self, x, exclusive=False, out=None, carry=None):
        return self.G.scan(x, exclusive=exclusive, out=out, carry=carry)


_TORCH_OP = None


def _torch_op(op):
    global _TORCH_OP
    if _TORCH_OP is None:
        _TORCH_OP = {0: dist.ReduceOp.SUM, 1: dist.ReduceOp.MAX, 2: dist.ReduceOp.MIN}
    return _TORCH_OP[op]


def reduce(op, map_, x, y=None, out_dtype=None, out=None, group=None, ops=None):
    """Global map-reduce of a sharded array: local reduce, then one scalar
    allreduce.  Every rank ends with the same bits (NCCL's result is
    identical on all ranks)."""
    comm = nccl_comm(group, x.device) if ops is None and x.is_cuda else None
    if comm is not None:
        from . import gpuarray as G
        return G.reduce(op, map_, x, y, out_dtype=out_dtype, out=out, nccl_comm=comm)
    ops = ops or CudaOps()
    r = ops.reduce(op, map_, x, y, out_dtype=out_dtype, out=out)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(r.view(1), op=_torch_op(op), group=group)
    return r


def reduce_many(specs, out, group=None, ops=None):
    """Several SUM reductions fused into one collective: specs is a list of
    (map, x, y); out is a 1-D tensor of len(specs) (results land in place)."""
    ops = ops or CudaOps()
    for k, (map_, x, y) in enumerate(specs):
        ops.reduce(0, map_, x, y, out_dtype=out.dtype, out=out[k:k + 1])
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def scan(x, exclusive=False, out=None, group=None, ops=None, totals=None, op=0, out_dtype=None):
    """Global scan (SUM / MAX / MIN) of a sharded array (integers wrap)."""
    comm = nccl_comm(group, x.device) if ops is None and x.is_cuda else None
    if comm is not None:
        from . import gpuarray as G
        return G.scan(x, exclusive=exclusive, out=out, op=op, out_dtype=out_dtype, nccl_comm=comm)
    if op != 0 or out_dtype not in (None, x.dtype):
        raise ValueError("the torch.distributed path scans with SUM in the element type only")
    ops = ops or CudaOps()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return ops.scan(x, exclusive=exclusive, out=out)
    rank = dist.get_rank(group)
    if totals is None or totals.numel() != world + 1:
        totals = torch.empty(world + 1, dtype=x.dtype, device=x.device)
    mine, gathered = totals[world:], totals[:world]
    ops.reduce(0, 0, x, None, out_dtype=x.dtype, out=mine)
    dist.all_gather_into_tensor(gathered, mine, group=group)
    carry = gathered[:rank] if rank > 0 else None
    return ops.scan(x, exclusive=exclusive, out=out, carry=carry)


# ---------------------------------------------------------------- fused cross-GPU finish (NEXT-1)
class Exchange:
    """Exchange buffers for gpuarray_reduce_xgpu: `peers` is a device array
    of every rank's buffer address as seen from this rank, `rank`/`world`
    this rank's place, `seq` the per-call sequence number (identical on all
    ranks because every rank makes the same calls in the same order)."""

    def __init__(self, peers, rank, world, keepalive=None):
        self.peers = peers
        self.rank = rank
        self.world = world
        self.seq = 0
        self._keepalive = keepalive

    def next_seq(self):
        self.seq += 1
        return self.seq

    @classmethod
    def symmetric(cls, group=None, device=None):
        """Buffers in torch symmetric memory (NVLink-mapped on every peer)."""
        from torch.distributed import _symmetric_memory as symm_mem

        from . import _abi
        device = device or torch.device("cuda", torch.cuda.current_device())
        nbytes = _abi.gpuarray_xgpu_buffer_bytes()
        buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
        buf.zero_()
        group = group or dist.group.WORLD
        hdl = symm_mem.rendezvous(buf, group)
        peers = torch.tensor([int(p) for p in hdl.buffer_ptrs], dtype=torch.int64, device=device)
        torch.cuda.synchronize(device)
        dist.barrier(group)
        return cls(peers, hdl.rank, hdl.world_size, keepalive=(buf, hdl))


def reduce_fused(op, map_, x, y=None, out_dtype=None, out=None, exchange=None, prefix_only=False):
    """Global map-reduce of a sharded array in ONE kernel per rank: the
    local reduction's last block publishes its result to every rank over
    NVLink and folds all ranks' results in rank order (include/gpuarray.h,
    gpuarray_reduce_xgpu)."""
    from . import _abi
    from . import gpuarray as G
    G._check_array("x", x)
    has_y = map_ in (G.MUL, G.CONJ_MUL)
    if has_y:
        if y is None:
            raise ValueError("maps MUL / CONJ_MUL need y")
        G._same(x, y, "y")
    if out_dtype is None:
        out_dtype = G._REAL_OF.get(x.dtype, x.dtype) if map_ == G.SQUARE else x.dtype
    if out is None:
        out = torch.empty((), dtype=out_dtype, device=x.device)
    in_dt, out_dt = G.ga_dtype(x.dtype), G.ga_dtype(out_dtype)
    s = G._stream(x)
    nb = _abi.gpuarray_reduce_workspace_bytes(out_dt, x.numel())
    w = G.workspace("reduce", x.device, s, nb)
    seq = exchange.next_seq()
    G.check(_abi.gpuarray_reduce_xgpu(op, map_, in_dt, out_dt, x.numel(), G._ptr(x),
                                      G._ptr(y) if has_y else None, out.data_ptr(), w.data_ptr(), w.numel(),
                                      exchange.peers.data_ptr(), exchange.rank, exchange.world, seq,
                                      _abi.GA_XGPU_EXCLUSIVE_PREFIX if prefix_only else _abi.GA_XGPU_ALL, s))
    return out


def scan_fused(x, exclusive=False, out=None, exchange=None, offset=None):
    """Global prefix sum of a sharded integer array with no collective
    launch: the local reduce kernel's fused finish returns the fold of the
    totals of ranks < rank (the shard's offset, on the device), which the
    local scan takes as its carry-in."""
    from . import gpuarray as G
    if offset is None or offset.numel() != 1 or offset.dtype != x.dtype:
        offset = torch.empty(1, dtype=x.dtype, device=x.device)
    reduce_fused(G.SUM, G.ID, x, out_dtype=x.dtype, out=offset, exchange=exchange, prefix_only=True)
    return G.scan(x, exclusive=exclusive, out=out, carry=offset)
