"""Run the int32 exclusive scan (2^28) from a given libgpuarray build a few
times — a minimal target for ncu (tuning lab, GPU only).
    python tools/lab/scan_one.py LIB [calls]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tools/lab")
from ab_scan import load  # noqa: E402


def main():
    lib = load(sys.argv[1])
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda:0")
    n = 1 << 28
    k = torch.randint(0, 10, (n,), dtype=torch.int32, device=dev)
    o = torch.empty_like(k)
    need = lib.gpuarray_scan_workspace_bytes(2, n)
    ws = torch.zeros(need, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(calls):
        assert lib.gpuarray_scan(0, 1, 2, 2, n, k.data_ptr(), o.data_ptr(), None, 0, ws.data_ptr(), need, s) == 0
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
