"""Multi-GPU run of both cross-GPU paths under torchrun (one rank per GPU,
NCCL): skipped unless the box has >= 2 GPUs (gpurun leases one; the first
multi-GPU lease exercises the paths instead of discovering them).  Each rank
checks its shard of every result against the unsharded CPU oracle
(tests/mgpu/check_sharded.py), and the bench's N > 1 step runs with both
collectives."""
import glob
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
needs2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, args, env=None, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    return subprocess.run(cmd, cwd=ROOT, env={**os.environ, **(env or {})}, capture_output=True, text=True,
                          timeout=timeout)


@needs2
@pytest.mark.parametrize("nproc", sorted({2, min(NGPU, 8)}))
def test_sharded_paths_match_unsharded_oracle(tmp_path, nproc):
    r = _torchrun(nproc, [os.path.join(ROOT, "tests", "mgpu", "check_sharded.py")], env={"MGPU_OUT": str(tmp_path)})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    files = sorted(glob.glob(str(tmp_path / "rank*.json")))
    assert len(files) == nproc
    for fn in files:
        v = json.load(open(fn))
        assert v["world"] == nproc
        assert not v["fails"], (v["rank"], v["fails"])


@needs2
@pytest.mark.parametrize("collective", ["nccl", "fused"])
def test_bench_multigpu_step(collective):
    nproc = min(NGPU, 8)
    r = _torchrun(nproc, ["bench.py", "--gpus", str(nproc), "--steps", "3", "--warmup", "3", "--log2n-global", "28",
                          "--collective", collective, "--no-cpu-baseline", "--e2e-steps", "1", "--no-extras"])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == nproc and line["parity"]["ok"], line.get("parity")
