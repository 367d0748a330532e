"""The vocab-sharded path with its NCCL exchanges on >= 2 GPUs (torchrun, one rank
per GPU): tests/dist_gpu_worker.py, every rank against the unsharded oracle.
Skipped when fewer than 2 GPUs are visible (this run's GPU boxes have one; the
one-GPU stacked version of the same chain is tests/test_gpu_sharded.py)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2])
def test_sharded_nccl_path(world):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "tests", "dist_gpu_worker.py")]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    for k in range(world):
        assert f"rank {k} ok" in r.stdout
