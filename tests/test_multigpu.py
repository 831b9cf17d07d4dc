"""Multi-GPU (atom sharding + NCCL halo exchange) parity: runs tests/mgpu_worker.py under torchrun on
2 GPUs (skipped when fewer are visible); the sharded result must equal the unsharded one."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,mode,prec,shard", [("small", "integer", "fp64", "atom"), ("small", "random", "fp64", "atom"),
                                                 ("prof", "integer", "fp64", "atom"), ("small", "random", "fp32", "atom"),
                                                 ("prof", "integer", "fp32", "atom"),
                                                 ("small", "integer", "fp64", "energy"),
                                                 ("small", "random", "fp64", "energy"),
                                                 ("prof", "integer", "fp64", "energy"),
                                                 ("small", "integer", "fp32", "energy"),
                                                 ("prof", "random", "fp32", "energy")])
def test_sharded_matches_unsharded(cfg, mode, prec, shard):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs 2 GPUs")
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(root / "tests" / "mgpu_worker.py"), cfg, mode, prec, shard]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "mgpu ok" in r.stdout
