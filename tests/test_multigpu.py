"""Multi-GPU parity over real NCCL (halo exchange inside qt_sse_sigma_pi, Π reduction to sub-slab owners): runs
tests/mgpu_worker.py under torchrun on 2 (or 4) GPUs, skipped when fewer are visible. The same sharded kernels
are covered on ONE GPU by tests/test_gpu_loopback.py."""
import os
import signal
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


def _run(n, args):
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < n:
        pytest.skip(f"needs {n} GPUs")
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(root / "tests" / "mgpu_worker.py"), *args]
    # own process group: on a timeout torchrun AND its workers are stopped (an orphaned worker spinning on a GPU
    # would slow or break every later case on that GPU)
    pr = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=root,
                          start_new_session=True)
    try:
        out, err = pr.communicate(timeout=420)
    except subprocess.TimeoutExpired:
        os.killpg(pr.pid, signal.SIGTERM)
        try:
            out, err = pr.communicate(timeout=30)
        except subprocess.TimeoutExpired:
            os.killpg(pr.pid, signal.SIGKILL)
            out, err = pr.communicate()
        pytest.fail("multi-GPU worker timed out\n" + out[-3000:] + err[-3000:])
    assert pr.returncode == 0, out[-3000:] + err[-3000:]
    assert "mgpu ok" in out


@pytest.mark.parametrize("cfg,mode,prec,shard,call", [
    ("small", "integer", "fp64", "atom", "fused"), ("small", "random", "fp64", "atom", "separate"),
    ("prof", "integer", "fp64", "atom", "fused"), ("small", "random", "fp32", "atom", "fused"),
    ("prof", "integer", "fp32", "atom", "separate"),
    ("small", "integer", "fp64", "energy", "fused"), ("small", "random", "fp64", "energy", "separate"),
    ("prof", "integer", "fp64", "energy", "fused"), ("small", "integer", "fp32", "energy", "fused"),
    ("prof", "random", "fp32", "energy", "fused")])
def test_sharded_matches_unsharded_2gpu(cfg, mode, prec, shard, call):
    _run(2, [cfg, mode, prec, shard, "0", call])


@pytest.mark.parametrize("cfg,mode,prec", [("small", "integer", "fp64"), ("prof", "random", "fp64"),
                                           ("small", "integer", "fp32")])
def test_2d_grid_matches_unsharded_4gpu(cfg, mode, prec):
    """Ta x TE = 2 x 2: packed atom+energy halo boxes, D halo within the energy row, Π reduced per atom slab."""
    _run(4, [cfg, mode, prec, "2d", "2", "fused"])
