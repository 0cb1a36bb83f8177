"""Multi-rank path on real GPU memory: torchrun with 2 and 3 ranks (sharing the
box's GPUs; gloo when there are fewer GPUs than ranks) — sharded compute with
recomputed halos + all-gather must equal the single-process run and the oracle."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3])
def test_torchrun_sharded_equals_single(world):
    # world 1 runs the packed all-gather through a real NCCL communicator (one rank per GPU)
    backend = "nccl" if torch.cuda.device_count() >= world else "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "helpers", "dist_check.py"),
           "--backend", backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout


@pytest.mark.parametrize("world", [2, 3, 8])
def test_torchrun_fused_peer_gather(world):
    # every rank's own columns hold the whole job after the fused (peer-memory) gather
    backend = "nccl" if torch.cuda.device_count() >= world else "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "helpers", "p2p_check.py"),
           "--backend", backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == world
