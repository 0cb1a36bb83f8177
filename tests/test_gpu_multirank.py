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


def _torchrun(world, script, *args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, *script), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env={**os.environ, **(env or {})})


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one rank per GPU over NCCL)")
def test_nccl_one_rank_per_gpu():
    # world = every GPU of the box, real NCCL communicators: the packed all-gather and the
    # fused peer-memory gather both equal the single-process run; NCCL's INIT log names the size
    world = torch.cuda.device_count()
    env = {"NCCL_DEBUG": "INFO", "NCCL_DEBUG_SUBSYS": "INIT"}
    r = _torchrun(world, ("tests", "helpers", "dist_check.py"), "--backend", "nccl", env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout
    assert f"nranks {world}" in r.stdout + r.stderr
    r = _torchrun(world, ("tests", "helpers", "p2p_check.py"), "--backend", "nccl")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("PASS") == world


@pytest.mark.parametrize("gather", ["nccl", "p2p", "auto"])
def test_bench_two_ranks_strong_scaling(gather):
    # bench.py at N = 2 (strong scaling of a C2 prefix; NCCL + CUDA graphs on a >= 2-GPU box,
    # two ranks sharing the GPU over gloo otherwise) prints one line covering all frames
    import json
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    r = _torchrun(2, ("bench.py",), "--gpus", "2", "--steps", "3", "--warmup", "3", "--frames", "256",
                  "--no-e2e", "--no-cpu-baseline", "--dist-backend", backend, "--gather", gather)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["frames"] == 256 and line["config"]["frames_per_gpu"] == 128
    assert len(line["breakdown"]["compute_ms"]) == 2 and line["gpu_launches"] > 0
    # auto = the fused peer-memory gather for the hist + shot-diff step
    assert line["config"]["ops"].endswith("+nccl_allgather" if gather == "nccl" else "+fused_peer_gather")


def test_bench_p2p_fallback_to_allgather():
    # one rank cannot export its columns: every rank falls back to the all-gather, no hang
    import json
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    r = _torchrun(2, ("bench.py",), "--gpus", "2", "--steps", "3", "--warmup", "3", "--frames", "256",
                  "--no-e2e", "--no-cpu-baseline", "--dist-backend", backend, env={"SCN_TEST_P2P_FAIL_RANK": "1"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["config"]["ops"].endswith("+nccl_allgather")
    assert "fell back" in line["config"]["gather_note"]
