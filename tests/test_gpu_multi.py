"""NCCL-mode parity at world_size 2 (and 4 when available): runs
tests/multigpu_check.py under torchrun; skipped on single-GPU boxes."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def n_gpus() -> int:
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# "fused": collectives up to 2048 tiles per rank run as the cooperative
# small-collective kernel (every size the check uses); "split": the same
# checks through the separate K1 / finalize / K3 kernels (BL_SMALL_MAX_TILES=0).
@pytest.mark.parametrize("path", ["fused", "split"])
@pytest.mark.parametrize("world", [2, 4])
def test_nccl_mode_matches_sim_mode(world, path):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world + (10 if path == "split" else 0)),
           os.path.join(ROOT, "tests", "multigpu_check.py")]
    env = dict(os.environ)
    if path == "split":
        env["BL_SMALL_MAX_TILES"] = "0"
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0 and "MULTIGPU PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


# The reference's training loop on the B200 backend, deployed two ways: n
# workers simulated in one process, and n processes on n GPUs over the fused
# NVLink exchange (tests/cpp/train_dist_b200.cpp).  The per-step loss and
# per-layer c, r, ||v|| must be byte-identical.
@pytest.mark.parametrize("world", [2, 4])
def test_training_loop_multi_gpu_matches_single_process(world, tmp_path):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    exe = os.path.join(ROOT, "oracle", "_ref", "train_dist_b200")
    if not os.path.exists(exe):
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "accept"], check=True)
        else:
            pytest.fail("oracle/_ref/train_dist_b200 was not built")
    single, multi = tmp_path / "single.csv", tmp_path / "multi.csv"
    r = subprocess.run([exe, str(single), str(world), str(tmp_path / "unused.id")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--no-python", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
           "--master-port", str(29640 + world), exe, str(multi), str(world), str(tmp_path / "nccl.id")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    a, b = single.read_text(), multi.read_text()
    assert a.count("\n") == 601 and a == b
