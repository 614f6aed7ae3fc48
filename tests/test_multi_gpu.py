"""Multi-GPU parity: r-slab decomposition over 2 GPUs, one
process per GPU (torchrun), every case against the CPU oracle on the global grid.

Runs tools/mgpu_check.py: PC1 source surface / closed wall, PC2 with 1 and 2
ILU blocks per rank, CG1; iterations within 1 of the oracle's, rel L2 <= 1e-9, B
within 1e-7, a repeated solve in the same context bitwise identical; warm starts
(x0 = 0 bitwise the cold solve, a perturbed map from the previous Phi against the
oracle's warm start).  With two
or more GPUs the peer-memory exchange (CUDA IPC over NVLink) is in use
(exchange == 2 in pot3d_info); the NCCL fallback is run as well.
Skipped on boxes with fewer than two GPUs.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch

        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tools", "mgpu_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("xfer", ["1", "0"])
def test_two_gpu_parity(xfer):
    rc, out = _run({"POT3D_XFER": xfer})
    lines = [ln for ln in out.splitlines() if ln.startswith("[2 ranks]")]
    assert rc == 0 and lines and all(ln.endswith(")") and " OK " in ln for ln in lines), out[-4000:]
    want = "exchange 2" if xfer == "1" else "exchange 1"
    solves = [ln for ln in lines if " warm " not in ln]
    assert all(want in ln for ln in solves), out[-4000:]
    # warm starts across the ranks (pot3d_solve_from): PCG and CG1, x0 = 0 bitwise the cold solve
    warm = [ln for ln in lines if " warm " in ln]
    assert len(warm) == 3 and all("x0=0 same" in ln for ln in warm), out[-4000:]
