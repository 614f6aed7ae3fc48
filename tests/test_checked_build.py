"""The checked build (-DPOT3D_CHECK=1): device-side bounds checks of every store
of the fused passes, the PC2 sweeps (and their edge slots) and the CG1 passes,
the PC2 slot protocol (a producer must find its slot re-armed by the consumer),
the peer-memory edge stores (inside the neighbour's ghost shell) and the mailbox
order (sequence numbers only grow).  A violated invariant makes pot3d_solve fail.
compute-sanitizer is closed on the GPU pool, so this build is its stand-in
(VERDICT r1 item 7); tools/sanitize_cases.py runs every protocol on a small
grid (fused passes, PC2 with 1 and 2 blocks, loopback slabs with PC1 and PC2,
CG1 alone and on loopback slabs) and compares each with the oracle."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_checked_build_runs_every_protocol_clean():
    from paper_1709_01126_b200 import build

    out = build.PKG / "variants" / "libpot3d_check.so"
    out.parent.mkdir(exist_ok=True)
    build.build(defines=["POT3D_CHECK=1"], out=out)
    env = dict(os.environ, POT3D_LIB=str(out))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" OK") == 10, r.stdout
