"""PC2 apply vs oracle on growing grids: python tools/pc2_check.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

for dims in [(21, 31, 61), (20, 40, 100), (40, 80, 200), (76, 151, 301), (151, 301, 601)]:
    for blocks in (1, 4):
        rf, tf, pf = synth.grid(*dims)
        n = int(np.prod(dims))
        r = synth.random_vector(n, 7).reshape(dims[::-1])
        t = time.time()
        z_ref = oracle.precond(rf, tf, pf, r, pc=2, pc2_blocks=blocks)
        t1 = time.time()
        with Pot3d(rf, tf, pf, synth.br0_map(tf, pf, 0), pc=2, pc2_blocks=blocks) as s:
            z = s.precond(r)
            z2 = s.precond(r)
        err = np.abs(z - z_ref).max() / np.abs(z_ref).max()
        bad = np.argwhere(np.abs(z - z_ref) > 1e-10 * np.abs(z_ref).max())
        print(dims, blocks, f"err {err:.2e} rerun-equal {np.array_equal(z, z2)} nbad {len(bad)} first {bad[:3].tolist()} oracle {t1-t:.1f}s", flush=True)
