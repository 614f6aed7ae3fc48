"""PC2 tiny solve diagnostics: python tools/pc2_diag.py  (env POT3D_PC2_SWEEP=4 selects k_sweep4)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

c = synth.CONFIGS["tiny"]
rf, tf, pf = c.faces()
br = c.br0()
for blocks in (1, 2):
    ref = oracle.solve(rf, tf, pf, br, pc=2, pc2_blocks=blocks, rtol=1e-9)
    with Pot3d(rf, tf, pf, br, pc=2, pc2_blocks=blocks) as s:
        x = synth.random_vector(c.n, 3).reshape(c.np, c.nt, c.nr)
        z = s.precond(x)
        zr = oracle.precond(rf, tf, pf, x, pc=2, pc2_blocks=blocks)
        e1 = np.abs(z - zr).max() / np.abs(zr).max()
        z2 = s.precond(x)
        e2 = np.abs(z2 - zr).max() / np.abs(zr).max()
        try:
            res = s.solve(rtol=1e-9)
            msg = f"iters {res.iters} (oracle {ref['iters']}) rel {np.linalg.norm(res.phi - ref['x']) / np.linalg.norm(ref['x']):.2e}"
        except Exception as ex:
            msg = f"solve failed: {ex}"
        for k in (1, 2, 3):
            try:
                r = s.solve(rtol=0.0, maxit=k)
                o = oracle.solve(rf, tf, pf, br, pc=2, pc2_blocks=blocks, rtol=0.0, maxit=k)
                msg += f" | k={k} err {np.abs(r.phi - o['x']).max() / np.abs(o['x']).max():.2e}"
            except Exception as ex:
                msg += f" | k={k} failed {ex}"
    print(f"sweep={os.environ.get('POT3D_PC2_SWEEP', 'scan')} blocks {blocks}: apply {e1:.2e} / again {e2:.2e}; {msg}", flush=True)
