"""Repeat PC2 applies / factorizations and check bitwise reproducibility."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_1709_01126_b200 import Pot3d
cfg = sys.argv[1]; blocks = int(sys.argv[2]); nctx = int(sys.argv[3]); napp = int(sys.argv[4])
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
r = synth.random_vector(c.n, 7).reshape(c.np, c.nt, c.nr)
ref = None
for ic in range(nctx):
    with Pot3d(rf, tf, pf, c.br0(), pc=2, pc2_blocks=blocks) as s:
        for ia in range(napp):
            z = s.precond(r)
            if ref is None:
                ref = z.copy()
            d = np.abs(z - ref).max()
            nb = int((z != ref).sum())
            if nb:
                idx = np.argwhere(z != ref)
                print(f"ctx {ic} apply {ia}: {nb} cells differ, max {d:.3e}, first {idx[:3].tolist()}", flush=True)
print("done")
