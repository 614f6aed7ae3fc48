import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_1709_01126_b200 import Pot3d
cfg = sys.argv[1]; blocks = int(sys.argv[2]); maxit = int(sys.argv[3])
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), pc=2, pc2_blocks=blocks) as s:
    for rep in range(2):
        try:
            r = s.solve(rtol=1e-9, maxit=maxit)
            print("ok", r.iters, r.rel_residual, r.true_rel_residual)
        except Exception as e:
            h = s.history(maxit + 1)
            n = len(h)
            print("ERR", e, "iters", n - 1, "last hist", h[-6:])
