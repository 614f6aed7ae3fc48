import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, oracle
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS["tiny"]
rf, tf, pf = c.faces()
br = c.br0()
n = c.nr * c.nt * c.np
r = synth.random_vector(n, 7).reshape(c.np, c.nt, c.nr)
zref = oracle.precond(rf, tf, pf, r, pc=2, pc2_blocks=1)
with Pot3d(rf, tf, pf, br, pc=2) as s:
    for rep in range(3):
        z = s.precond(r)
        print("precond rep", rep, "err", np.abs(z - zref).max() / np.abs(zref).max(), flush=True)
    for k in (1, 2, 3, 5, 10):
        res = s.solve(rtol=0.0, maxit=k, true_residual=False)
        ref = oracle.solve(rf, tf, pf, br, pc=2, pc2_blocks=1, rtol=0.0, maxit=k)
        print("maxit", k, "x err", np.abs(res.phi - ref["x"]).max() / np.abs(ref["x"]).max(), flush=True)
