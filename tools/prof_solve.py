"""Short fixed-iteration solve for ncu captures (one GPU):
   python tools/prof_solve.py [config] [iters] [pc]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "medium"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
pc = int(sys.argv[3]) if len(sys.argv) > 3 else 1
blocks = int(sys.argv[4]) if len(sys.argv) > 4 else 1
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), pc=pc, pc2_blocks=blocks) as s:
    r = s.solve(rtol=0.0, maxit=iters, true_residual=False)
    print("iters", r.iters, "rel", r.rel_residual, "info", s.info())
