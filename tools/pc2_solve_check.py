"""PC2 fixed-iteration solves vs oracle: python tools/pc2_solve_check.py cfg blocks k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

cfg, blocks, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
br = c.br0()
ref = oracle.solve(rf, tf, pf, br, pc=2, pc2_blocks=blocks, rtol=0.0, maxit=k, history=True)
with Pot3d(rf, tf, pf, br, pc=2, pc2_blocks=blocks) as s:
    try:
        res = s.solve(rtol=0.0, maxit=k)
        h = s.history(k + 1)
        print("gpu hist", h)
        err = np.abs(res.phi - ref["x"]).max() / np.abs(ref["x"]).max()
        print(cfg, blocks, k, "err", err)
    except Exception as e:
        print("gpu error", e)
        print("gpu hist", s.history(k + 1) if False else None)
print("oracle hist", ref["hist"])
