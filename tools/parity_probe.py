"""Measures the GPU-vs-oracle differences the parity bars are set from
(fixed-iteration iterates k = 1, 2, 7 on the ragged grids, medium 10 and
large 5 iterations).  Prints max|dPhi| / max|Phi| per case."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

GRIDS = [(3, 5, 7), (5, 8, 64), (4, 9, 65), (6, 17, 130), (21, 31, 61), (9, 23, 129), (42, 62, 122)]


def case(rf, tf, pf, br, k, pc=1):
    ref = oracle.solve(rf, tf, pf, br, rtol=0.0, maxit=k, pc=pc)
    with Pot3d(rf, tf, pf, br, pc=pc) as s:
        res = s.solve(rtol=0.0, maxit=k, true_residual=False)
    return np.abs(res.phi - ref["x"]).max() / np.abs(ref["x"]).max()


for dims in GRIDS:
    rf, tf, pf = synth.grid(*dims)
    br = synth.br0_map(tf, pf, lmax=4, seed=2)
    print(dims, " ".join(f"k={k}: pc1 {case(rf, tf, pf, br, k):.2e} pc2 {case(rf, tf, pf, br, k, 2):.2e}"
                         for k in (1, 2, 7, 30)), flush=True)
for name, k in (("medium", 10), ("large", 5)):
    c = synth.CONFIGS[name]
    rf, tf, pf = c.faces()
    print(name, k, f"{case(rf, tf, pf, c.br0(), k):.2e}", flush=True)
