"""Live pass durations (pot3d_kernel_trace over the last <= 64 iterations) of a
fixed-iteration solve: python tools/pass_times.py [config] [iters] [variant]
Prints mean microseconds of pass A, pass B (even / odd iterations) and the
algorithmic GB/s of each (PC1: 24, 24, 40 B/cell)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), variant=variant) as s:
    s.trace(True)
    s.solve(rtol=0.0, maxit=iters, true_residual=False)
    s.solve(rtol=0.0, maxit=iters, true_residual=False)
    it, ua, ub = s.kernel_trace()
    inf = s.info()
n = c.n
ev, od = ub[it % 2 == 0].mean(), ub[it % 2 == 1].mean()
a = ua.mean()
ba, bb = (8 if variant else 24), (48 if variant else 24)
bo = 64 if variant else 40
print(f"{cfg} chunks A {inf['chunks_a']} B {inf['chunks_b']} env A={os.environ.get('POT3D_CHUNKS', '-')} "
      f"B={os.environ.get('POT3D_CHUNKS_B', '-')}: passA {a:.1f} us ({ba * n / a / 1e3:.0f} GB/s)  "
      f"B even {ev:.1f} us ({bb * n / ev / 1e3:.0f})  B odd {od:.1f} us ({bo * n / od / 1e3:.0f})  "
      f"iteration {(a + (ev + od) / 2):.1f} us", flush=True)
