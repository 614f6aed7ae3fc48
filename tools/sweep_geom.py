"""PC2 sweep time vs tile-grid shape: python tools/sweep_geom.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1709_01126_b200 import Pot3d
GEOMS = [(151, 8, 120), (151, 64, 120), (151, 8, 600), (151, 301, 120), (151, 64, 600), (151, 301, 601)]
if len(sys.argv) > 1:
    GEOMS = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for (nr, nt, np_) in GEOMS:
    rf, tf, pf = synth.grid(nr, nt, np_)
    with Pot3d(rf, tf, pf, synth.br0_map(tf, pf, 0), pc=2) as s:
        s.solve(rtol=0.0, maxit=4, true_residual=False, want_phi=False)
        a, b, p = s.profile(6)
        ntj, ntk = (nt + 7) // 8, (np_ + 3 + 127) // 128
        scan = os.environ.get("POT3D_PC2_SWEEP", "0") != "4"
        steps = nr + 8 - 1 if scan else nr + 8 + 32 - 2
        print(f"{'scan' if scan else 'sweep4'} {nr}x{nt}x{np_}: tiles {ntj}x{ntk} sweeps {p*1e3:.0f} us  "
              f"per sweep-step {p*1e3/2/steps:.2f} us", flush=True)
