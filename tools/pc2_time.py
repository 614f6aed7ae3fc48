"""Time the PC2 sweeps: python tools/pc2_time.py cfg blocks"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1709_01126_b200 import Pot3d
cfg, blocks = sys.argv[1], int(sys.argv[2])
c = synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), pc=2, pc2_blocks=blocks) as s:
    s.solve(rtol=0.0, maxit=10, true_residual=False)
    a, b, p = s.profile(10)
    print(f"sweep={os.environ.get("POT3D_PC2_SWEEP", "scan")} {cfg} blocks {blocks}: pass A {a*1e3:.0f} us, pass B {b*1e3:.0f} us, sweeps {p*1e3:.0f} us")
