import sys, time
sys.path.insert(0, ".")
import torch, synth
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "medium"]
for rep in range(2):
    for u in (8, 16, 32):
        with Pot3d(*c.faces(), c.br0(), unroll=u) as s:
            s.solve(rtol=1e-9, want_phi=False, true_residual=False)
            torch.cuda.synchronize(); t = time.perf_counter()
            r = s.solve(rtol=1e-9, want_phi=False, true_residual=False)
            dt = time.perf_counter() - t
            print(f"unroll {u}: iters {r.iters} {dt*1e3:.1f} ms {r.iters/dt:.1f} it/s", flush=True)
