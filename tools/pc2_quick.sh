# PC2 parity tests + sweep timing + full PC2 solve time (medium)
timeout 600 python -m pytest tests -q -m gpu -x -k "pc2 or PC2" 2>&1 | tail -3
timeout 300 python tools/pc2_time.py medium 1
timeout 300 python tools/pc2_time.py medium 4
timeout 300 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import torch, synth
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS["medium"]
for pc in (1, 2):
    with Pot3d(*c.faces(), c.br0(), pc=pc) as s:
        s.solve(rtol=1e-9, want_phi=False, true_residual=False)
        torch.cuda.synchronize(); t = time.perf_counter()
        r = s.solve(rtol=1e-9, want_phi=False, true_residual=True)
        dt = time.perf_counter() - t
        print(f"medium PC{pc}: iters {r.iters} {dt:.3f} s true_res {r.true_rel_residual:.2e}", flush=True)
PY
