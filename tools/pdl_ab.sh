# A/B of programmatic dependent launch on the full solve: tools/pdl_ab.sh config
cfg=${1:-medium}
for pdl in 0 1 0 1; do
POT3D_PDL=$pdl python - "$cfg" "$pdl" <<'PY'
import sys, time
sys.path.insert(0, ".")
import torch
import synth
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS[sys.argv[1]]
with Pot3d(*c.faces(), c.br0()) as s:
    s.solve(rtol=1e-9, want_phi=False, true_residual=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = s.solve(rtol=1e-9, want_phi=False, true_residual=False)
    dt = time.perf_counter() - t
    print(f"{sys.argv[1]} PDL={sys.argv[2]}: iters {r.iters} {dt*1e3:.1f} ms {r.iters/dt:.1f} iters/s", flush=True)
PY
done
