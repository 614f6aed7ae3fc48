# A/B of an environment switch on pass timings and a full solve: tools/ab_env.sh VAR "v1 v2" config
var=$1; vals=$2; cfg=${3:-medium}
for rep in 1 2; do for v in $vals; do
env $var=$v python - "$cfg" "$var=$v" <<'PY'
import sys, time
sys.path.insert(0, ".")
import torch, synth
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS[sys.argv[1]]
with Pot3d(*c.faces(), c.br0()) as s:
    s.solve(rtol=1e-9, want_phi=False, true_residual=False)
    torch.cuda.synchronize(); t = time.perf_counter()
    r = s.solve(rtol=1e-9, want_phi=False, true_residual=False)
    dt = time.perf_counter() - t
    a, b, p = s.profile(20)
    print(f"{sys.argv[1]} {sys.argv[2]}: iters {r.iters} solve {dt*1e3:.1f} ms ({r.iters/dt:.0f} it/s) | pass A {a*1e3:.1f} us pass B {b*1e3:.1f} us", flush=True)
PY
done; done
