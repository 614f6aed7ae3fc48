# 2-D sweep of pass A / pass B chunk counts: tools/chunk_sweep2.sh config "a1 a2" "b1 b2"
cfg=$1
for ca in $2; do for cb in $3; do
  POT3D_CHUNKS=$ca POT3D_CHUNKS_B=$cb python - "$cfg" <<'PY'
import sys
sys.path.insert(0, ".")
import synth
from paper_1709_01126_b200 import Pot3d
c = synth.weak_config(1) if sys.argv[1] == "weak" else synth.CONFIGS[sys.argv[1]]
with Pot3d(*c.faces(), c.br0()) as s:
    s.solve(rtol=0.0, maxit=20, true_residual=False, want_phi=False)
    a, b, p = s.profile(20)
    inf = s.info()
    print(f"{sys.argv[1]} A {inf['chunks_a']} B {inf['chunks_b']}: A {a*1e3:.1f} B {b*1e3:.1f} sum {(a+b)*1e3:.1f} us", flush=True)
PY
done; done
