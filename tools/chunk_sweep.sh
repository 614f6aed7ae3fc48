# pass A/B time vs POT3D_CHUNKS: tools/chunk_sweep.sh config "c1 c2 ..."
cfg=$1
for c in $2; do
  POT3D_CHUNKS=$c POT3D_CHUNKS_B=$c python - "$cfg" "$c" <<'PY'
import sys
sys.path.insert(0, ".")
import synth
from paper_1709_01126_b200 import Pot3d
c = synth.weak_config(1) if sys.argv[1] == "weak" else synth.CONFIGS[sys.argv[1]]
with Pot3d(*c.faces(), c.br0()) as s:
    s.solve(rtol=0.0, maxit=20, true_residual=False, want_phi=False)
    a, b, p = s.profile(20)
    n = c.n
    inf = s.info()
    print(f"{sys.argv[1]} chunks {sys.argv[2]} (A {inf['chunks_a']} B {inf['chunks_b']}): pass A {a*1e3:.1f} us {24*n/a/1e6:.0f} GB/s | pass B {b*1e3:.1f} us {40*n/b/1e6:.0f} GB/s", flush=True)
PY
done
