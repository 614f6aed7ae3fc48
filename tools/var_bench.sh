#!/bin/bash
# time the fused passes of each variant on one config: tools/var_bench.sh [config]
cfg=${1:-medium}
for v in paper_1709_01126_b200/variants/*.so; do
  echo "== $v"
  POT3D_LIB=$v python - "$cfg" <<'PY'
import sys, time
sys.path.insert(0, ".")
import synth
from paper_1709_01126_b200 import Pot3d
c = synth.CONFIGS[sys.argv[1]]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0()) as s:
    s.solve(rtol=0.0, maxit=40, true_residual=False)
    a, b, p = s.profile(40)
    n = c.n
    cs = synth.CONFIGS["small"]
    with Pot3d(*cs.faces(), cs.br0()) as s2:
        r2 = s2.solve(rtol=1e-9)
    print(f"small: iters {r2.iters} true_res {r2.true_rel_residual:.3e}")
    print(f"pass A {a*1e3:.1f} us {24*n/a/1e6:.0f} GB/s | pass B {b*1e3:.1f} us {40*n/b/1e6:.0f} GB/s | loop {64*n/(a+b)/1e6:.0f} GB/s chunks={s.info()}")
PY
done
