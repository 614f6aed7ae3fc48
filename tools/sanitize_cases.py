"""Small runs of every synchronisation protocol of the library, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
fused passes with TMA + mbarriers (PC1 solve), the PC2 factor and the
sentinel-slot D-ILU sweeps (1 and 2 blocks), the loopback slab exchange
(peer-memory edge stores, halo flags, mailboxes; PC1 and PC2), CG1, and the
fused diagnostic applies.  Exits 0 when every case matches the oracle."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d  # noqa: E402

rf, tf, pf = synth.grid(10, 17, 70)
br = synth.br0_map(tf, pf, lmax=3, seed=1)
cases = [dict(pc=1), dict(pc=2), dict(pc=2, pc2_blocks=2), dict(pc=1, loopback_slabs=2),
         dict(pc=2, loopback_slabs=2), dict(pc=1, variant=1), dict(pc=1, variant=1, loopback_slabs=2),
         dict(pc=3), dict(pc=3, loopback_slabs=2), dict(pc=1, nrhs=2)]
ok = True
for kw in cases:
    blocks = kw.get("pc2_blocks", 1) * max(1, kw.get("loopback_slabs", 1))
    ref = oracle.solve(rf, tf, pf, br, pc=kw["pc"], pc2_blocks=blocks, rtol=1e-9,
                       variant=kw.get("variant", 0))
    nrhs = kw.get("nrhs", 1)
    with Pot3d(rf, tf, pf, np.stack([br] * nrhs) if nrhs > 1 else br, **kw) as s:
        res = s.solve(rtol=1e-9)
        if nrhs > 1:  # a batch of the same map twice: both problems are this solve
            assert np.array_equal(res.phi[0], res.phi[1])
            res.phi, res.iters = res.phi[0], int(res.iters[0])
        if kw == cases[0]:
            s.field()
            x = synth.random_vector(10 * 17 * 70, 1).reshape(70, 17, 10)
            for w in (0, 1, 2):
                s.apply(x, which=w)
    rel = np.linalg.norm(res.phi - ref["x"]) / np.linalg.norm(ref["x"])
    good = abs(res.iters - ref["iters"]) <= 1 and rel <= 1e-9
    ok &= good
    print(kw, "iters", res.iters, "oracle", ref["iters"], f"rel {rel:.2e}", "OK" if good else "MISMATCH", flush=True)
sys.exit(0 if ok else 1)
