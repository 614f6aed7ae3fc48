"""Sensitivity of the oracle's own iteration count to the rounding order (oracle
only; no CUDA path).  Builds oracle/pot3d_oracle.c with -DORC_DOT_REVERSE (every
inner product summed in reverse index order) or -DORC_ILU_DFORM (the same ILU0
applied in D-ILU form) -- equally valid fp64 evaluations -- into /tmp, solves one config to rtol 1e-9 and records the iteration count and
the solution's distance to the committed golden (tests/golden/oracle_<cfg>_pc<pc>_b<b>.json)
in tests/golden/oracle_<cfg>_pc<pc>_b<b>_spread_<variant>.json.  Where the residual
hovers near rtol, a rounding-order change alone moves the stopping iteration by
more than one; the GPU parity bar for that config is this spread (A24).

Usage: python tools/oracle_spread.py medium 2 [blocks] [DOT_REVERSE|ILU_DFORM]
"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

name = sys.argv[1]
pc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 1
variant = sys.argv[4] if len(sys.argv) > 4 else "DOT_REVERSE"   # or ILU_DFORM (PC2)
so = Path(f"/tmp/liboracle_{variant}_{os.getpid()}.so")
subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", f"-DORC_{variant}",
                       "-shared", "-fPIC", "-std=c11", "-o", str(so), str(ROOT / "oracle" / "pot3d_oracle.c"), "-lm"])
os.environ["POT3D_ORACLE_LIB"] = str(so)
import oracle  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[name]
rf, tf, pf = c.faces()
t0 = time.time()
o = oracle.solve(rf, tf, pf, c.br0((rf, tf, pf)), bc=c.bc, pc=pc, pc2_blocks=blocks, rtol=c.rtol, maxit=200000,
                 history=True)
g = json.loads((ROOT / "tests" / "golden" / f"oracle_{name}_pc{pc}_b{blocks}.json").read_text())
x = o["x"].reshape(-1)
samp = x[:: g["stride"]]
ref = np.asarray(g["sample"])
rec = {"written_by": f"tools/oracle_spread.py (oracle/ only, -DORC_{variant})", "variant": variant,
       "config": name, "pc": pc, "pc2_blocks": blocks,
       "iters_variant": o["iters"], "iters_golden": g["iters"],
       "delta_iters": o["iters"] - g["iters"],
       "rel_l2_sample_vs_golden": float(np.linalg.norm(samp - ref) / np.linalg.norm(ref)),
       "rel_res": o["rel_res"], "hist_every": g["hist_every"],
       "hist_rel_diff_max": float(np.max(np.abs(o["hist"][:: g["hist_every"]][: len(g["hist"])] /
                                                np.asarray(g["hist"])[: len(o["hist"][:: g["hist_every"]])] - 1))),
       "seconds": time.time() - t0}
(ROOT / "tests" / "golden" / f"oracle_{name}_pc{pc}_b{blocks}_spread_{variant.lower()}.json").write_text(
    json.dumps(rec, indent=1) + "\n")
print(rec)
