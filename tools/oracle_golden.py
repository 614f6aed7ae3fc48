"""Writes the full-solve oracle goldens under tests/golden/ (oracle-only script).

Calls ONLY `oracle/` (and `synth/` for the seeded inputs); nothing here touches
the CUDA path.  For one configuration it runs the oracle's PCG to rtol 1e-9
(A9) and stores a compact record the GPU parity tests compare with:

  iters, rel_res (recurrence), true_rel_res, ||Phi||_2,
  Phi at a fixed strided subsample of flat r-fastest indices (m = s*stride),
  the recurrence residual history ||r_k||/||b|| every `hist_every` iterations.

Usage:  python tools/oracle_golden.py medium 1 [blocks] [fixed_iters]   (pc 1 or 2)
        fixed_iters > 0: exactly that many iterations (rtol 0) -- the `large` grid,
        whose ~14.5k-iteration oracle solve does not fit a CPU session, gets a
        300-iteration golden (oracle_large_pc1_b1_it300.json).
        OMP_NUM_THREADS sets the oracle's element-wise threads.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
import synth  # noqa: E402

N_SAMPLES = 4096
HIST_EVERY = 64


def golden_path(name: str, pc: int, blocks: int) -> Path:
    return ROOT / "tests" / "golden" / f"oracle_{name}_pc{pc}_b{blocks}.json"


def stride_for(n: int) -> int:
    """An odd stride near n / N_SAMPLES that is coprime with the grid's axes
    in practice, so the samples spread over r, theta and phi."""
    s = max(1, n // N_SAMPLES)
    s |= 1
    while any(s % p == 0 for p in (3, 5, 7)):
        s += 2
    return s


def main() -> None:
    name = sys.argv[1]
    pc = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    fixed = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    c = synth.CONFIGS[name]
    rf, tf, pf = c.faces()
    br = c.br0((rf, tf, pf))
    t0 = time.time()
    o = oracle.solve(rf, tf, pf, br, bc=c.bc, pc=pc, pc2_blocks=blocks, rtol=0.0 if fixed else c.rtol,
                     maxit=fixed if fixed else 200000, history=True)
    secs = time.time() - t0
    x = o["x"].reshape(-1)
    stride = stride_for(x.size)
    idx = np.arange(0, x.size, stride)
    hist = o["hist"]
    rec = {
        "written_by": "tools/oracle_golden.py (oracle/ only; no CUDA path)",
        "cite": "P:270 (rtol 1e-9, fp64, iteration counts); A9 (recurrence residual)",
        "config": name, "grid": [c.nr, c.nt, c.np], "uniform": c.uniform, "lmax": c.lmax,
        "seed": c.seed, "bc": c.bc, "pc": pc, "pc2_blocks": blocks, "rtol": 0.0 if fixed else c.rtol,
        "fixed_iters": fixed,
        "status": o["status"], "iters": o["iters"], "rel_res": o["rel_res"],
        "true_rel_res": o["true_rel_res"], "phi_norm2": float(np.linalg.norm(x)),
        "phi_max_abs": float(np.abs(x).max()),
        "stride": stride, "sample": [float(v) for v in x[idx]],
        "hist_every": HIST_EVERY,
        "hist": [float(v) for v in hist[::HIST_EVERY]],
        "oracle_seconds": secs, "omp_threads": os.environ.get("OMP_NUM_THREADS", "default"),
    }
    p = golden_path(name, pc, blocks)
    if fixed:
        p = p.with_name(p.stem + f"_it{fixed}.json")
    p.write_text(json.dumps(rec, indent=0) + "\n")
    print(f"{p.name}: iters {o['iters']} status {o['status']} rel {o['rel_res']:.3e} "
          f"true {o['true_rel_res']:.3e} in {secs:.0f} s")


if __name__ == "__main__":
    main()
