"""Multi-GPU parity check, run under torchrun (one process per GPU):
   torchrun --nproc-per-node N tools/mgpu_check.py
Solves configs with the r-slab decomposition and compares the gathered Phi with
the CPU oracle (PC1: iterations +-1, rel L2 <= 1e-9; PC2 with N*b blocks)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_1709_01126_b200 import Pot3d, gather_slabs  # noqa: E402

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
fails = 0
cases = [("tiny", 1, 1, synth.SOURCE_SURFACE, 0), ("small", 1, 1, synth.SOURCE_SURFACE, 0),
         ("small", 1, 1, synth.CLOSED_WALL, 0), ("small", 2, 1, synth.SOURCE_SURFACE, 0),
         ("small", 2, 2, synth.SOURCE_SURFACE, 0), ("small", 2, 1, synth.CLOSED_WALL, 0)]
# the thinnest legal slabs: 2 shells per rank
cases.append(("thin", 1, 1, synth.SOURCE_SURFACE, 0))
cases.append(("thin", 2, 1, synth.SOURCE_SURFACE, 0))
# CG1 (single-reduction PCG) across ranks: NCCL halo + one all-gather
cases += [("tiny", 1, 1, synth.SOURCE_SURFACE, 1), ("small", 1, 1, synth.CLOSED_WALL, 1),
          ("thin", 1, 1, synth.SOURCE_SURFACE, 1)]
# PC3 (Chebyshev-accelerated Jacobi) across ranks: a halo of d between the steps
cases += [("small", 3, 1, synth.SOURCE_SURFACE, 0), ("small", 3, 1, synth.CLOSED_WALL, 0),
          ("thin", 3, 1, synth.SOURCE_SURFACE, 0)]
for name, pc, blocks, bc, variant in cases:
    c = synth.Config("thin", 2 * world, 17, 33, lmax=4) if name == "thin" else synth.CONFIGS[name]
    rf, tf, pf = c.faces()
    br = c.br0()
    t0 = time.time()
    with Pot3d(rf, tf, pf, br, bc=bc, pc=pc, rank=rank, nranks=world, pc2_blocks=blocks, variant=variant) as s:
        res = s.solve(rtol=1e-9)
        exch = s.info()["exchange"]
        # a second solve in the same context (new epoch of the peer sequence numbers)
        res2 = s.solve(rtol=1e-9)
        same = res2.iters == res.iters and np.array_equal(res2.phi, res.phi)
        br_f, bt_f, bp_f = s.field()
        phi = gather_slabs(torch.from_numpy(res.phi).cuda(), c.nr)
        brg = gather_slabs(torch.from_numpy(np.ascontiguousarray(br_f)).cuda(), c.nr + 1)
    if rank == 0:
        import oracle

        ref = oracle.solve(rf, tf, pf, br, bc=bc, pc=pc, pc2_blocks=world * blocks, rtol=1e-9, variant=variant)
        phi = phi.cpu().numpy()
        rel = np.linalg.norm(phi - ref["x"]) / np.linalg.norm(ref["x"])
        obr, _, _ = oracle.field(rf, tf, pf, br, ref["x"], bc=bc)
        ferr = np.abs(brg.cpu().numpy() - obr).max() / np.abs(obr).max()
        ok = abs(res.iters - ref["iters"]) <= 1 and rel <= 1e-9 and ferr <= 1e-7 and same
        fails += 0 if ok else 1
        print(f"[{world} ranks] {name} pc{pc}{' cg1' if variant else ''} blocks/rank {blocks} bc {bc}: iters {res.iters} "
              f"(oracle {ref['iters']}) rel {rel:.2e} field {ferr:.2e} true_res "
              f"{res.true_rel_residual:.2e} exchange {exch} repeat {'same' if same else 'DIFF'} "
              f"{'OK' if ok else 'FAIL'} ({time.time() - t0:.1f}s)",
              flush=True)
# warm starts across ranks (pot3d_solve_from): x0 = 0 reproduces the cold
# solve bitwise; a perturbed map from the previous Phi matches the oracle's warm start
for name, variant in (("small", 0), ("small", 1), ("thin", 0)):
    c = synth.Config("thin", 2 * world, 17, 33, lmax=4) if name == "thin" else synth.CONFIGS[name]
    rf, tf, pf = c.faces()
    a = c.br0()
    b = a + 0.02 * synth.br0_map(tf, pf, 4, 9)
    t0 = time.time()
    with Pot3d(rf, tf, pf, a, rank=rank, nranks=world, variant=variant) as s:
        cold = s.solve(rtol=1e-9)
        zero = s.solve(rtol=1e-9, x0=np.zeros_like(cold.phi))
        same = zero.iters == cold.iters and np.array_equal(zero.phi, cold.phi)
        pa = gather_slabs(torch.from_numpy(cold.phi).cuda(), c.nr)
        s.set_br0(b)
        warm = s.solve(rtol=1e-9, warm=True)
        pw = gather_slabs(torch.from_numpy(warm.phi).cuda(), c.nr)
    if rank == 0:
        import oracle

        ow = oracle.solve(rf, tf, pf, b, rtol=1e-9, variant=variant, x0=pa.cpu().numpy())
        oc = oracle.solve(rf, tf, pf, b, rtol=1e-9, variant=variant)
        rel = np.linalg.norm(pw.cpu().numpy() - ow["x"]) / np.linalg.norm(ow["x"])
        ok = same and abs(warm.iters - ow["iters"]) <= 1 and rel <= 1e-9 and warm.iters < oc["iters"]
        fails += 0 if ok else 1
        print(f"[{world} ranks] warm {name}{' cg1' if variant else ''}: x0=0 {'same' if same else 'DIFF'}, "
              f"from the previous Phi {warm.iters} iterations (oracle warm {ow['iters']}, cold {oc['iters']}) "
              f"rel {rel:.2e} {'OK' if ok else 'FAIL'} ({time.time() - t0:.1f}s)", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(1 if fails else 0)
