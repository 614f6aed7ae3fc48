"""Per-sub-step timing of one multi-GPU PCG iteration (torchrun): tools/mg_prof.py cfg"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import synth
from paper_1709_01126_b200 import Pot3d
cfg = sys.argv[1]
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0")); torch.cuda.set_device(local)
if world > 1: dist.init_process_group("nccl", device_id=torch.device("cuda", local))
c = synth.CONFIGS[cfg]; rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), rank=rank, nranks=world) as s:
    s.solve(rtol=0.0, maxit=20, true_residual=False, want_phi=False)
    parts = s.profile_iteration(20)
    if rank == 0:
        tot = sum(v for _, v in parts)
        print(f"{cfg} N={world}: total {tot*1e3:.1f} us | " + " | ".join(f"{n} {v*1e3:.1f}" for n, v in parts), flush=True)
if world > 1: dist.destroy_process_group()
