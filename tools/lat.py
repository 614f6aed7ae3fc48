"""Per-iteration time of fixed-iteration solves (latency study), torchrun or single.
   tools/lat.py cfg iters"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import synth
from paper_1709_01126_b200 import Pot3d
cfg, iters = sys.argv[1], int(sys.argv[2])
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0")); torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
if "x" in cfg:  # nr x nt x np, nonuniform like the BASELINE configs
    nr, nt, np_ = (int(v) for v in cfg.split("x"))
    c = synth.Config(cfg, nr, nt, np_)
else:
    c = synth.weak_config(world) if cfg == "weak" else synth.CONFIGS[cfg]
rf, tf, pf = c.faces()
with Pot3d(rf, tf, pf, c.br0(), rank=rank, nranks=world) as s:
    s.solve(rtol=0.0, maxit=50, true_residual=False, want_phi=False)
    ts = []
    for _ in range(3):
        if world > 1: dist.barrier()
        torch.cuda.synchronize(); t = time.perf_counter()
        s.solve(rtol=0.0, maxit=iters, true_residual=False, want_phi=False)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    a, b, p = s.profile(20)
    if rank == 0:
        print(f"{cfg} N={world}: {min(ts)/iters*1e6:.1f} us/iter (passA {a*1e3:.0f} us, passB {b*1e3:.0f} us isolated)", flush=True)
if world > 1:
    dist.destroy_process_group()
