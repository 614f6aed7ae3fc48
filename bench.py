#!/usr/bin/env python
"""Benchmark of the B200 fp64 PCG potential-field solve (BASELINE.json metric:
"fp64 PCG iters/s & GB/s vs HBM peak at 1/2/4/8 B200; time-to-solve").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config medium] [--impl reference]

One step = the whole hot path on one synthetic magnetogram:
RHS from Br0 (a2) -> PCG to rtol 1e-9 (a3-a10) -> finish + B = grad Phi (a11);
the metric setup (a1) happens once in pot3d_setup, like the paper's start-up
(P:270).  N > 1: one process per GPU under torchrun; the grid is split into
r-slabs with NCCL halo exchange + all-gathered dot products (strong scaling of
the same grid).  Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (oracle/, the plain C fp64 PCG written
from the paper) on this box's host cores on a bounded sample of the same
workload (fixed iteration count per step); under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="medium",
                    choices=["tiny", "small", "medium", "large", "pc2", "weak"])
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--pc2-blocks", type=int, default=1)
    ap.add_argument("--weak-iters", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=20)
    ap.add_argument("--cpu-sample-iters", type=int, default=0,
                    help="oracle iterations per cpu sample (0 = auto, ~10-30 s)")
    return ap.parse_args()


def make_config(args, world):
    if args.config == "weak":
        return synth.weak_config(world)
    return synth.CONFIGS[args.config]


def workload_desc(c, args):
    law = "uniform" if c.uniform else "nonuniform (A13)"
    mp = "dipole" if c.lmax == 0 else f"dipole + l<={c.lmax} multipoles seed {c.seed} (A14)"
    return (f"{c.name} {c.nr}x{c.nt}x{c.np} {law}, {mp}, "
            f"{'source surface' if c.bc == 0 else 'closed wall'}, PC{c.pc}")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


# --------------------------------------------------------------------------- oracle legs
def oracle_sample(c, iters):
    """Oracle PCG loop on the config: returns (iters/s, loop seconds)."""
    import oracle

    rf, tf, pf = c.faces()
    br = c.br0((rf, tf, pf))
    _, _, _, secs = oracle.solve_fixed(rf, tf, pf, br, iters, bc=c.bc, pc=c.pc)
    return iters / secs, secs


def auto_cpu_iters(c):
    # ~ 0.25 s / iteration / 27M cells on 8 cores: aim for ~15 s of loop time
    per_iter = 0.25 * c.n / 27.3e6 * (2.5 if c.pc == 2 else 1.0)
    return int(max(3, min(200, 15.0 / max(per_iter, 1e-4))))


def cpu_baseline(c, args):
    import oracle

    oracle.build()
    iters = args.cpu_sample_iters or auto_cpu_iters(c)
    v, secs = oracle_sample(c, iters)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": v, "unit": "iters/s", "cores": cores, "kind": "oracle",
            "sample": f"{iters} PCG iterations of {c.name} (oracle C fp64, DIA, OpenMP on "
                      f"{cores} threads; assembly excluded), loop {secs:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    c = make_config(args, world)
    import oracle

    oracle.build()
    iters = args.cpu_sample_iters or max(3, auto_cpu_iters(c) // 3)
    for _ in range(args.warmup):
        oracle_sample(c, iters)
    tot_it, tot_s = 0, 0.0
    for _ in range(args.steps):
        v, secs = oracle_sample(c, iters)
        tot_it += iters
        tot_s += secs
    value = tot_it / tot_s
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": "fp64 PCG iters/s", "value": value, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(c, args),
                   "step": f"{iters} oracle PCG iterations (bounded sample)"},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "oracle",
                         "sample": f"{iters} PCG iterations per step of {c.name}"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- own impl
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1709_01126_b200 import Pot3d

    c = make_config(args, world)
    rf, tf, pf = c.faces()
    br_np = c.br0((rf, tf, pf))
    s = Pot3d(rf, tf, pf, br_np, bc=c.bc, pc=c.pc, rank=rank, nranks=world,
              pc2_blocks=args.pc2_blocks, unroll=32)  # fresh NCCL id broadcast inside
    s.trace(True)  # in-situ pass durations of the timed solves (%globaltimer, no extra launches)
    info = s.info()
    fixed_iters = args.weak_iters if args.config == "weak" else 0
    rtol = 0.0 if fixed_iters else c.rtol
    maxit = fixed_iters if fixed_iters else 10**6

    dev = torch.device("cuda", local)
    br_dev = torch.from_numpy(br_np).to(dev)
    phi_dev = torch.empty((c.np, c.nt, s.nr_loc), dtype=torch.float64, device=dev)
    nbr = info["br_shells"]
    B_dev = (torch.empty((c.np, c.nt, nbr), dtype=torch.float64, device=dev),
             torch.empty((c.np, c.nt + 1, s.nr_loc), dtype=torch.float64, device=dev),
             torch.empty((c.np, c.nt, s.nr_loc), dtype=torch.float64, device=dev))
    from paper_1709_01126_b200.pot3d import _ptr

    def step_device():
        s.set_br0(br_dev)
        res = s.solve(rtol=rtol, maxit=maxit, phi=phi_dev, true_residual=False)
        s._check(s._L.pot3d_field(s._ctx, _ptr(B_dev[0])[0], _ptr(B_dev[1])[0], _ptr(B_dev[2])[0]))
        return res

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    for _ in range(args.warmup):
        step_device()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    stream = torch.cuda.current_stream(dev)
    launches0 = s.info()["kernel_launches"]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    iters = []
    for _ in range(args.steps):
        res = step_device()
        iters.append(res.iters)
    ev1.record(stream)
    barrier()
    clocks = clk.stop()
    launches = s.info()["kernel_launches"] - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    tot_iters = int(sum(iters))
    value = tot_iters / (ms / 1e3)
    # live durations of pass A / pass B inside the last timed solve (last <= 64 iterations)
    us_a_live, us_b_live, n_live = s.kernel_times()

    # end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        br_h = torch.from_numpy(br_np).pin_memory()
        phi_h = torch.empty((c.np, c.nt, s.nr_loc), dtype=torch.float64).pin_memory()
        B_h = tuple(torch.empty(b.shape, dtype=torch.float64).pin_memory() for b in B_dev)

        def step_host():
            s.set_br0(br_h)
            r = s.solve(rtol=rtol, maxit=maxit, phi=phi_h, true_residual=False)
            s._check(s._L.pot3d_field(s._ctx, _ptr(B_h[0])[0], _ptr(B_h[1])[0], _ptr(B_h[2])[0]))
            return r

        step_host()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        it_h = 0
        for _ in range(args.steps):
            it_h += step_host().iters
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        t = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        h2d = br_h.numel() * 8
        d2h = (phi_h.numel() + sum(b.numel() for b in B_h)) * 8
        e2e = {"value": it_h / (ems / 1e3), "unit": "iters/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.steps,
               "note": "C-ABI calls with pinned host buffers: Br0 H2D, Phi + Br/Bt/Bp D2H per step"}

    # roofline of the dominant kernel: live durations from the timed solve; the
    # same passes launched separately between CUDA events are reported beside them
    ms_a_iso, ms_b_iso, ms_pc = s.profile(args.profile_iters)
    if n_live > 0:
        ms_a, ms_b, timing = us_a_live / 1e3, us_b_live / 1e3, (
            f"live: mean first-block-start to last-block-end (%globaltimer) of the last {n_live} "
            f"iterations of the last timed solve")
    else:
        ms_a, ms_b, timing = ms_a_iso, ms_b_iso, "isolated launches between CUDA events"
    cells_loc = s.nr_loc * c.nt * c.np
    bytes_a, bytes_b = 24 * cells_loc, 40 * cells_loc
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    gbs_a = bytes_a / (ms_a * 1e-3) / 1e9
    gbs_b = bytes_b / (ms_b * 1e-3) / 1e9
    dom = "k_pass_a_pc1" if ms_a >= ms_b else "k_pass_b_pc1"
    if c.pc == 2:
        dom = dom.replace("pc1", "pc2")
    achieved = gbs_a if ms_a >= ms_b else gbs_b
    dom_bytes, dom_ms = (bytes_a, ms_a) if ms_a >= ms_b else (bytes_b, ms_b)
    if c.pc == 2 and ms_pc > max(ms_a, ms_b):
        # PC2: the forward + backward ILU sweeps dominate (24 + 32 B per cell per apply)
        dom = "k_sweep4 (forward + backward)"
        dom_bytes, dom_ms = 56 * cells_loc, ms_pc
        achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get(c.name, {}).get(dom)
    except Exception:
        pass
    loop_ms = (ms_a + ms_b + ms_pc)
    per_iter_bytes = info["bytes_per_iter"]

    if rank != 0:
        s.close()
        if world > 1:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c, args)
    line = {
        "metric": "fp64 PCG iters/s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.config == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": workload_desc(c, args),
            "cells": c.n, "grid": [c.nr, c.nt, c.np], "rtol": rtol,
            "iters_per_step": iters, "fixed_iters": bool(fixed_iters),
            "step": "rhs(a2) + PCG solve to rtol (a3-a10) + finish + field B (a11)",
            "parallelism": f"r-slabs x{world}" if world > 1 else "1 GPU",
            "l2": f"inputs larger than L2: working set {info['device_bytes'] / 1e9:.2f} GB per rank "
                  f"> 126 MB L2 (no flush)",
        },
        "time_to_solve_s": ms / args.steps / 1e3,
        "cell_updates_per_s": c.n * value,
        "loop_gbs_algorithmic": per_iter_bytes * world * value / 1e9,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "ms_per_launch": dom_ms,
                     "timing": timing,
                     "pass_a": {"ms": ms_a, "gbs": gbs_a, "bytes_per_cell": 24},
                     "pass_b": {"ms": ms_b, "gbs": gbs_b, "bytes_per_cell": 40},
                     "isolated": {"pass_a_ms": ms_a_iso, "pass_b_ms": ms_b_iso,
                                  "pass_b_gbs": bytes_b / (ms_b_iso * 1e-3) / 1e9,
                                  "note": "pot3d_profile: 20 launches between CUDA events after the timed region"},
                     "precond_ms": ms_pc,
                     "loop_gbs": (bytes_a + bytes_b) / (loop_ms * 1e-3) / 1e9 if c.pc == 1 else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
