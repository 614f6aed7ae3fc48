#!/usr/bin/env python
"""Benchmark of the B200 fp64 PCG potential-field solve (BASELINE.json metric:
"fp64 PCG iters/s & GB/s vs HBM peak at 1/2/4/8 B200; time-to-solve").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config large] [--impl reference]

Default workload: `large` (301x601x1201 = 217 M cells), the >= 200 M-cell
configuration BASELINE.json's metric is quoted on (north star; the paper's
case is 207 M points).  One step = the whole hot path (SURVEY.md
§8(a)) on one synthetic magnetogram: RHS from Br0 (a2) -> PCG to rtol 1e-9
(a3-a10) -> finish + B = grad Phi (a11); the metric setup (a1) happens once in
pot3d_setup, like the paper's start-up.  `value` is device time (CUDA
events around solve + field, inputs resident); `e2e` is the wall clock of the
same steps including the pinned H2D of Br0 and the D2H of Phi and B.  N > 1:
one process per GPU under torchrun; the grid is split into r-slabs (strong
scaling of the same grid).  Rank 0 prints ONE JSON line.

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
    ap.add_argument("--config", default="large",
                    choices=["tiny", "small", "medium", "large", "pc2", "pc3", "pc3large", "batch", "batchsmall", "batchpc2", "large8slab",
                             "batchpc3",
                             "weak"])
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--pc2-blocks", type=int, default=1)
    ap.add_argument("--variant", type=int, default=0, choices=[0, 1],
                    help="0 standard PCG, 1 single-reduction CG1 (PC1; SURVEY 8(f)-1)")
    ap.add_argument("--poly", default="4,100",
                    help="PC3: Chebyshev steps m and the interval ratio (pot3d_runtime.poly_degree, poly_ratio)")
    ap.add_argument("--weak-iters", type=int, default=300)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    k = c.extra.get("nrhs", 1)
    mp = "dipole" if c.lmax == 0 else f"dipole + l<={c.lmax} multipoles seed {c.seed} (A14)"
    if k > 1:
        mp = f"a batch of {k} maps: dipole + l<={c.lmax} multipoles seeds {c.seed}-{c.seed + k - 1} (A14)"
    poly = getattr(args, "poly", "4,100")
    return (f"{c.name} {c.nr}x{c.nt}x{c.np} {law}, {mp}, "
            f"{'source surface' if c.bc == 0 else 'closed wall'}, PC{c.pc}"
            f"{f' (m, ratio = {poly})' if c.pc == 3 else ''}"
            f"{', CG1 single-reduction PCG' if getattr(args, 'variant', 0) else ''}")


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
def host_cpu():
    """CPU model (lscpu) and logical core count of this host."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count()


def auto_cpu_iters(c):
    # ~ 0.12 s / iteration / 27M cells on 16 host threads: aim for ~15 s of loop time
    per_iter = 0.12 * c.n / 27.3e6 * (2.5 if c.pc == 2 else 4.0 if c.pc == 3 else 1.0)
    return int(max(3, min(200, 15.0 / max(per_iter, 1e-4))))


class OracleRun:
    """The CPU oracle (oracle/, the plain C fp64 PCG written from the paper) on
    this box's host cores: the system is assembled once (oracle.Session), each
    sample is the unchanged PCG loop from x0 = 0 for a fixed iteration count."""

    def __init__(self, c):
        import oracle

        oracle.build()
        rf, tf, pf = c.faces()
        t0 = time.perf_counter()
        self.sess = oracle.Session(rf, tf, pf, c.br0((rf, tf, pf)), bc=c.bc, pc=c.pc)
        self.setup_s = time.perf_counter() - t0
        self.cores = oracle.threads()
        self.model, self.ncpu = host_cpu()

    def sample(self, iters):
        _, secs = self.sess.solve_fixed(iters)
        return iters / secs, secs

    def desc(self, c, iters):
        return (f"{iters} PCG iterations of {c.name} from x0 = 0 (oracle C fp64, DIA bands, OpenMP "
                f"element-wise loops on {self.cores} threads, sequential dots; assembly "
                f"{self.setup_s:.1f} s excluded); host: {self.model or 'unknown CPU'}, "
                f"{self.ncpu} logical CPUs")


def cpu_baseline(c, args):
    o = OracleRun(c)
    iters = args.cpu_sample_iters or auto_cpu_iters(c)
    v, secs = o.sample(iters)
    out = {"value": v, "unit": "iters/s", "cores": o.cores, "kind": "oracle",
           "sample": o.desc(c, iters) + f", loop {secs:.1f} s", "cpu_model": o.model}
    o.sess.close()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    c = make_config(args, world)
    o = OracleRun(c)
    iters = args.cpu_sample_iters or max(2, auto_cpu_iters(c) // 4)
    for _ in range(args.warmup):
        o.sample(iters)
    tot_it, tot_s = 0, 0.0
    for _ in range(args.steps):
        _, secs = o.sample(iters)
        tot_it += iters
        tot_s += secs
    value = tot_it / tot_s
    line = {
        "impl": "reference", "metric": "fp64 PCG iters/s", "value": value, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(c, args),
                   "step": f"{iters} oracle PCG iterations (bounded sample of the solve)"},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": o.cores, "kind": "oracle",
                         "sample": o.desc(c, iters), "cpu_model": o.model},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def traffic_of(config, kernel):
    """ncu DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
    `kernel` on `config` from the committed ncu capture summary, or None."""
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return tr.get(config, {}).get(kernel)
    except Exception:
        return None


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
    from paper_1709_01126_b200.pot3d import _ptr

    c = make_config(args, world)
    rf, tf, pf = c.faces()
    kb = c.extra.get("nrhs", 1)  # a multi-RHS batch: k problems per solve
    if kb > 1 and world > 1:
        raise SystemExit(f"--config {args.config}: batches run on one GPU (pot3d_runtime.nrhs, DESIGN.md §7.8)")
    br_np = synth.batch_maps(c, (rf, tf, pf)) if kb > 1 else c.br0((rf, tf, pf))
    s = Pot3d(rf, tf, pf, br_np, bc=c.bc, pc=c.pc, rank=rank, nranks=world,
              pc2_blocks=args.pc2_blocks, unroll=32, variant=args.variant, nrhs=kb,
              poly=(int(args.poly.split(",")[0]), float(args.poly.split(",")[1])))  # fresh NCCL id inside
    lead = (kb,) if kb > 1 else ()
    s.trace(True)  # in-situ pass durations of the timed solves (%globaltimer, no extra launches)
    info = s.info()
    fixed_iters = args.weak_iters if args.config == "weak" else 0
    rtol = 0.0 if fixed_iters else c.rtol
    maxit = fixed_iters if fixed_iters else 10**6

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    nbr = info["br_shells"]
    phi_dev = torch.empty(lead + (c.np, c.nt, s.nr_loc), dtype=torch.float64, device=dev)
    B_dev = (torch.empty(lead + (c.np, c.nt, nbr), dtype=torch.float64, device=dev),
             torch.empty(lead + (c.np, c.nt + 1, s.nr_loc), dtype=torch.float64, device=dev),
             torch.empty(lead + (c.np, c.nt, s.nr_loc), dtype=torch.float64, device=dev))
    # pinned host buffers: the step's input (Br0) and its results (Phi, B)
    br_h = torch.from_numpy(br_np).pin_memory()
    phi_h = torch.empty(phi_dev.shape, dtype=torch.float64).pin_memory()
    B_h = tuple(torch.empty(b.shape, dtype=torch.float64).pin_memory() for b in B_dev)
    h2d = br_h.numel() * 8
    d2h = (phi_h.numel() + sum(b.numel() for b in B_h)) * 8

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(ev):
        """One step of the hot path through the public API: Br0 from pinned host
        memory (pot3d_set_br0: H2D + a2), the solve (a3-a10) and B (a11) into
        device buffers between CUDA events ev[0], ev[1] (the device-resident
        `value`), then Phi and B read back into pinned host memory (e2e)."""
        s.set_br0(br_h)
        ev[0].record(stream)
        res = s.solve(rtol=rtol, maxit=maxit, phi=phi_dev, true_residual=False)
        s._check(s._L.pot3d_field(s._ctx, _ptr(B_dev[0])[0], _ptr(B_dev[1])[0], _ptr(B_dev[2])[0]))
        ev[1].record(stream)
        phi_h.copy_(phi_dev, non_blocking=True)
        for bh, bd in zip(B_h, B_dev):
            bh.copy_(bd, non_blocking=True)
        stream.synchronize()
        return res

    def evpair():
        return (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    for _ in range(args.warmup):
        step(evpair())
    barrier()
    clk = ClockSampler(local)
    clk.start()
    launches0 = s.info()["kernel_launches"]
    evs = [evpair() for _ in range(args.steps)]
    iters = []
    barrier()
    w0 = time.perf_counter()
    for ev in evs:
        iters.append(int(np.sum(step(ev).iters)))  # a batch: the iterations of all its problems
    barrier()
    wall = time.perf_counter() - w0
    clocks = clk.stop()
    launches = s.info()["kernel_launches"] - launches0
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms, wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, wall = float(t[0].item()), float(t[1].item())
    tot_iters = int(sum(iters))
    value = tot_iters / (ms / 1e3)
    e2e = {"value": tot_iters / wall, "unit": "iters/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * wall / args.steps,
           "note": "wall clock (max over ranks) around every timed step: pot3d_set_br0 from pinned "
                   "host memory (H2D), solve + field, Phi and Br/Bt/Bp copied to pinned host memory"}
    # live durations of pass A / pass B inside the last timed solve (last <= 64 iterations);
    # PC1's pass B moves 24 B/cell on even and 40 B/cell on odd iterations (A23)
    k_it, k_ua, k_ub = s.kernel_trace()
    n_live = len(k_it) if kb == 1 else 0  # a batch's last iterations cover fewer problems: isolated

    # roofline of the dominant kernel: live durations from the timed solve; the
    # same passes launched separately between CUDA events are reported beside them
    cg1 = args.variant == 1
    if cg1:  # pot3d_profile runs the standard passes only
        ms_a_iso = ms_b_iso = ms_pc = 0.0
    else:
        ms_a_iso, ms_b_iso, ms_pc = s.profile(args.profile_iters)
    cells_loc = s.nr_loc * c.nt * c.np * kb  # per launch: a batch's passes cover its k problems
    pc1 = info["pc"] == 1
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    # kernels of one iteration: (name, algorithmic bytes per launch, launches per iteration, ms)
    if n_live > 0:
        timing = (f"live: mean first-block-start to last-block-end (%globaltimer) of the last {n_live} "
                  f"iterations of the last timed solve")
        ms_a = float(np.mean(k_ua)) / 1e3
        if pc1:
            ev, od = k_ub[k_it % 2 == 0], k_ub[k_it % 2 == 1]
            ms_be = float(np.mean(ev)) / 1e3 if len(ev) else float(np.mean(k_ub)) / 1e3
            ms_bo = float(np.mean(od)) / 1e3 if len(od) else float(np.mean(k_ub)) / 1e3
        else:
            ms_b = float(np.mean(k_ub)) / 1e3
    else:
        timing = "isolated launches between CUDA events"
        ms_a, ms_be, ms_bo, ms_b = ms_a_iso, ms_b_iso, ms_b_iso, ms_b_iso
    if cg1:  # the trace's "pass A" slot is the dots kernel, "pass B" the update kernel
        kern = [("k_cg1_dots", 8 * cells_loc, 1.0, ms_a), ("k_cg1_update_even", 48 * cells_loc, 0.5, ms_be),
                ("k_cg1_update_odd", 64 * cells_loc, 0.5, ms_bo)]
    else:
        kern = [("k_pass_a", 24 * cells_loc, 1.0, ms_a)]
    if cg1:
        pass
    elif pc1:
        kern += [("k_pass_b_pc1_even", 24 * cells_loc, 0.5, ms_be), ("k_pass_b_pc1_odd", 40 * cells_loc, 0.5, ms_bo)]
    elif info["pc"] == 2:
        kern += [("k_pass_b_pc2", 40 * cells_loc, 1.0, ms_b),
                 ("k_sweepS (forward + backward)", 56 * cells_loc, 1.0, ms_pc)]
    else:  # PC3: the Chebyshev steps (48 m - 24 B/cell per apply)
        pm = int(args.poly.split(",")[0])
        kern += [("k_pass_b_pc2", 40 * cells_loc, 1.0, ms_b),
                 ("k_poly_init + k_poly_step/last", (48 * pm - 24) * cells_loc, 1.0, ms_pc)]
    table = {k: {"bytes_per_launch": by, "launches_per_iter": lp, "ms": t, "gbs": by / (t * 1e-3) / 1e9,
                 "frac": by / (t * 1e-3) / 1e9 / peak} for k, by, lp, t in kern}
    dom, dom_bytes, _, dom_ms = max(kern, key=lambda k: k[2] * k[3])
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    loop_ms = sum(lp * t for _, _, lp, t in kern)
    loop_bytes = sum(lp * by for _, by, lp, _ in kern)
    per_iter_bytes = info["bytes_per_iter"]

    if rank != 0:
        s.close()
        if world > 1:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c, args)
    ws = info["device_bytes"]
    line = {
        "metric": "fp64 PCG iters/s", "value": value, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.config == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": workload_desc(c, args),
            "cells": c.n, "grid": [c.nr, c.nt, c.np], "rtol": rtol,
            "iters_per_step": iters, "fixed_iters": bool(fixed_iters), "nrhs": kb,
            "step": "rhs(a2) + PCG solve to rtol (a3-a10) + finish + field B (a11)" +
                    (f" for each of the batch's {kb} problems in one loop; value counts the iterations "
                     f"of every problem" if kb > 1 else ""),
            "parallelism": f"r-slabs x{world}" if world > 1 else "1 GPU",
            "l2": (f"inputs larger than L2: working set {ws / 1e9:.2f} GB per rank > 126 MB L2 (no flush)"
                   if ws > L2_BYTES else
                   f"working set {ws / 1e6:.1f} MB per rank fits the 126 MB L2 (latency-bound config)"),
        },
        "time_to_solve_s": ms / args.steps / 1e3,
        "cell_updates_per_s": c.n * value,
        "loop_gbs_algorithmic": per_iter_bytes / kb * world * value / 1e9,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic_of(c.name, dom.split(" ")[0]),
                     "traffic_source": "profiles/traffic.json (ncu --set full dram__bytes_read.sum + "
                                       "dram__bytes_write.sum per launch, this config)",
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "ms_per_launch": dom_ms,
                     "timing": timing,
                     "kernels": table,
                     "isolated": {"pass_a_ms": ms_a_iso, "pass_b_ms": ms_b_iso,
                                  "note": f"pot3d_profile: {args.profile_iters} launches between CUDA "
                                          f"events after the timed region (pass B: both parities)"},
                     "loop": {"bytes_per_iter": loop_bytes, "ms_per_iter": loop_ms,
                              "gbs": loop_bytes / (loop_ms * 1e-3) / 1e9,
                              "frac": loop_bytes / (loop_ms * 1e-3) / 1e9 / peak}},
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
