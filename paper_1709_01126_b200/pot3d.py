"""Thin ctypes binding of libpot3d.so (include/pot3d.h) -- argument marshalling only.

Every step of the solve runs in the CUDA kernels of libpot3d.so.  PyTorch is
used only as plumbing: the device allocator (caching allocator callbacks), the
stream all work is ordered on, and torch.distributed to broadcast the NCCL id.
There is no CPU fallback: on a machine without the built library or without a
CUDA device the constructor raises.

Array arguments may be numpy arrays (host) or torch tensors (host or cuda);
layouts are those of include/pot3d.h (phi: shape (np, nt, nr_loc), r fastest;
br0: shape (np, nt), theta fastest).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

SOURCE_SURFACE = 0
CLOSED_WALL = 1
PC1 = 1
PC2 = 2
PC3 = 3  # Chebyshev-accelerated Jacobi

OK = 0
NOT_CONVERGED = 1
PC2_FELL_BACK = 2
STATUS_NAMES = {0: "ok", 1: "not_converged", 2: "pc2_fell_back", -1: "invalid", -2: "cuda",
                -3: "nccl", -4: "indefinite", -5: "oom", -6: "state"}

EXPORTS = ["pot3d_setup", "pot3d_set_br0", "pot3d_solve", "pot3d_solve_from", "pot3d_field", "pot3d_apply", "pot3d_apply_fused", "pot3d_kernel_trace",
           "pot3d_precond", "pot3d_history", "pot3d_info", "pot3d_profile",
           "pot3d_profile_iteration", "pot3d_trace_enable", "pot3d_kernel_times",
           "pot3d_nccl_unique_id",
           "pot3d_destroy", "pot3d_last_error"]

_ALLOC = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Pot3dError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Grid(ctypes.Structure):
    _fields_ = [("nr", ctypes.c_int32), ("nt", ctypes.c_int32), ("np", ctypes.c_int32),
                ("r_faces", ctypes.POINTER(ctypes.c_double)),
                ("t_faces", ctypes.POINTER(ctypes.c_double)),
                ("p_faces", ctypes.POINTER(ctypes.c_double))]


class _Runtime(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p),
                ("alloc", _ALLOC), ("free", _FREE), ("alloc_ctx", ctypes.c_void_p),
                ("pc2_blocks", ctypes.c_int32), ("device", ctypes.c_int32),
                ("unroll", ctypes.c_int32), ("loopback_slabs", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("poly_degree", ctypes.c_int32),
                ("poly_ratio", ctypes.c_double), ("nrhs", ctypes.c_int32)]


class _Info(ctypes.Structure):
    _fields_ = [("i0", ctypes.c_int32), ("i1", ctypes.c_int32), ("nr_loc", ctypes.c_int32),
                ("br_shells", ctypes.c_int32), ("pc", ctypes.c_int32),
                ("pc2_blocks_total", ctypes.c_int32), ("graph_kernels_per_iter", ctypes.c_int64),
                ("bytes_per_iter", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("exchange", ctypes.c_int32),
                ("chunks_a", ctypes.c_int32), ("chunks_b", ctypes.c_int32),
                ("nrhs", ctypes.c_int32)]


_lib = None


def library(build_if_missing: bool = True):
    """Load libpot3d.so (building it with nvcc if it is missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        try:
            _build.build()
        except Exception:
            if not _build.LIB.exists():
                raise
    path = os.environ.get("POT3D_LIB") or str(_build.LIB)  # POT3D_LIB: tuning variants only
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    vp, d, i64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
    L.pot3d_setup.argtypes = [ctypes.POINTER(_Grid), vp, ctypes.c_int32, ctypes.c_int32,
                              ctypes.POINTER(_Runtime), ctypes.POINTER(vp)]
    L.pot3d_set_br0.argtypes = [vp, vp]
    L.pot3d_solve.argtypes = [vp, ctypes.c_double, ctypes.c_int64, vp, i64, d, d]
    L.pot3d_solve_from.argtypes = [vp, vp, ctypes.c_double, ctypes.c_int64, vp, i64, d, d]
    L.pot3d_field.argtypes = [vp, vp, vp, vp]
    L.pot3d_apply.argtypes = [vp, vp, vp]
    L.pot3d_precond.argtypes = [vp, vp, vp]
    L.pot3d_apply_fused.argtypes = [vp, vp, vp, ctypes.c_int32]
    L.pot3d_history.argtypes = [vp, vp, ctypes.c_int64]
    L.pot3d_history.restype = ctypes.c_int64
    L.pot3d_info.argtypes = [vp, ctypes.POINTER(_Info)]
    L.pot3d_profile.argtypes = [vp, ctypes.c_int32, d, d, d]
    L.pot3d_profile_iteration.argtypes = [vp, ctypes.c_int32, d, ctypes.c_char_p, ctypes.c_int32]
    L.pot3d_trace_enable.argtypes = [vp, ctypes.c_int32]
    L.pot3d_kernel_times.argtypes = [vp, d, d, ctypes.POINTER(ctypes.c_int32)]
    L.pot3d_kernel_trace.argtypes = [vp, vp, vp, vp, ctypes.c_int32]
    L.pot3d_nccl_unique_id.argtypes = [vp]
    L.pot3d_destroy.argtypes = [vp]
    L.pot3d_last_error.argtypes = [vp]
    L.pot3d_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def slab_bounds(nr: int, nranks: int, rank: int, pc2_blocks: int = 1, pc: int = PC1):
    """This rank's shells [i0, i1) -- the same leading-remainder partition the
    library uses: PC1 splits nr over ranks; PC2 over nranks*pc2_blocks
    ILU blocks, a rank owning pc2_blocks consecutive blocks (host logic only)."""
    def bounds(n, parts, b):
        base, rem = divmod(n, parts)
        a = b * base + min(b, rem)
        return a, a + base + (1 if b < rem else 0)

    if pc == PC1:
        return bounds(nr, nranks, rank)
    B = nranks * max(1, pc2_blocks)
    return bounds(nr, B, rank * pc2_blocks)[0], bounds(nr, B, (rank + 1) * pc2_blocks - 1)[1]


def gather_slabs(local, nr: int, group=None, dst: int = 0):
    """Assemble the global r-fastest array (np, nt, nr) from every rank's slab
    (np, nt, nr_loc) with torch.distributed (gloo for CPU tensors, NCCL for CUDA
    tensors).  Returns the full array on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist

    t = local if isinstance(local, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(local))
    world = dist.get_world_size(group)
    sizes = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[-1]], dtype=torch.int64, device=t.device), group=group)
    widths = [int(s.item()) for s in sizes]
    if sum(widths) != nr:
        raise ValueError(f"slab widths {widths} do not tile nr={nr}")
    wmax = max(widths)
    pad = torch.zeros(t.shape[:-1] + (wmax,), dtype=t.dtype, device=t.device)
    pad[..., : t.shape[-1]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    if dist.get_rank(group) != dst:
        return None
    return torch.cat([b[..., :w] for b, w in zip(bufs, widths)], dim=-1)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = library().pot3d_nccl_unique_id(buf)
    if rc:
        raise Pot3dError(rc, "ncclGetUniqueId failed")
    return buf.raw


def _ptr(a):
    """(pointer, keepalive) of a numpy array or torch tensor, fp64 contiguous."""
    try:
        import torch

        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("torch tensors must be contiguous float64")
            return ctypes.c_void_p(a.data_ptr()), a
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return ctypes.c_void_p(arr.ctypes.data), arr


@dataclass
class SolveResult:
    phi: object
    iters: int
    rel_residual: float
    true_rel_residual: float
    status: int


class Pot3d:
    """One context of the C ABI (one rank's r-slab on one GPU)."""

    def __init__(self, r_faces, t_faces, p_faces, br0, bc=SOURCE_SURFACE, pc=PC1, *, rank=0,
                 nranks=1, nccl_id: bytes | None = None, stream=None, pc2_blocks=1, device=None,
                 unroll=32, torch_allocator=True, loopback_slabs=0, variant=0, poly=(4, 100.0), nrhs=1):
        """loopback_slabs = k > 1 (single process): the grid is split into k r-slabs on
        this one device, exchanging halos and reductions through the multi-GPU
        peer-memory kernels (include/pot3d.h); arrays are then the whole grid.
        variant: 0 standard PCG, 1 single-reduction CG1.
        pc=3: Chebyshev-accelerated Jacobi with poly = (steps m, interval ratio).
        nrhs = k > 1: a multi-RHS batch -- br0 holds k maps (k, np, nt);
        solve() returns phi (k, np, nt, nr) and per-problem iteration counts and
        residuals; field() arrays gain the leading k."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("pot3d needs a CUDA device (no CPU fallback)")
        L = library()
        self._L = L
        self.rf = np.ascontiguousarray(r_faces, dtype=np.float64)
        self.tf = np.ascontiguousarray(t_faces, dtype=np.float64)
        self.pf = np.ascontiguousarray(p_faces, dtype=np.float64)
        self.nr, self.nt, self.np = len(self.rf) - 1, len(self.tf) - 1, len(self.pf) - 1
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = dev
        torch.cuda.set_device(dev)
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        g = _Grid(self.nr, self.nt, self.np,
                  self.rf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                  self.tf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                  self.pf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        if nranks > 1 and nccl_id is None:
            # a ncclUniqueId is single-use: every context gets a fresh one from rank 0
            import torch.distributed as dist

            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nccl_id = obj[0]
        rt = _Runtime()
        rt.rank, rt.nranks = rank, nranks
        self._nccl_id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        rt.nccl_unique_id = ctypes.cast(self._nccl_id, ctypes.c_void_p) if nccl_id else None
        rt.cuda_stream = self.stream.cuda_stream
        if torch_allocator:
            stream_handle = self.stream

            def _alloc(nbytes, _ctx):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, stream_handle)
                except Exception:
                    return None

            def _free(ptr, _ctx):
                torch.cuda.caching_allocator_delete(ptr)

            self._cb = (_ALLOC(_alloc), _FREE(_free))
            rt.alloc, rt.free = self._cb
        rt.pc2_blocks = pc2_blocks
        rt.loopback_slabs = int(loopback_slabs)
        rt.variant = int(variant)
        rt.poly_degree, rt.poly_ratio = int(poly[0]), float(poly[1])
        rt.nrhs = int(nrhs)
        rt.device = dev
        rt.unroll = unroll
        p_br, keep = _ptr(br0)
        ctx = ctypes.c_void_p()
        rc = L.pot3d_setup(ctypes.byref(g), p_br, bc, pc, ctypes.byref(rt), ctypes.byref(ctx))
        del keep
        if rc < 0:
            raise Pot3dError(rc, L.pot3d_last_error(None).decode())
        self._ctx = ctx
        self.bc, self.pc_requested = bc, pc
        inf = self.info()
        self.i0, self.i1, self.nr_loc = inf["i0"], inf["i1"], inf["nr_loc"]
        self.nrhs = inf["nrhs"]
        self._lead = (self.nrhs,) if self.nrhs > 1 else ()  # batch: the leading axis

    # -- helpers ----------------------------------------------------------
    def _check(self, rc):
        if rc < 0:
            raise Pot3dError(rc, self._L.pot3d_last_error(self._ctx).decode())
        return rc

    def _out(self, shape, out):
        if out == "numpy":
            return np.empty(shape, dtype=np.float64)
        import torch

        return torch.empty(shape, dtype=torch.float64, device=out)

    def info(self):
        inf = _Info()
        self._check(self._L.pot3d_info(self._ctx, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in _Info._fields_}

    # -- API ----------------------------------------------------------------
    def set_br0(self, br0):
        p, keep = _ptr(br0)
        self._check(self._L.pot3d_set_br0(self._ctx, p))

    def solve(self, rtol=1e-9, maxit=100000, want_phi=True, true_residual=True, out="numpy",
              phi=None, x0=None, warm=False):
        """PCG from x0 = 0 (pot3d_solve); x0 (array of phi's shape) or warm=True (the
        context's last solution) start from there instead (pot3d_solve_from)."""
        if want_phi and phi is None:
            phi = self._out(self._lead + (self.np, self.nt, self.nr_loc), out)
        p_phi = _ptr(phi)[0] if phi is not None else None
        k = max(1, self.nrhs)
        it = np.zeros(k, dtype=np.int64)
        rr = np.zeros(k)
        tr = np.full(k, np.nan)
        outs = (p_phi, it.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                rr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if true_residual else None)
        if x0 is not None or warm:
            p0, keep = _ptr(x0) if x0 is not None else (None, None)
            rc = self._L.pot3d_solve_from(self._ctx, p0, float(rtol), int(maxit), *outs)
            del keep
        else:
            rc = self._L.pot3d_solve(self._ctx, float(rtol), int(maxit), *outs)
        self._check(rc)
        if self.nrhs > 1:
            return SolveResult(phi, it, rr, tr, rc)
        return SolveResult(phi, int(it[0]), float(rr[0]), float(tr[0]), rc)

    def field(self, out="numpy"):
        inf = self.info()
        br = self._out(self._lead + (self.np, self.nt, inf["br_shells"]), out)
        bt = self._out(self._lead + (self.np, self.nt + 1, self.nr_loc), out)
        bp = self._out(self._lead + (self.np, self.nt, self.nr_loc), out)
        self._check(self._L.pot3d_field(self._ctx, _ptr(br)[0], _ptr(bt)[0], _ptr(bp)[0]))
        return br, bt, bp

    def apply(self, x, out="numpy", which=0):
        """y = A x through the loop's pass B (which=0), D^-1 A x through PC1's
        pass B (which=1) or A x from pass A's stencil (which=2)."""
        px, keep = _ptr(x)
        y = self._out((self.np, self.nt, self.nr_loc), out)
        self._check(self._L.pot3d_apply_fused(self._ctx, px, _ptr(y)[0], int(which)))
        return y

    def precond(self, r, out="numpy"):
        pr, keep = _ptr(r)
        z = self._out((self.np, self.nt, self.nr_loc), out)
        self._check(self._L.pot3d_precond(self._ctx, pr, _ptr(z)[0]))
        return z

    def trace(self, on=True):
        """Record in-situ pass durations in the solve loop (see kernel_times)."""
        self._check(self._L.pot3d_trace_enable(self._ctx, 1 if on else 0))

    def kernel_times(self):
        """Mean device microseconds of pass A and pass B over the last <= 64 loop
        iterations of the last solve (first block start -> last block end)."""
        a, b, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        self._check(self._L.pot3d_kernel_times(self._ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def kernel_trace(self):
        """(iteration index, pass A us, pass B us) arrays over the last <= 64 loop
        iterations of the last solve (pot3d_kernel_trace)."""
        it = np.zeros(64, dtype=np.int64)
        ua, ub = np.zeros(64), np.zeros(64)
        n = self._check(self._L.pot3d_kernel_trace(self._ctx, it.ctypes.data, ua.ctypes.data, ub.ctypes.data, 64))
        return it[:n], ua[:n], ub[:n]

    def history(self, n):
        h = np.empty(int(n), dtype=np.float64)
        m = self._L.pot3d_history(self._ctx, ctypes.c_void_p(h.ctypes.data), int(n))
        self._check(m)
        return h[:m]

    def profile(self, iters=20):
        """Mean device ms per launch of pass A, pass B and the PC2 sweeps (events on
        the context stream); continues the current recurrences and invalidates the
        last solution."""
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._check(self._L.pot3d_profile(self._ctx, int(iters), ctypes.byref(a), ctypes.byref(b),
                                          ctypes.byref(c)))
        return a.value, b.value, c.value

    def profile_iteration(self, iters=10):
        """[(sub-step name, mean ms)] of one PCG iteration, events between sub-steps."""
        ms = (ctypes.c_double * 32)()
        names = ctypes.create_string_buffer(1024)
        n = self._check(self._L.pot3d_profile_iteration(self._ctx, int(iters), ms, names, 32))
        return list(zip(names.value.decode().split(";")[:n], list(ms)[:n]))

    def close(self):
        if getattr(self, "_ctx", None):
            self._L.pot3d_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
