"""ctypes front-end of the CPU fp64 oracle (oracle/pot3d_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product path
(paper_1709_01126_b200/) never imports it and shares no code with it.

Array conventions follow synth/: faces 1-D; br0 shape (np, nt); Phi and every
cell array shape (np, nt, nr) in C order (r fastest, m = i + nr*(j + nt*k),
the Fortran x(i,j,k) of PAPER.md P:222-224).

Parity status of each function:
  assemble/apply   pinned: symmetry, null space, closed-form dipole/multipole,
                   hand-evaluated coefficients, dense brute force.
  rhs              pinned: closed form, S:234 hand evaluation, Σb = 0 (CW).
  pcg (standard)   pinned: SPEC 2x2 worked example through orc_pcg,
                   exact termination of random SPD n <= 30, dense
                   brute force.
  pcg (CG1)        pinned: the same SPEC 2x2 / random SPD / brute-force pins,
                   and exact-arithmetic equivalence with the standard
                   variant (iterates agree to rounding, iterations +-1).
  pcg (warm, X0)   pinned: x0 = 0 reproduces the cold loop bitwise; the SPEC 2x2
                   from its exact solution stops at 0 iterations and from
                   another x0 terminates in <= 2; on random SPD
                   systems warm(x0) equals x0 + cold(b - A x0) with the
                   tolerance rescaled (the same Krylov sequence, to rounding);
                   a POT3D map solved from its own converged Phi stops at 0.
  cheb_apply (PC3) pinned: the closed form (I - R_m(D^-1 A)) A^-1 with the
                   Chebyshev residual polynomial on random SPD matrices.
  solve (PC1/PC2)  pinned: dense brute force, closed form, the survey's
                   independent iteration counts (tiny PC1 229, PC2 91/96/104/
                   114 for 1/2/4/8 blocks, closed wall 428, small 913),
                   monotone PC2 degradation.
  slab_bounds      pinned: explicit sizes (21 shells / 8 -> 3,3,3,3,3,2,2,2,
                   S:392) and PC2 with 8 blocks = block-diagonal ILU0 of the
                   explicitly listed slabs.
  ilu0             pinned: defining property (LU)_ij = a_ij on the pattern,
                   tridiagonal exact LU.
  field            pinned: Br(r0) = Br0, Phi=r -> Br=1, V div B = b - A Phi,
                   closed-form dipole field, polar-face Btheta of an m=1 field
                   against its closed-form derivative (second order, A19).
  polar_average    pinned: constant ring, cos(phi) ring.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "pot3d_oracle.c"
_LIB = _HERE / "liboracle.so"

SOURCE_SURFACE = 0
CLOSED_WALL = 1

STATUS = {0: "converged", 1: "not_converged", 2: "pc2_fell_back_to_pc1",
          -1: "invalid_argument", -4: "indefinite"}


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (plain IEEE fp64: no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared",
               "-fPIC", "-std=c11", "-o", str(tmp), str(_SRC), "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
LINOP = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                         ctypes.POINTER(ctypes.c_double))
STANDARD = 0   # orc_pcg variants: standard two-reduction PCG
X0 = 16        # orc_pcg flag: x holds x0 on entry (warm start, A28)
CG1 = 1        # Chronopoulos-Gear single-reduction PCG


def lib():
    global _lib
    if _lib is None:
        # POT3D_ORACLE_LIB: a deliberately broken build (tools/oracle_mutants.py
        # checks that the pins catch it); never set outside that script
        alt = os.environ.get("POT3D_ORACLE_LIB")
        if not alt:
            build()
        L = ctypes.CDLL(alt or str(_LIB))
        P = ctypes.POINTER
        d = P(ctypes.c_double)
        i64 = P(ctypes.c_int64)
        ci = ctypes.c_int
        L.orc_assemble.argtypes = [ci, ci, ci, d, d, d, ci, d, d]
        L.orc_apply.argtypes = [ci, ci, ci, d, d, d, d]
        L.orc_apply.restype = None
        L.orc_rhs.argtypes = [ci, ci, ci, d, d, d, ci, d, d, d]
        L.orc_solve.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, d, ctypes.c_double,
                                ctypes.c_int64, d, i64, d, d, d]
        L.orc_precond.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, d, d]
        L.orc_block_ilu0.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, i64, i64, d, d]
        L.orc_ilu0_csr.argtypes = [ctypes.c_int64, i64, i64, d]
        L.orc_polar_average.argtypes = [ci, ci, ci, d, d, ci, d]
        L.orc_polar_average.restype = None
        L.orc_field.argtypes = [ci, ci, ci, d, d, d, ci, d, d, d, d, d]
        L.orc_volumes.argtypes = [ci, ci, ci, d, d, d, d]
        L.orc_solve_v.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, d, ctypes.c_double,
                                  ctypes.c_int64, ci, d, i64, d, d, d]
        L.orc_pcg.argtypes = [ctypes.c_int64, LINOP, ctypes.c_void_p, LINOP, ctypes.c_void_p, d,
                              ctypes.c_double, ctypes.c_int64, ci, d, i64, d, d]
        L.orc_slab_bounds.argtypes = [ci, ci, ci, P(ci), P(ci)]
        L.orc_set_poly.argtypes = [ci, ctypes.c_double]
        L.orc_set_poly.restype = None
        L.orc_cheb_apply.argtypes = [ctypes.c_int64, LINOP, ctypes.c_void_p, d, ci, ctypes.c_double,
                                     ctypes.c_double, d, d]
        L.orc_cheb_apply.restype = None
        L.orc_slab_bounds.restype = None
        L.orc_session_create.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, d]
        L.orc_session_create.restype = ctypes.c_void_p
        L.orc_session_solve.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ci, d, i64,
                                        d, d]
        L.orc_session_free.argtypes = [ctypes.c_void_p]
        L.orc_session_free.restype = None
        L.orc_threads.restype = ci
        L.orc_solve_fixed.argtypes = [ci, ci, ci, d, d, d, ci, ci, ci, d, ctypes.c_int64, d, d, d]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class System:
    """The discrete problem on one grid: DIA bands + wrap couplings."""

    def __init__(self, rf, tf, pf, bc=SOURCE_SURFACE):
        self.rf, self.tf, self.pf = _f(rf), _f(tf), _f(pf)
        self.nr, self.nt, self.np = len(rf) - 1, len(tf) - 1, len(pf) - 1
        self.bc = bc
        self.N = self.nr * self.nt * self.np
        self.bands = np.zeros((7, self.N))
        self.wrap = np.zeros((2, self.nr * self.nt))
        rc = lib().orc_assemble(self.nr, self.nt, self.np, _d(self.rf), _d(self.tf), _d(self.pf),
                                bc, _d(self.bands), _d(self.wrap))
        if rc:
            raise ValueError("invalid grid")

    @property
    def shape(self):
        return (self.np, self.nt, self.nr)

    def apply(self, x):
        x = _f(x).reshape(-1)
        y = np.empty_like(x)
        lib().orc_apply(self.nr, self.nt, self.np, _d(self.bands), _d(self.wrap), _d(x), _d(y))
        return y.reshape(self.shape)

    def diag(self):
        return self.bands[3].reshape(self.shape).copy()

    def rhs(self, br0, return_adjusted=False):
        br0 = _f(br0)
        b = np.empty(self.N)
        adj = np.empty(self.nt * self.np)
        lib().orc_rhs(self.nr, self.nt, self.np, _d(self.rf), _d(self.tf), _d(self.pf), self.bc,
                      _d(br0), _d(b), _d(adj))
        if return_adjusted:
            return b.reshape(self.shape), adj.reshape(self.np, self.nt)
        return b.reshape(self.shape)

    def volumes(self):
        v = np.empty(self.N)
        lib().orc_volumes(self.nr, self.nt, self.np, _d(self.rf), _d(self.tf), _d(self.pf), _d(v))
        return v.reshape(self.shape)

    def dense(self):
        """Materialise A by applying it to unit vectors (small grids only)."""
        if self.N > 4096:
            raise ValueError("dense_of refuses n > 4096 (S:148)")
        A = np.empty((self.N, self.N))
        e = np.zeros(self.N)
        for c in range(self.N):
            e[c] = 1.0
            A[:, c] = self.apply(e).reshape(-1)
            e[c] = 0.0
        return A


POLY_DEFAULT = (4, 100.0)  # PC3: Chebyshev steps m, interval ratio b/a (b = 2)


def set_poly(m=POLY_DEFAULT[0], ratio=POLY_DEFAULT[1]):
    """Parameters of PC3 (Chebyshev-accelerated Jacobi) for the following calls."""
    lib().orc_set_poly(int(m), float(ratio))


def cheb_apply(A, inv_d, r, m, a, b=2.0):
    """z = (I - R_m(D^-1 A)) A^-1 r by the oracle's Chebyshev loop (orc_cheb_apply)
    on a caller operator (dense matrix or callable)."""
    r = _f(r).reshape(-1)
    n = r.size
    fa = (lambda v: A @ v) if isinstance(A, np.ndarray) else A

    def cb(_ctx, x, y):
        np.ctypeslib.as_array(y, shape=(n,))[:] = fa(np.ctypeslib.as_array(x, shape=(n,)).copy())

    c = LINOP(cb)
    z = np.empty(n)
    lib().orc_cheb_apply(n, c, None, _d(_f(inv_d)), int(m), float(a), float(b), _d(r), _d(z))
    return z


def solve(rf, tf, pf, br0, bc=SOURCE_SURFACE, pc=1, pc2_blocks=1, rtol=1e-9, maxit=100000,
          history=False, variant=STANDARD, poly=POLY_DEFAULT, x0=None):
    """Oracle PCG solve.  Returns dict(x, iters, rel_res, true_rel_res, status[, hist]).
    variant: STANDARD or CG1 (Chronopoulos-Gear).
    pc: 1 Jacobi, 2 block ILU0, 3 Chebyshev-accelerated Jacobi (poly = (m, b/a)).
    x0 (np, nt, nr): warm start from x0 instead of 0 (orc_pcg flag X0, A28)."""
    set_poly(*poly)
    rf, tf, pf, br0 = _f(rf), _f(tf), _f(pf), _f(br0)
    nr, nt, np_ = len(rf) - 1, len(tf) - 1, len(pf) - 1
    x = np.zeros(nr * nt * np_) if x0 is None else _f(x0).reshape(-1).copy()
    if x0 is not None:
        if x.size != nr * nt * np_:
            raise ValueError("x0 must have nr*nt*np entries")
        variant = int(variant) | X0
    it = np.zeros(1, dtype=np.int64)
    rr = np.zeros(1)
    tr = np.zeros(1)
    hist = np.zeros(int(maxit) + 1) if history else None
    st = lib().orc_solve_v(nr, nt, np_, _d(rf), _d(tf), _d(pf), bc, pc, pc2_blocks, _d(br0),
                           float(rtol), int(maxit), int(variant), _d(x), _i(it), _d(rr), _d(tr),
                           _d(hist) if history else None)
    out = dict(x=x.reshape(np_, nt, nr), iters=int(it[0]), rel_res=float(rr[0]),
               true_rel_res=float(tr[0]), status=st)
    if history:
        out["hist"] = hist[: out["iters"] + 1]
    return out


def pcg(A, b, rtol=1e-9, maxit=1000, minv=None, variant=STANDARD, history=False, x0=None):
    """The oracle's PCG loop (orc_pcg) on a caller operator: A is a dense
    matrix or a callable x -> A x, minv (optional) a callable r -> M^-1 r.
    Used for the SPEC worked example and random SPD systems.
    x0: warm start (flag X0).  Returns dict(x, iters, rel_res, status[, hist])."""
    b = _f(b).reshape(-1)
    n = b.size
    fa = (lambda v: A @ v) if isinstance(A, np.ndarray) else A
    fm = minv if minv is not None else (lambda v: v.copy())

    def wrap(f):
        def cb(_ctx, x, y):
            xv = np.ctypeslib.as_array(x, shape=(n,))
            np.ctypeslib.as_array(y, shape=(n,))[:] = f(xv.copy())
        return LINOP(cb)

    ca, cm = wrap(fa), wrap(fm)
    x = np.zeros(n) if x0 is None else _f(x0).reshape(-1).copy()
    if x0 is not None:
        variant = int(variant) | X0
    it = np.zeros(1, dtype=np.int64)
    rr = np.zeros(1)
    hist = np.zeros(int(maxit) + 1) if history else None
    st = lib().orc_pcg(n, ca, None, cm, None, _d(b), float(rtol), int(maxit), int(variant), _d(x),
                       _i(it), _d(rr), _d(hist) if history else None)
    out = dict(x=x, iters=int(it[0]), rel_res=float(rr[0]), status=st)
    if history:
        out["hist"] = hist[: out["iters"] + 1]
    return out


def slab_bounds(nr, nblocks):
    """[(i0, i1)] of the r-slab blocks (S:392 leading-remainder rule)."""
    out = []
    for b in range(nblocks):
        i0, i1 = ctypes.c_int(), ctypes.c_int()
        lib().orc_slab_bounds(nr, nblocks, b, ctypes.byref(i0), ctypes.byref(i1))
        out.append((i0.value, i1.value))
    return out


def precond(rf, tf, pf, r, bc=SOURCE_SURFACE, pc=1, pc2_blocks=1, poly=POLY_DEFAULT):
    set_poly(*poly)
    rf, tf, pf, r = _f(rf), _f(tf), _f(pf), _f(r).reshape(-1)
    nr, nt, np_ = len(rf) - 1, len(tf) - 1, len(pf) - 1
    z = np.empty_like(r)
    rc = lib().orc_precond(nr, nt, np_, _d(rf), _d(tf), _d(pf), bc, pc, pc2_blocks, _d(r), _d(z))
    if rc:
        raise RuntimeError(f"preconditioner build failed ({rc})")
    return z.reshape(np_, nt, nr)


def block_ilu0(rf, tf, pf, i0, i1, bc=SOURCE_SURFACE):
    """CSR pattern, A values and ILU0 values of the r-slab block [i0, i1)."""
    rf, tf, pf = _f(rf), _f(tf), _f(pf)
    nr, nt, np_ = len(rf) - 1, len(tf) - 1, len(pf) - 1
    n = (i1 - i0) * nt * np_
    rowptr = np.zeros(n + 1, dtype=np.int64)
    col = np.zeros(7 * n, dtype=np.int64)
    aval = np.zeros(7 * n)
    lu = np.zeros(7 * n)
    rc = lib().orc_block_ilu0(nr, nt, np_, _d(rf), _d(tf), _d(pf), bc, i0, i1, _i(rowptr),
                              _i(col), _d(aval), _d(lu))
    nnz = int(rowptr[-1])
    return rowptr, col[:nnz], aval[:nnz], lu[:nnz], rc


def ilu0_csr(rowptr, col, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    v = _f(val).copy()
    rc = lib().orc_ilu0_csr(len(rowptr) - 1, _i(rowptr), _i(col), _d(v))
    return v, rc


def polar_average(pf, x, south=False):
    x = _f(x)
    np_, nt, nr = x.shape
    avg = np.empty(nr)
    lib().orc_polar_average(nr, nt, np_, _d(_f(pf)), _d(x), int(south), _d(avg))
    return avg


def field(rf, tf, pf, br0, x, bc=SOURCE_SURFACE):
    rf, tf, pf, br0, x = _f(rf), _f(tf), _f(pf), _f(br0), _f(x)
    nr, nt, np_ = len(rf) - 1, len(tf) - 1, len(pf) - 1
    br = np.empty((np_, nt, nr + 1))
    bt = np.empty((np_, nt + 1, nr))
    bp = np.empty((np_, nt, nr))
    rc = lib().orc_field(nr, nt, np_, _d(rf), _d(tf), _d(pf), bc, _d(br0), _d(x), _d(br), _d(bt),
                         _d(bp))
    if rc:
        raise ValueError("invalid grid")
    return br, bt, bp


def solve_fixed(rf, tf, pf, br0, iters, bc=SOURCE_SURFACE, pc=1, pc2_blocks=1):
    """Exactly `iters` PCG iterations (rtol = 0): the timed cpu_baseline sample.
    Returns (x, rel_res, status, seconds spent in the PCG loop)."""
    rf, tf, pf, br0 = _f(rf), _f(tf), _f(pf), _f(br0)
    nr, nt, np_ = len(rf) - 1, len(tf) - 1, len(pf) - 1
    x = np.zeros(nr * nt * np_)
    rr = np.zeros(1)
    secs = np.zeros(1)
    st = lib().orc_solve_fixed(nr, nt, np_, _d(rf), _d(tf), _d(pf), bc, pc, pc2_blocks, _d(br0),
                               int(iters), _d(x), _d(rr), _d(secs))
    return x.reshape(np_, nt, nr), float(rr[0]), st, float(secs[0])


class Session:
    """Timing harness for bench.py (cpu_baseline / --impl reference): the
    oracle system is assembled once, then solve_fixed(iters) runs the
    unchanged PCG loop from x0 = 0 for `iters` iterations and returns
    (rel_res, loop seconds).  Not part of the method."""

    def __init__(self, rf, tf, pf, br0, bc=SOURCE_SURFACE, pc=1, pc2_blocks=1):
        rf, tf, pf, br0 = _f(rf), _f(tf), _f(pf), _f(br0)
        self.nr, self.nt, self.np = len(rf) - 1, len(tf) - 1, len(pf) - 1
        self.N = self.nr * self.nt * self.np
        self._h = lib().orc_session_create(self.nr, self.nt, self.np, _d(rf), _d(tf), _d(pf), bc, pc,
                                           pc2_blocks, _d(br0))
        if not self._h:
            raise ValueError("invalid grid")
        self.x = np.zeros(self.N)

    def solve_fixed(self, iters, variant=STANDARD):
        it = np.zeros(1, dtype=np.int64)
        rr = np.zeros(1)
        secs = np.zeros(1)
        lib().orc_session_solve(self._h, 0.0, int(iters), int(variant), _d(self.x), _i(it), _d(rr),
                                _d(secs))
        return float(rr[0]), float(secs[0])

    def close(self):
        if self._h:
            lib().orc_session_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def threads():
    """OpenMP threads of the oracle's element-wise loops."""
    return int(lib().orc_threads())
