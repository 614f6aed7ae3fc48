"""Seeded synthetic inputs shared by the oracle tests, the CUDA path and bench.py.

This module holds ONLY input recipes: the nonuniform
grid law and the synthetic photospheric Br maps.  It contains none of the
method's arithmetic (no metric coefficients, no operator, no RHS, no PCG), so
the oracle (`oracle/`) and the product path (`paper_1709_01126_b200/`) can both
consume it without sharing any computation.

Readings:
  A12  configuration triples count cells (unknowns), ghosts excluded.
  A13  mesh law: r geometric with dr_last/dr_first = 10, theta faces
       tf(s) = pi*(s - 0.3*sin(2*pi*s)/(2*pi)), s = j/Nt (denser at the poles),
       phi uniform; the `tiny` case is uniform in all three axes; r0=1, r1=2.5.
  A14  the paper's observed magnetogram is replaced by
       Br0 = cos(theta) + sum_{l=2..lmax} sum_{m=-l..l} c_lm * Yhat_lm,
       c_lm = 0.3*N(0,1)/l drawn from numpy.random.default_rng(seed) in (l, m)
       order, Yhat the real spherical harmonic (Re for m>=0, Im of |m| for m<0)
       scaled so that max|Yhat| = 1 on the grid.

Array conventions (identical for the oracle and the C-ABI):
  faces: 1-D float64 arrays of length n+1.
  br0:   float64 array of shape (np, nt) in C order, i.e. theta fastest, the
         Fortran br0(j,k) layout of PAPER.md P:222-224.
  phi:   float64 array of shape (np, nt, nr) in C order, i.e. r fastest, the
         Fortran x(i,j,k) layout.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

R0 = 1.0
R1 = 2.5

SOURCE_SURFACE = 0
CLOSED_WALL = 1


def r_faces(nr: int, r0: float = R0, r1: float = R1, ratio: float = 10.0) -> np.ndarray:
    """Geometric radial faces, dr_{nr-1}/dr_0 = ratio (A13). ratio=1 -> uniform."""
    if nr < 1:
        raise ValueError("nr must be >= 1")
    if ratio == 1.0 or nr == 1:
        return np.linspace(r0, r1, nr + 1)
    q = ratio ** (1.0 / (nr - 1))
    dr = q ** np.arange(nr)
    dr *= (r1 - r0) / dr.sum()
    f = np.empty(nr + 1)
    f[0] = r0
    f[1:] = r0 + np.cumsum(dr)
    f[-1] = r1
    return f


def t_faces(nt: int, stretch: float = 0.3) -> np.ndarray:
    """Theta faces on [0, pi], denser at the poles (A13). stretch=0 -> uniform."""
    s = np.arange(nt + 1) / nt
    f = math.pi * (s - stretch * np.sin(2 * math.pi * s) / (2 * math.pi))
    f[0] = 0.0
    f[-1] = math.pi
    return f


def p_faces(np_: int) -> np.ndarray:
    """Uniform phi faces on [0, 2 pi]."""
    return np.linspace(0.0, 2 * math.pi, np_ + 1)


def centres(faces: np.ndarray) -> np.ndarray:
    return 0.5 * (faces[1:] + faces[:-1])


def grid(nr: int, nt: int, np_: int, uniform: bool = False):
    """(r_faces, t_faces, p_faces) for a config (A13)."""
    if uniform:
        return r_faces(nr, ratio=1.0), t_faces(nt, stretch=0.0), p_faces(np_)
    return r_faces(nr), t_faces(nt), p_faces(np_)


def _assoc_legendre(l: int, m: int, x: np.ndarray) -> np.ndarray:
    from scipy.special import lpmv

    return lpmv(m, l, x)


def real_harmonic(l: int, m: int, tf: np.ndarray, pf: np.ndarray) -> np.ndarray:
    """Yhat_lm sampled at cell centres, shape (np, nt), max|.| = 1 (A14)."""
    tc = centres(tf)
    pc = centres(pf)
    leg = _assoc_legendre(l, abs(m), np.cos(tc))
    ang = np.cos(m * pc) if m >= 0 else np.sin(abs(m) * pc)
    y = ang[:, None] * leg[None, :]
    mx = np.abs(y).max()
    if mx > 0:
        y = y / mx
    return y


def br0_map(tf: np.ndarray, pf: np.ndarray, lmax: int = 0, seed: int = 1,
            amp: float = 0.3) -> np.ndarray:
    """Synthetic magnetogram (A14): dipole cos(theta) + seeded multipoles l=2..lmax."""
    tc = centres(tf)
    npc = len(pf) - 1
    br = np.broadcast_to(np.cos(tc)[None, :], (npc, len(tc))).copy()
    if lmax >= 2:
        rng = np.random.default_rng(seed)
        for l in range(2, lmax + 1):
            for m in range(-l, l + 1):
                c = amp * rng.standard_normal() / l
                br += c * real_harmonic(l, m, tf, pf)
    return np.ascontiguousarray(br)


@dataclass
class Config:
    name: str
    nr: int
    nt: int
    np: int
    uniform: bool = False
    lmax: int = 8
    seed: int = 1
    bc: int = SOURCE_SURFACE
    pc: int = 1
    rtol: float = 1e-9
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.nr * self.nt * self.np

    def faces(self):
        return grid(self.nr, self.nt, self.np, self.uniform)

    def br0(self, faces=None):
        rf, tf, pf = faces if faces is not None else self.faces()
        return br0_map(tf, pf, self.lmax, self.seed)


# BASELINE.json "configs", in order, plus the desk-scale parity cases.
CONFIGS = {
    "tiny": Config("tiny", 21, 31, 61, uniform=True, lmax=0,
                   note="BASELINE configs[0]: uniform dipole, closed-form check"),
    "small": Config("small", 42, 62, 122, note="parity case (oracle in seconds)"),
    "medium": Config("medium", 151, 301, 601, note="BASELINE configs[1]: 1xB200, PC1"),
    "large": Config("large", 301, 601, 1201, note="BASELINE configs[2]: r-sharded strong scaling"),
    "pc2": Config("pc2", 151, 301, 601, pc=2, note="BASELINE configs[3]: PC2 block ILU0"),
    "pc3": Config("pc3", 151, 301, 601, pc=3, note="SURVEY 8(f)-2: Chebyshev-accelerated Jacobi"),
    "pc3large": Config("pc3large", 301, 601, 1201, pc=3, note="SURVEY 8(f)-2 on the large grid"),
    "large8slab": Config("large8slab", 152, 601, 1201,
                         note="4 GPUs x 38 shells: the per-GPU slab of large on 8 GPUs (thin-slab tuning)"),
    "batch": Config("batch", 151, 301, 601, note="SURVEY 8(f)-3: 4 magnetograms (seeds 1-4) per solve",
                    extra={"nrhs": 4}),
    "batchsmall": Config("batchsmall", 42, 62, 122, note="SURVEY 8(f)-3 on a latency-bound grid: 8 maps",
                         extra={"nrhs": 8}),
    "batchpc2": Config("batchpc2", 151, 301, 601, pc=2, note="SURVEY 8(f)-3 with PC2: 4 maps, interleaved sweeps",
                       extra={"nrhs": 4}),
    "batchpc3": Config("batchpc3", 151, 301, 601, pc=3, note="SURVEY 8(f)-3 with PC3: 4 maps",
                       extra={"nrhs": 4}),
}


def batch_maps(c: Config, faces=None) -> np.ndarray:
    """The k = c.extra["nrhs"] maps of a batch config: seeds seed .. seed+k-1 (A14)."""
    rf, tf, pf = faces if faces is not None else c.faces()
    k = c.extra.get("nrhs", 1)
    return np.stack([br0_map(tf, pf, c.lmax, c.seed + q) for q in range(k)])


def weak_config(gpus: int) -> Config:
    """BASELINE configs[4]: ~400M cells per GPU (554 shells per GPU)."""
    return Config(f"weak{gpus}", 554 * gpus, 601, 1201, note="BASELINE configs[4]")


def random_vector(n: int, seed: int = 0) -> np.ndarray:
    """Random operand for operator tests: default_rng(seed).standard_normal(n)."""
    return np.random.default_rng(seed).standard_normal(n)
