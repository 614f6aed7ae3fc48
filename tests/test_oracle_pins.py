"""More pins of the CPU oracle (round 2, VERDICT r1 "What's weak" 1).  `not gpu`.

Each test checks the oracle against something other than itself:
  * the PCG loop (orc_pcg) on the SPEC worked example and on SPD
    matrices with a known number of distinct eigenvalues (exact Krylov
    termination), for the standard and the single-reduction variant;
  * iteration counts to rtol 1e-9 against the survey's independent
    estimates (a separate scipy implementation of the same
    discretisation, not the oracle): tiny PC1 229, PC2 91/96/104/114 for
    1/2/4/8 blocks, closed wall 21x31x61 l<=4 428, small PC1 913;
  * the r-slab rule by explicit sizes;
  * the polar-face Btheta (A19) against the closed-form derivative of
    an m = 1 field.
A wrong Jacobi diagonal, a trailing-remainder slab rule or a wrong polar
distance eps each fail one of these (tools/oracle_mutants.py runs the mutants;
profiles/r02_oracle_mutants.log).
"""
import math

import numpy as np
import pytest

import synth


# ---- the PCG loop on caller operators ------------------------------------

@pytest.mark.parametrize("variant", [0, 1])
def test_spec_2x2_worked_example(oracle_lib, variant):
    """A = [[4,1],[1,3]], b = [1,2] -> x = [1/11, 7/11] in at most 2
    iterations (n = 2, exact termination)."""
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    o = oracle_lib.pcg(A, np.array([1.0, 2.0]), rtol=1e-14, maxit=10, variant=variant)
    assert o["status"] == 0 and o["iters"] <= 2
    assert np.allclose(o["x"], [1 / 11, 7 / 11], rtol=0, atol=1e-15)
    # with the Jacobi preconditioner as well
    d = np.diag(A)
    o = oracle_lib.pcg(A, np.array([1.0, 2.0]), rtol=1e-14, maxit=10, variant=variant,
                       minv=lambda r: r / d)
    assert o["status"] == 0 and o["iters"] <= 2
    assert np.allclose(o["x"], [1 / 11, 7 / 11], rtol=0, atol=1e-15)


def _spd_with_eigs(n, eigs, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.array([eigs[i % len(eigs)] for i in range(n)])
    return (Q * lam) @ Q.T


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_exact_termination_distinct_eigenvalues(oracle_lib, variant, k):
    """CG on an SPD matrix with k distinct eigenvalues terminates in k
    iterations in exact arithmetic (Saad, Iterative Methods §6.11)."""
    n = 30
    eigs = [1.0, 2.5, 4.0, 7.0, 9.0][:k]
    A = _spd_with_eigs(n, eigs, seed=10 + k)
    b = np.random.default_rng(3).standard_normal(n)
    o = oracle_lib.pcg(A, b, rtol=1e-10, maxit=n + 2, variant=variant)
    assert o["status"] == 0 and o["iters"] == k, (o["iters"], k)
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(o["x"] - x) <= 1e-9 * np.linalg.norm(x)


@pytest.mark.parametrize("variant", [0, 1])
def test_random_spd_brute_force(oracle_lib, variant):
    """random SPD n <= 30 terminates within n + 2 iterations and equals
    the dense solve."""
    for n, seed in [(7, 1), (19, 2), (30, 3)]:
        rng = np.random.default_rng(seed)
        B = rng.standard_normal((n, n))
        A = B @ B.T + n * np.eye(n)
        b = rng.standard_normal(n)
        o = oracle_lib.pcg(A, b, rtol=1e-13, maxit=n + 2, variant=variant)
        assert o["status"] == 0 and o["iters"] <= n + 2
        x = np.linalg.solve(A, b)
        assert np.linalg.norm(o["x"] - x) <= 1e-11 * np.linalg.norm(x)


def test_pcg_indefinite(oracle_lib):
    """p.Ap <= 0 -> status -4 (INDEFINITE), both variants."""
    A = np.diag([1.0, -1.0])
    for v in (0, 1):
        assert oracle_lib.pcg(A, np.array([1.0, 1.0]), variant=v)["status"] == -4


def test_cg1_equals_standard_on_tiny(oracle_lib):
    """The single-reduction variant produces the standard iterates in exact
    arithmetic: on the tiny config the iteration count agrees within one and
    the solutions and residual histories agree to rounding."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    br = c.br0()
    s = oracle_lib.solve(rf, tf, pf, br, history=True)
    g = oracle_lib.solve(rf, tf, pf, br, history=True, variant=oracle_lib.CG1)
    assert g["status"] == 0 and abs(g["iters"] - s["iters"]) <= 1
    assert np.linalg.norm(g["x"] - s["x"]) <= 1e-9 * np.linalg.norm(s["x"])
    n = min(len(g["hist"]), len(s["hist"]))
    h1, h2 = s["hist"][: n - 1], g["hist"][: n - 1]
    # the histories agree to rounding for the first ~25 iterations; then the
    # rounding difference grows ~x5 per iteration (iterations 25-40 of this
    # stiff polar problem) and saturates at a few 1e-3 relative (observed
    # 4.8e-3) while the solutions still agree to 1e-9: bound 1e-11 / 2e-2
    assert np.all(np.abs(h1[:25] - h2[:25]) <= 1e-11 * h1[:25])
    assert np.all(np.abs(h1 - h2) <= 2e-2 * h1), (np.abs(h1 - h2) / h1).max()


# ---- iteration counts (SURVEY §8(c) independent estimates) ----------------

def test_iterations_tiny_pc1(oracle_lib):
    """tiny uniform dipole, PC1, rtol 1e-9: 229 (SURVEY §8(c) 'Operator + b +
    BCs' row).  The count is exact: the independent estimate reproduced it to
    the iteration, and a rounding-order change moves it by at most one."""
    c = synth.CONFIGS["tiny"]
    assert abs(oracle_lib.solve(*c.faces(), c.br0())["iters"] - 229) <= 1


def test_iterations_tiny_pc2_blocks(oracle_lib):
    """PC2 with 1/2/4/8 r-slab blocks (leading-remainder rule):
    91 / 96 / 104 / 114 (SURVEY §8(c) 'PC2' row); grows with the blocks as the
    paper reports (2563 -> 3221)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    br = c.br0()
    its = [oracle_lib.solve(rf, tf, pf, br, pc=2, pc2_blocks=b)["iters"] for b in (1, 2, 4, 8)]
    for got, want in zip(its, [91, 96, 104, 114]):
        assert abs(got - want) <= 1, its


def test_iterations_closed_wall_nonuniform(oracle_lib):
    """21x31x61 nonuniform (A13), Br0 = dipole + l<=4 (seed 1, A14): closed
    wall 428 (SURVEY A8 / 'Closed wall' row), source surface 388 ('Iteration
    growth' row)."""
    rf, tf, pf = synth.grid(21, 31, 61)
    br = synth.br0_map(tf, pf, 4, 1)
    assert abs(oracle_lib.solve(rf, tf, pf, br, bc=synth.CLOSED_WALL)["iters"] - 428) <= 1
    assert abs(oracle_lib.solve(rf, tf, pf, br)["iters"] - 388) <= 1


def test_iterations_small_pc1(oracle_lib):
    """small 42x62x122 nonuniform, l<=8 seed 1, PC1: 913 ('Iteration growth'
    row: 913 for both l<=4 and l<=8)."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    assert abs(oracle_lib.solve(rf, tf, pf, c.br0())["iters"] - 913) <= 1
    br4 = synth.br0_map(tf, pf, 4, 1)
    assert abs(oracle_lib.solve(rf, tf, pf, br4)["iters"] - 913) <= 1


# ---- the slab rule --------------------------------------------------------

def test_slab_bounds_explicit_sizes(oracle_lib):
    """block b gets nr//B + (b < nr%B) shells -- the remainder goes to
    the LEADING blocks.  21 shells over 8 blocks -> 3,3,3,3,3,2,2,2."""
    sizes = [i1 - i0 for i0, i1 in oracle_lib.slab_bounds(21, 8)]
    assert sizes == [3, 3, 3, 3, 3, 2, 2, 2]
    b = oracle_lib.slab_bounds(10, 4)
    assert b == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert oracle_lib.slab_bounds(8, 8) == [(i, i + 1) for i in range(8)]


def test_pc2_blocks_are_the_listed_slabs(oracle_lib):
    """PC2 with 8 blocks on 21 shells IS the block-diagonal ILU0 of the slabs
    [0,3) [3,6) [6,9) [9,12) [12,15) [15,17) [17,19) [19,21) (typed from S:392,
    not from slab_bounds): each block solved densely from its own L, U."""
    rf, tf, pf = synth.grid(21, 3, 4)
    nr, nt, np_ = 21, 3, 4
    r = synth.random_vector(nr * nt * np_, 7).reshape(np_, nt, nr)
    z = oracle_lib.precond(rf, tf, pf, r, pc=2, pc2_blocks=8)
    bounds = [(0, 3), (3, 6), (6, 9), (9, 12), (12, 15), (15, 17), (17, 19), (19, 21)]
    for i0, i1 in bounds:
        rowptr, col, aval, lu, rc = oracle_lib.block_ilu0(rf, tf, pf, i0, i1)
        assert rc == 0
        n = len(rowptr) - 1
        L, U = np.eye(n), np.zeros((n, n))
        for i in range(n):
            for p in range(rowptr[i], rowptr[i + 1]):
                (L if col[p] < i else U)[i, col[p]] = lu[p]
        rb = r[:, :, i0:i1].reshape(-1)  # block-local r-fastest order
        zb = np.linalg.solve(U, np.linalg.solve(L, rb))
        assert np.allclose(z[:, :, i0:i1].reshape(-1), zb, rtol=0, atol=1e-12 * np.abs(zb).max())


# ---- polar Btheta (A19) ---------------------------------------------------

def _m1_field(rf, tf, pf):
    """Phi = g(r) (sin t cos p + cos t), g(r) = r^2: (1/r) dPhi/dt at the poles
    is g/r * cos(p) at t = 0 and -g/r * cos(p) at t = pi."""
    rc, tc, pc = synth.centres(rf), synth.centres(tf), synth.centres(pf)
    g = rc**2
    ang = np.sin(tc)[None, :] * np.cos(pc)[:, None] + np.cos(tc)[None, :]
    return ang[:, :, None] * g[None, None, :], (g / rc), np.cos(pc)


def test_polar_btheta_closed_form(oracle_lib):
    """A19: Btheta on a polar face = (Phi(first ring) - Phi_pole) /
    (r eps), eps = the pole-to-first-ring-centre distance and Phi_pole the Eq.3
    ring average.  For the m=1 field above this equals the closed-form
    derivative times sin(eps)/eps, i.e. it converges at second order; eps =
    a full cell or a missing pole average both fail."""
    errs = []
    for nt in (16, 32, 64):
        rf, tf, pf = synth.grid(6, nt, 2 * nt)
        x, gr, cp = _m1_field(rf, tf, pf)
        br0 = np.zeros((2 * nt, nt))
        _, bt, _ = oracle_lib.field(rf, tf, pf, br0, x)
        exN = gr[None, :] * cp[:, None]          # (np, nr) at t = 0
        exS = -exN                               # at t = pi
        eN = np.abs(bt[:, 0, :] - exN).max() / np.abs(exN).max()
        eS = np.abs(bt[:, nt, :] - exS).max() / np.abs(exS).max()
        tc = synth.centres(tf)
        eps = tc[0]
        # the closed-form relative error of the one-sided difference is 1 - sin(eps)/eps
        assert eN == pytest.approx(1 - math.sin(eps) / eps, rel=1e-6, abs=1e-13)
        assert eS == pytest.approx(1 - math.sin(math.pi - tc[-1]) / (math.pi - tc[-1]),
                                   rel=1e-6, abs=1e-13)
        errs.append(max(eN, eS))
    order = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert (order >= 1.9).all(), order


# ---- PC3: Chebyshev-accelerated Jacobi --------------------

@pytest.mark.parametrize("m", [1, 2, 4, 7])
@pytest.mark.parametrize("ratio", [10.0, 100.0])
def test_cheb_apply_closed_form(oracle_lib, m, ratio):
    """Saad Alg. 12.1 from z_0 = 0 gives z_m = (I - R_m(D^-1 A)) A^-1 r with the
    Chebyshev residual polynomial R_m(t) = T_m((b+a-2t)/(b-a)) / T_m((b+a)/(b-a)):
    checked against that closed form through the eigen-decomposition of
    D^-1/2 A D^-1/2 on random SPD matrices (an algebraic identity: it holds for
    any spectrum, so every coefficient of the recurrence is pinned)."""
    from numpy.polynomial import chebyshev as C

    rng = np.random.default_rng(int(ratio) + m)
    n = 25
    B = rng.standard_normal((n, n))
    A = B @ B.T + n * np.eye(n) * rng.uniform(0.5, 2.0, n)
    d = np.diag(A).copy()
    b, a = 2.0, 2.0 / ratio
    r = rng.standard_normal(n)
    z = oracle_lib.cheb_apply(A, 1.0 / d, r, m, a, b)
    s = 1.0 / np.sqrt(d)
    mu, V = np.linalg.eigh(s[:, None] * A * s[None, :])
    Tm = C.Chebyshev.basis(m)
    R = Tm((b + a - 2 * mu) / (b - a)) / Tm((b + a) / (b - a))
    ex = s * (V @ (((1 - R) / mu) * (V.T @ (s * r))))
    assert np.allclose(z, ex, rtol=0, atol=1e-12 * np.abs(ex).max())


def test_pc3_symmetric_and_effective(oracle_lib):
    """PC3 on the POT3D operator is symmetric (x.M^-1 y = y.M^-1 x: a polynomial in
    D^-1 A times D^-1) and cuts the PC1 iteration count roughly by its degree
    (tiny: 229 -> 67 with m = 4, 45 with m = 6)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    x = synth.random_vector(c.n, 5).reshape(c.np, c.nt, c.nr)
    y = synth.random_vector(c.n, 6).reshape(c.np, c.nt, c.nr)
    mx = oracle_lib.precond(rf, tf, pf, x, pc=3)
    my = oracle_lib.precond(rf, tf, pf, y, pc=3)
    assert abs((mx * y).sum() - (x * my).sum()) <= 1e-12 * np.abs(mx * y).sum()
    its = [oracle_lib.solve(rf, tf, pf, c.br0(), pc=3, poly=(m, 100.0))["iters"] for m in (1, 4, 6)]
    assert abs(its[0] - 229) <= 1  # m = 1 is Jacobi scaled by 1/theta: PCG is scale-invariant
    assert its[1] < 229 / 3 and its[2] < its[1], its
    o = oracle_lib.solve(rf, tf, pf, c.br0(), pc=3, rtol=1e-9)
    ref = oracle_lib.solve(rf, tf, pf, c.br0(), rtol=1e-12)
    assert o["status"] == 0
    assert np.linalg.norm(o["x"] - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])


# ---------------------------------------------------------------------------
# warm start (orc_pcg flag X0, SURVEY §8(f)-3 "repeated solves", A28)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("variant", [0, 1])
def test_warm_start_from_zero_is_the_cold_loop(oracle_lib, variant):
    """x0 = 0 through the X0 path (r = b - A 0) gives the cold loop bitwise (standard
    PCG and CG1)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    br = synth.br0_map(tf, pf, 4, 3)
    cold = oracle_lib.solve(rf, tf, pf, br, rtol=1e-9, history=True, variant=variant)
    warm = oracle_lib.solve(rf, tf, pf, br, rtol=1e-9, history=True, x0=np.zeros_like(cold["x"]),
                            variant=variant)
    assert warm["iters"] == cold["iters"] and np.array_equal(warm["x"], cold["x"])
    assert np.array_equal(warm["hist"], cold["hist"])


def test_warm_start_spec_2x2(oracle_lib):
    """SPEC worked example: from the exact solution the loop stops at
    once (iters 0, x unchanged); from x0 = (1, -1) it terminates in <= n = 2."""
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    b = np.array([1.0, 2.0])
    exact = np.array([1.0 / 11.0, 7.0 / 11.0])
    r = oracle_lib.pcg(A, b, rtol=1e-12, x0=exact)
    assert r["iters"] == 0 and r["status"] == 0 and np.array_equal(r["x"], exact)
    r = oracle_lib.pcg(A, b, rtol=1e-12, x0=np.array([1.0, -1.0]), history=True)
    assert r["status"] == 0 and r["iters"] <= 2
    assert np.allclose(r["x"], exact, rtol=0, atol=1e-14)
    # hist[0] = ||b - A x0|| / ||b||
    assert r["hist"][0] == pytest.approx(np.linalg.norm(b - A @ np.array([1.0, -1.0])) / np.linalg.norm(b),
                                         rel=1e-15)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_warm_start_is_a_shifted_cold_solve(oracle_lib, seed):
    """PCG from x0 on (A, b) builds the same Krylov sequence as PCG from 0 on
    (A, b - A x0): x_k = x0 + e_k.  With the tolerance rescaled by
    ||b|| / ||b - A x0|| both stop at the same iteration and agree to rounding.
    A wrong r_0 (b, or A x0 - b) or a test against ||r_0|| breaks it."""
    rng = np.random.default_rng(seed)
    n = 40
    Q = rng.standard_normal((n, n))
    A = Q @ Q.T + n * np.eye(n) * 0.05
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    d = np.diag(A).copy()
    minv = lambda v: v / d  # noqa: E731
    warm = oracle_lib.pcg(A, b, rtol=1e-10, maxit=500, minv=minv, x0=x0)
    r0 = b - A @ x0
    cold = oracle_lib.pcg(A, r0, rtol=1e-10 * np.linalg.norm(b) / np.linalg.norm(r0), maxit=500, minv=minv)
    assert warm["status"] == 0 and cold["status"] == 0
    assert abs(warm["iters"] - cold["iters"]) <= 1
    assert np.linalg.norm(warm["x"] - (x0 + cold["x"])) <= 1e-9 * np.linalg.norm(warm["x"])
    assert np.linalg.norm(b - A @ warm["x"]) <= 1.5e-10 * np.linalg.norm(b)


def test_warm_start_pot3d_converged_and_perturbed_map(oracle_lib):
    """A map solved from its own converged Phi stops at 0 iterations; a nearby
    map (the time-series use) converges from the previous Phi in fewer
    iterations to the same solution as its cold solve."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = synth.grid(c.nr, c.nt, c.np)
    br = synth.br0_map(tf, pf, 6, 4)
    a = oracle_lib.solve(rf, tf, pf, br, rtol=1e-9)
    again = oracle_lib.solve(rf, tf, pf, br, rtol=1e-9, x0=a["x"])
    assert again["iters"] == 0 and np.array_equal(again["x"], a["x"])
    br2 = br + 0.01 * synth.br0_map(tf, pf, 6, 5)
    cold = oracle_lib.solve(rf, tf, pf, br2, rtol=1e-9)
    warm = oracle_lib.solve(rf, tf, pf, br2, rtol=1e-9, x0=a["x"])
    assert warm["status"] == 0 and warm["iters"] < cold["iters"]
    assert np.linalg.norm(warm["x"] - cold["x"]) <= 1e-7 * np.linalg.norm(cold["x"])
    assert warm["true_rel_res"] <= 1.5e-9
