"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here is `not gpu`.  None of them compares the oracle with itself:
closed-form Laplace solutions, symmetry, null spaces,
dense brute-force solves, the ILU0 defining property,
the SPEC worked examples (S:n, cited per test), exact Krylov termination,
the discrete divergence identity for B = grad Phi.
"""
import math

import numpy as np
import pytest

import synth

R0, R1 = synth.R0, synth.R1


def dipole_exact(rf, tf, bc=synth.SOURCE_SURFACE):
    """Closed form Phi = (a r + b r^-2) cos(theta) with dPhi/dr(r0) = cos(theta)
    (Eq.2) and Phi(r1)=0 (source surface) or dPhi/dr(r1)=0 (closed
    wall).  Radial part solves (1/r^2)(r^2 f')' - 2 f / r^2 = 0."""
    if bc == synth.SOURCE_SURFACE:
        # a - 2 b r0^-3 = 1 ; a r1 + b r1^-2 = 0
        M = np.array([[1.0, -2.0 / R0**3], [R1, R1**-2]])
    else:
        M = np.array([[1.0, -2.0 / R0**3], [1.0, -2.0 / R1**3]])
    a, b = np.linalg.solve(M, np.array([1.0, 0.0]))
    rc = synth.centres(rf)
    tc = synth.centres(tf)
    return (a * rc[None, None, :] + b * rc[None, None, :] ** -2) * np.cos(tc)[None, :, None]


def harmonic_exact(rf, tf, pf, l, m, bc=synth.SOURCE_SURFACE):
    """Phi = (a r^l + b r^{-l-1}) Yhat_lm for Br0 = Yhat_lm."""
    if bc == synth.SOURCE_SURFACE:
        M = np.array([[l * R0 ** (l - 1), -(l + 1) * R0 ** (-l - 2)], [R1**l, R1 ** (-l - 1)]])
    else:
        M = np.array([[l * R0 ** (l - 1), -(l + 1) * R0 ** (-l - 2)],
                      [l * R1 ** (l - 1), -(l + 1) * R1 ** (-l - 2)]])
    a, b = np.linalg.solve(M, np.array([1.0, 0.0]))
    rc = synth.centres(rf)
    Y = synth.real_harmonic(l, m, tf, pf)
    return (a * rc**l + b * rc ** (-l - 1))[None, None, :] * Y[:, :, None]


def test_dipole_closed_form_values():
    # SURVEY §8(c) pin: a = 1/32.25, b = -15.625/32.25, Phi(r0) = -0.4534883721 cos(theta)
    M = np.array([[1.0, -2.0], [R1, R1**-2]])
    a, b = np.linalg.solve(M, np.array([1.0, 0.0]))
    assert a == pytest.approx(1 / 32.25, rel=1e-12)
    assert b == pytest.approx(-15.625 / 32.25, rel=1e-12)
    assert a + b == pytest.approx(-0.4534883721, abs=1e-10)


@pytest.mark.parametrize("uniform", [True, False])
def test_dipole_second_order(oracle_lib, uniform):
    """'globally second-order' with the full spherical metric (A1, A17)."""
    errs = []
    for (a, b, c) in [(8, 12, 24), (16, 24, 48), (32, 48, 96)]:
        rf, tf, pf = synth.grid(a, b, c, uniform=uniform)
        br = synth.br0_map(tf, pf, 0)
        o = oracle_lib.solve(rf, tf, pf, br, rtol=1e-12)
        assert o["status"] == 0
        e = o["x"] - dipole_exact(rf, tf)
        errs.append((np.abs(e).max(), np.sqrt((e**2).mean())))
    errs = np.array(errs)
    order = np.log2(errs[:-1] / errs[1:])
    assert errs[-1, 1] < 2.5e-4
    assert (order[:, 1] >= 1.85).all(), order
    assert (order[:, 0] >= 1.4).all(), order


def test_tiny_config_closed_form(oracle_lib):
    """BASELINE configs[0] (tiny uniform dipole, rtol 1e-9): the closed-form
    check of SURVEY §8(c) (L2 4.26e-4 expected by the survey estimate)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    o = oracle_lib.solve(rf, tf, pf, c.br0(), rtol=1e-9)
    assert o["status"] == 0 and o["rel_res"] <= 1e-9
    e = o["x"] - dipole_exact(rf, tf)
    ex = dipole_exact(rf, tf)
    l2rel = math.sqrt((e**2).mean() / (ex**2).mean())
    assert l2rel < 6e-4
    assert abs(o["true_rel_res"] - o["rel_res"]) < 1e-11


@pytest.mark.parametrize("l,m", [(2, 0), (3, 2), (2, -1)])
def test_multipole_closed_form(oracle_lib, l, m):
    errs = []
    for (a, b, c) in [(10, 16, 32), (20, 32, 64)]:
        rf, tf, pf = synth.grid(a, b, c)
        br = synth.real_harmonic(l, m, tf, pf)
        o = oracle_lib.solve(rf, tf, pf, br, rtol=1e-12)
        ex = harmonic_exact(rf, tf, pf, l, m)
        errs.append(np.sqrt(((o["x"] - ex) ** 2).mean() / (ex**2).mean()))
    assert errs[1] < errs[0] / 3.2, errs   # second order: ratio ~4


def test_closed_wall_closed_form(oracle_lib):
    """Closed wall Br(r1)=0: l=1 solution, zero-mean gauge."""
    errs = []
    for (a, b, c) in [(10, 16, 32), (20, 32, 64)]:
        rf, tf, pf = synth.grid(a, b, c)
        br = synth.br0_map(tf, pf, 0)
        o = oracle_lib.solve(rf, tf, pf, br, bc=synth.CLOSED_WALL, rtol=1e-12)
        assert o["status"] == 0
        ex = dipole_exact(rf, tf, synth.CLOSED_WALL)
        errs.append(np.sqrt(((o["x"] - ex) ** 2).mean() / (ex**2).mean()))
        S = oracle_lib.System(rf, tf, pf, synth.CLOSED_WALL)
        V = S.volumes()
        assert abs((V * o["x"]).sum()) <= 1e-12 * (V * np.abs(o["x"])).sum()
    assert errs[1] < errs[0] / 3.2, errs


@pytest.mark.parametrize("bc", [synth.SOURCE_SURFACE, synth.CLOSED_WALL])
def test_symmetry_dense(oracle_lib, bc):
    """A is symmetric (A3), polar rows included (A5)."""
    rf, tf, pf = synth.grid(4, 6, 8)
    S = oracle_lib.System(rf, tf, pf, bc)
    A = S.dense()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    # positive (semi)definite: -V lap (A4)
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    if bc == synth.SOURCE_SURFACE:
        assert ev.min() > 0
    else:
        assert ev.min() > -1e-12 * ev.max()
        assert np.sort(ev)[1] > 1e-8 * ev.max()   # one-dimensional null space


@pytest.mark.parametrize("bc", [synth.SOURCE_SURFACE, synth.CLOSED_WALL])
def test_symmetry_random_vectors(oracle_lib, bc):
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    S = oracle_lib.System(rf, tf, pf, bc)
    x = synth.random_vector(S.N, 0).reshape(S.shape)
    y = synth.random_vector(S.N, 1).reshape(S.shape)
    lhs = (x * S.apply(y)).sum()
    rhs = (y * S.apply(x)).sum()
    assert abs(lhs - rhs) <= 1e-13 * (np.abs(x * S.apply(y))).sum()


def test_null_space(oracle_lib):
    """Closed wall: A 1 = 0; source surface: A 1 nonzero only
    on the outermost shell."""
    rf, tf, pf = synth.grid(6, 8, 12)
    S = oracle_lib.System(rf, tf, pf, synth.CLOSED_WALL)
    y = S.apply(np.ones(S.shape))
    assert np.abs(y).max() <= 1e-14 * S.diag().max() * 7
    S2 = oracle_lib.System(rf, tf, pf, synth.SOURCE_SURFACE)
    y2 = S2.apply(np.ones(S2.shape))
    assert np.abs(y2[:, :, :-1]).max() <= 1e-14 * S2.diag().max() * 7
    assert (y2[:, :, -1] > 0).all()


def test_coefficient_hand_evaluation(oracle_lib):
    """on a uniform 4x4x8 grid the r coupling between i and i+1 is the
    face area over the centre distance r_{i+1/2}^2 sin t_j dt_j dp_k / dr_{i+1/2}
    (the r_i^2 of the cell volume cancels the 1/r^2 of the Laplacian)."""
    rf, tf, pf = synth.grid(4, 4, 8, uniform=True)
    S = oracle_lib.System(rf, tf, pf)
    nr, nt = 4, 4
    i, j, k = 1, 2, 5
    m = i + nr * (j + nt * k)
    tc = synth.centres(tf)
    dr = rf[1] - rf[0]
    expected = rf[i + 1] ** 2 * math.sin(tc[j]) * (tf[1] - tf[0]) * (pf[1] - pf[0]) / dr
    assert -S.bands[4, m] == pytest.approx(expected, rel=1e-14)
    # an interior row: diagonal = sum of its six couplings (flux form)
    mi = 2 + nr * (1 + nt * 3)
    offd = -(S.bands[:, mi].sum() - S.bands[3, mi])
    assert S.bands[3, mi] == pytest.approx(offd, rel=1e-13)


def test_pole_rows_have_no_polar_coupling(oracle_lib):
    """A5: the pole face weight is sin(0) = 0, so A Phi does not depend on any
    pole value; the row sum of the theta couplings at j=0 has one term only."""
    rf, tf, pf = synth.grid(4, 6, 8)
    S = oracle_lib.System(rf, tf, pf, synth.CLOSED_WALL)
    nr, nt = 4, 6
    for k in range(8):
        for i in range(nr):
            m0 = i + nr * (0 + nt * k)
            m1 = i + nr * (nt - 1 + nt * k)
            assert S.bands[1, m0] == 0.0 and S.bands[5, m1] == 0.0
            # diag equals the sum of present couplings (zero-flux pole face)
            present = -(S.bands[[0, 2, 4, 5, 6], m0].sum())
            wrapc = S.wrap[0, i + nr * 0] if k == 0 else 0.0
            wrapc += S.wrap[1, i + nr * 0] if k == 7 else 0.0
            assert S.bands[3, m0] == pytest.approx(present + wrapc, rel=1e-13)


def test_polar_average_spec_examples(oracle_lib):
    """Eq.3 discrete ring average."""
    rf, tf, pf = synth.grid(3, 4, 16)
    pc = synth.centres(pf)
    x = np.ones((16, 4, 3)) * 2.5
    assert np.allclose(oracle_lib.polar_average(pf, x), 2.5, rtol=0, atol=1e-15)
    x = np.broadcast_to(np.cos(pc)[:, None, None], (16, 4, 3)).copy()
    assert np.abs(oracle_lib.polar_average(pf, x)).max() < 1e-15
    assert np.abs(oracle_lib.polar_average(pf, x, south=True)).max() < 1e-15


def test_rhs_dipole_hand_evaluation(oracle_lib):
    """b(0,j,k) = -r0^2 sin t_j dt_j dp_k Br0(j,k), zero elsewhere."""
    rf, tf, pf = synth.grid(5, 7, 9)
    S = oracle_lib.System(rf, tf, pf)
    br = synth.br0_map(tf, pf, 0)
    b = S.rhs(br)
    tc = synth.centres(tf)
    dt = np.diff(tf)
    dp = np.diff(pf)
    ex = -R0**2 * (np.sin(tc) * dt)[None, :] * dp[:, None] * br
    assert np.allclose(b[:, :, 0], ex, rtol=1e-13, atol=0)
    assert (b[:, :, 1:] == 0).all()
    assert oracle_lib.System(rf, tf, pf).rhs(np.zeros_like(br)).any() == False


def test_rhs_closed_wall_solvability(oracle_lib):
    """S:233, A8: after mean removal sum(b) = 0 (discrete divergence theorem)."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    S = oracle_lib.System(rf, tf, pf, synth.CLOSED_WALL)
    br = c.br0() + 5.0
    b, adj = S.rhs(br, return_adjusted=True)
    assert abs(b.sum()) <= 1e-12 * np.abs(b).sum()  # offset 5 -> cancellation
    # map of a constant is removed entirely ("map = 5 -> 0")
    _, adj5 = S.rhs(np.full_like(br, 5.0), return_adjusted=True)
    assert np.abs(adj5).max() < 5.0 * 1e-13  # relative to the removed constant


@pytest.mark.parametrize("dims", [(4, 6, 8), (6, 8, 12)])
@pytest.mark.parametrize("bc", [synth.SOURCE_SURFACE, synth.CLOSED_WALL])
def test_dense_brute_force(oracle_lib, dims, bc):
    """PCG at rtol 1e-13 vs a dense direct solve (SURVEY §8(c) 'Whole solver')."""
    rf, tf, pf = synth.grid(*dims)
    br = synth.br0_map(tf, pf, lmax=3, seed=2)
    S = oracle_lib.System(rf, tf, pf, bc)
    A = S.dense()
    b = S.rhs(br).reshape(-1)
    if bc == synth.SOURCE_SURFACE:
        xd = np.linalg.solve(A, b)
    else:
        xd = np.linalg.lstsq(A, b, rcond=None)[0]
        V = S.volumes().reshape(-1)
        xd -= (V * xd).sum() / V.sum()
    for pc in (1, 2):
        o = oracle_lib.solve(rf, tf, pf, br, bc=bc, pc=pc, rtol=1e-13)
        assert o["status"] == 0
        err = np.linalg.norm(o["x"].reshape(-1) - xd) / np.linalg.norm(xd)
        assert err <= 1e-10, (pc, err)


def test_exact_termination(oracle_lib):
    """SPD n <= 30 terminates in <= n+2 iterations at tol 1e-14."""
    rf, tf, pf = synth.grid(2, 3, 4)   # n = 24
    br = synth.br0_map(tf, pf, lmax=2, seed=3)
    o = oracle_lib.solve(rf, tf, pf, br, rtol=1e-14)
    assert o["status"] == 0 and o["iters"] <= 26


def test_zero_rhs(oracle_lib):
    """b = 0 -> x = x0 = 0, zero iterations."""
    rf, tf, pf = synth.grid(4, 6, 8)
    o = oracle_lib.solve(rf, tf, pf, np.zeros((8, 6)))
    assert o["iters"] == 0 and o["status"] == 0 and not o["x"].any()


def test_maxit_not_converged(oracle_lib):
    rf, tf, pf = synth.grid(6, 8, 12)
    o = oracle_lib.solve(rf, tf, pf, synth.br0_map(tf, pf, 0), maxit=3)
    assert o["status"] == 1 and o["iters"] == 3 and o["rel_res"] > 1e-9


def _dense_ilu0(A, pattern):
    """Brute-force dense-pattern ILU0 (KIJ form, Saad Alg. 10.4): independent of
    the oracle's CSR IKJ code."""
    n = A.shape[0]
    a = A.copy()
    for k in range(n - 1):
        for i in range(k + 1, n):
            if pattern[i, k]:
                a[i, k] /= a[k, k]
                for j in range(k + 1, n):
                    if pattern[i, j]:
                        a[i, j] -= a[i, k] * a[k, j]
    return a


def test_ilu0_spec_tridiagonal(oracle_lib):
    """{-1, 2, -1}, n=4 -> U diag [2, 3/2, 4/3, 5/4] (exact LU, no fill)."""
    n = 4
    rowptr = [0]
    col, val = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                col.append(j)
                val.append(2.0 if i == j else -1.0)
        rowptr.append(len(col))
    lu, rc = oracle_lib.ilu0_csr(rowptr, col, val)
    assert rc == 0
    diag = [lu[p] for i in range(n) for p in range(rowptr[i], rowptr[i + 1]) if col[p] == i]
    assert np.allclose(diag, [2.0, 1.5, 4 / 3, 1.25], rtol=1e-15)


@pytest.mark.parametrize("blocks", [(0, 4), (0, 2), (2, 4)])
def test_ilu0_defining_property(oracle_lib, blocks):
    """ILU0 (P:88 'zero-fill incomplete LU'): L unit lower, U upper on the
    pattern P of A, and (LU)_ij = a_ij for every (i,j) in P; entrywise equal to
    a brute-force dense-pattern ILU0.  The r-slab block [i0,i1) drops the
    couplings leaving the block and the phi wrap (A11)."""
    rf, tf, pf = synth.grid(4, 5, 6)
    i0, i1 = blocks
    rowptr, col, aval, lu, rc = oracle_lib.block_ilu0(rf, tf, pf, i0, i1)
    assert rc == 0
    n = len(rowptr) - 1
    A = np.zeros((n, n))
    P = np.zeros((n, n), dtype=bool)
    L = np.eye(n)
    U = np.zeros((n, n))
    for i in range(n):
        for p in range(rowptr[i], rowptr[i + 1]):
            j = col[p]
            A[i, j] = aval[p]
            P[i, j] = True
            if j < i:
                L[i, j] = lu[p]
            else:
                U[i, j] = lu[p]
    LU = L @ U
    assert np.abs((LU - A)[P]).max() <= 1e-13 * np.abs(A).max()
    ref = _dense_ilu0(A, P)
    assert np.abs(ref[P] - (np.tril(L, -1) + U)[P]).max() <= 1e-13 * np.abs(A).max()
    # pattern: structural 7-point couplings inside the block only
    nb = i1 - i0
    assert P.sum() == n + 2 * ((nb - 1) * 5 * 6 + nb * 4 * 6 + nb * 5 * 5)


def test_pc2_apply_is_lu_inverse(oracle_lib):
    rf, tf, pf = synth.grid(4, 5, 6)
    rowptr, col, aval, lu, rc = oracle_lib.block_ilu0(rf, tf, pf, 0, 4)
    n = len(rowptr) - 1
    L = np.eye(n)
    U = np.zeros((n, n))
    for i in range(n):
        for p in range(rowptr[i], rowptr[i + 1]):
            (L if col[p] < i else U)[i, col[p]] = lu[p]
    r = synth.random_vector(n, 4)
    z = oracle_lib.precond(rf, tf, pf, r, pc=2).reshape(-1)
    assert np.allclose(L @ U @ z, r, rtol=0, atol=1e-12 * np.abs(r).max())


def test_pc2_symmetric_pairing(oracle_lib):
    """<M^-1 r1, r2> = <r1, M^-1 r2> (ILU0 of a symmetric matrix with
    symmetric pattern is an L D L^T factorisation)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    n = 21 * 31 * 61
    r1 = synth.random_vector(n, 5)
    r2 = synth.random_vector(n, 6)
    for blocks in (1, 3):
        z1 = oracle_lib.precond(rf, tf, pf, r1, pc=2, pc2_blocks=blocks).reshape(-1)
        z2 = oracle_lib.precond(rf, tf, pf, r2, pc=2, pc2_blocks=blocks).reshape(-1)
        assert abs(z1 @ r2 - r1 @ z2) <= 1e-12 * np.abs(z1 * r2).sum()


def test_pc2_iterations_grow_with_blocks(oracle_lib):
    """P:270 (2563 -> 3221 'less effective as the number of processors
    increases'), S:428, S:580 (PC2 <= 0.75 PC1)."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    br = c.br0()
    pc1 = oracle_lib.solve(rf, tf, pf, br)["iters"]
    its = [oracle_lib.solve(rf, tf, pf, br, pc=2, pc2_blocks=b)["iters"] for b in (1, 2, 4, 8)]
    assert its[0] <= 0.75 * pc1
    assert all(its[i] <= its[i + 1] for i in range(3)), its
    assert its[0] < its[-1]


def test_field_boundary_and_linear(oracle_lib):
    """B = grad Phi: Br on the r0 face reproduces Br0 (Eq.2); Phi = r
    gives Br = 1 on interior faces, Bt = Bp = 0; Phi = const -> B = 0
    away from the inhomogeneous faces."""
    rf, tf, pf = synth.grid(6, 8, 12)
    br0 = synth.br0_map(tf, pf, lmax=3)
    rc = synth.centres(rf)
    x = np.broadcast_to(rc[None, None, :], (12, 8, 6)).copy()
    br, bt, bp = oracle_lib.field(rf, tf, pf, br0, x)
    assert np.allclose(br[:, :, 0], br0, rtol=0, atol=1e-13)
    assert np.allclose(br[:, :, 1:-1], 1.0, rtol=0, atol=1e-13)
    assert np.abs(bt).max() < 1e-13 and np.abs(bp).max() < 1e-13


@pytest.mark.parametrize("bc", [synth.SOURCE_SURFACE, synth.CLOSED_WALL])
def test_divergence_identity(oracle_lib, bc):
    """A16: with B on staggered faces, V div_h B (net outward face flux) equals
    the residual b - A Phi exactly, so div B ~ 0 at convergence."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = synth.grid(10, 14, 20)
    br0 = synth.br0_map(tf, pf, lmax=4, seed=2)
    o = oracle_lib.solve(rf, tf, pf, br0, bc=bc, rtol=1e-6)
    S = oracle_lib.System(rf, tf, pf, bc)
    br, bt, bp = oracle_lib.field(rf, tf, pf, br0, o["x"], bc=bc)
    rc, tc = synth.centres(rf), synth.centres(tf)
    dr, dt, dp = np.diff(rf), np.diff(tf), np.diff(pf)
    st = np.sin(tc)
    sf = np.sin(tf)
    sf[0] = sf[-1] = 0.0
    # face areas (np, nt, n*) consistent with B = grad Phi
    ar = (rf**2)[None, None, :] * (st * dt)[None, :, None] * dp[:, None, None]
    at = (rc * dr)[None, None, :] * sf[None, :, None] * dp[:, None, None]
    ap = (rc * dr)[None, None, :] * dt[None, :, None] * np.ones((20, 1, 1))
    Fr = ar * br
    Ft = at * bt
    Fp = ap * bp
    div = (Fr[:, :, 1:] - Fr[:, :, :-1]) + (Ft[:, 1:, :] - Ft[:, :-1, :]) + (Fp - np.roll(Fp, 1, axis=0))
    b = S.rhs(br0)
    res = b - S.apply(o["x"])
    assert np.abs(div - res).max() <= 1e-12 * np.abs(b).max()
    assert np.linalg.norm(div) <= 1.01e-6 * np.linalg.norm(b) + 1e-14


def test_dipole_field_closed_form(oracle_lib):
    """Br at interior r faces vs d/dr of the closed form (second order)."""
    errs = []
    for dims in [(10, 16, 32), (20, 32, 64)]:
        rf, tf, pf = synth.grid(*dims)
        br0 = synth.br0_map(tf, pf, 0)
        o = oracle_lib.solve(rf, tf, pf, br0, rtol=1e-12)
        br, bt, bp = oracle_lib.field(rf, tf, pf, br0, o["x"])
        M = np.array([[1.0, -2.0 / R0**3], [R1, R1**-2]])
        a, b = np.linalg.solve(M, np.array([1.0, 0.0]))
        tc = synth.centres(tf)
        ex = (a - 2 * b * rf**-3)[None, None, :] * np.cos(tc)[None, :, None]
        errs.append(np.sqrt(((br - ex) ** 2).mean() / (ex**2).mean()))
    assert errs[1] < errs[0] / 3.0, errs
