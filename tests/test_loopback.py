"""The multi-GPU r-slab path on ONE GPU:
pot3d_runtime.loopback_slabs = k splits the grid into k slab contexts on the
same device whose kernels exchange exactly as the rank processes of a k-GPU
job do -- the edge shells of p_k stored into the siblings' ghost shells with a
halo flag per iteration, every reduction posted into every slab's mailbox and
summed in rank order -- with the launches ordered on one stream.
Every case against the CPU oracle on the global grid: iterations within 1,
relative L2 <= 1e-9 (north star), PC2 with k slabs = the oracle's block ILU0
with k blocks (leading-remainder slabs, A11)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
SS, CW = synth.SOURCE_SURFACE, synth.CLOSED_WALL


def solver(rf, tf, pf, br, k, **kw):
    from paper_1709_01126_b200 import Pot3d

    return Pot3d(rf, tf, pf, br, loopback_slabs=k, **kw)


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("pc", [1, 2])
def test_loopback_solve_matches_oracle(k, pc):
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    br = c.br0()
    ref = oracle.solve(rf, tf, pf, br, pc=pc, pc2_blocks=k, rtol=1e-9)
    with solver(rf, tf, pf, br, k, pc=pc) as s:
        inf = s.info()
        assert inf["exchange"] == 3 and inf["nr_loc"] == c.nr and inf["pc"] == pc
        res = s.solve(rtol=1e-9)
        again = s.solve(rtol=1e-9)
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    rel = np.linalg.norm(res.phi - ref["x"]) / np.linalg.norm(ref["x"])
    assert rel <= 1e-9, rel
    assert res.true_rel_residual <= 1.5e-9
    # a repeated solve in the same group is bitwise identical (rank-order sums)
    assert again.iters == res.iters and np.array_equal(again.phi, res.phi)


@pytest.mark.parametrize("bc", [SS, CW])
def test_loopback_small_and_field(bc):
    """small (42 shells over 4 slabs of 11/11/10/10, both boundary conditions) and
    B = grad Phi assembled across the slabs (the r faces between slabs use the
    halo of x)."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    br = c.br0()
    ref = oracle.solve(rf, tf, pf, br, bc=bc, rtol=1e-9)
    with solver(rf, tf, pf, br, 4, bc=bc) as s:
        res = s.solve(rtol=1e-9)
        b_r, b_t, b_p = s.field()
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    assert np.linalg.norm(res.phi - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
    obr, obt, obp = oracle.field(rf, tf, pf, br, res.phi, bc=bc)
    for a, b in ((b_r, obr), (b_t, obt), (b_p, obp)):
        assert a.shape == b.shape
        assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()


@pytest.mark.parametrize("k", [2, 5])
def test_loopback_fused_applies_across_slabs(k):
    """A x through the loop's fused passes with the slab halos filled from the
    siblings (pass B stencil, pass A stencil, PC1's pass B), element-wise."""
    rf, tf, pf = synth.grid(13, 29, 70)
    S = oracle.System(rf, tf, pf)
    x = synth.random_vector(S.N, 3).reshape(S.shape)
    y_ref = S.apply(x)
    z_ref = oracle.precond(rf, tf, pf, y_ref, pc=1)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0), k) as s:
        y0 = s.apply(x, which=0)
        y2 = s.apply(x, which=2)
        z1 = s.apply(x, which=1)
        zp = s.precond(x)
    sc = np.abs(y_ref).max()
    assert np.abs(y0 - y_ref).max() <= 1e-13 * sc
    assert np.abs(y2 - y_ref).max() <= 1e-13 * sc
    assert np.abs(z1 - z_ref).max() <= 1e-13 * max(np.abs(z_ref).max(), np.abs(x).max())
    zp_ref = oracle.precond(rf, tf, pf, x, pc=1)
    assert np.abs(zp - zp_ref).max() <= 1e-14 * np.abs(zp_ref).max()


def test_loopback_thin_slabs_pc2():
    """The thinnest legal slabs (2 shells each: 8 slabs over 16 shells), PC2: one
    ILU block per slab = the oracle's 8 blocks."""
    rf, tf, pf = synth.grid(16, 20, 40)
    br = synth.br0_map(tf, pf, lmax=4, seed=4)
    ref = oracle.solve(rf, tf, pf, br, pc=2, pc2_blocks=8, rtol=1e-9)
    with solver(rf, tf, pf, br, 8, pc=2) as s:
        res = s.solve(rtol=1e-9)
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    assert np.linalg.norm(res.phi - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
