"""The single-reduction PCG variant (SURVEY.md §8(f)-1, pot3d_runtime.variant = 1,
PC1) against its own oracle (oracle/ orc_pcg variant CG1: Chronopoulos & Gear as
stated by Ghysels & Vanroose 2014, Alg. 2, step by step): same seeded inputs,
iteration count within 1, solution relative L2 <= 1e-9 (the north star's bar);
fixed-iteration iterates element-wise; the loopback slab groups run the peer-memory
exchange of the rank processes (cg1.cu: K1 stores u's edge shells into the siblings'
ghost shells and raises their halo flags, K2 waits for them and posts its three sums
to every mailbox, k_finalize_cg1_mail sums them in rank order)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
SS, CW = synth.SOURCE_SURFACE, synth.CLOSED_WALL


def solver(rf, tf, pf, br, **kw):
    from paper_1709_01126_b200 import Pot3d

    return Pot3d(rf, tf, pf, br, variant=1, **kw)


def _check(rf, tf, pf, br, bc=SS, k=0, rtol=1e-9):
    ref = oracle.solve(rf, tf, pf, br, bc=bc, rtol=rtol, variant=oracle.CG1)
    with solver(rf, tf, pf, br, bc=bc, loopback_slabs=k) as s:
        res = s.solve(rtol=rtol)
        h = s.history(res.iters + 1)
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    rel = np.linalg.norm(res.phi - ref["x"]) / np.linalg.norm(ref["x"])
    assert rel <= 1e-9, rel
    assert res.rel_residual <= rtol and res.true_rel_residual <= 1.5 * rtol
    assert h[0] == 1.0 and abs(h[-1] - res.rel_residual) <= 1e-15
    return res, ref


def test_cg1_tiny_matches_oracle_and_pcg():
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    res, ref = _check(rf, tf, pf, c.br0())
    # the same discrete solution as the standard recurrences (exact-arithmetic equivalence)
    std = oracle.solve(rf, tf, pf, c.br0(), rtol=1e-9)
    assert abs(res.iters - std["iters"]) <= 2
    assert np.linalg.norm(res.phi - std["x"]) <= 1e-9 * np.linalg.norm(std["x"])


@pytest.mark.parametrize("bc", [SS, CW])
def test_cg1_small_matches_oracle(bc):
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    _check(rf, tf, pf, c.br0(), bc=bc)


@pytest.mark.parametrize("dims", [(3, 5, 7), (9, 23, 129), (21, 31, 61), (42, 62, 122)])
@pytest.mark.parametrize("k", [1, 2, 7])
def test_cg1_fixed_iterations(dims, k):
    rf, tf, pf = synth.grid(*dims)
    br = synth.br0_map(tf, pf, lmax=4, seed=2)
    ref = oracle.solve(rf, tf, pf, br, rtol=0.0, maxit=k, variant=oracle.CG1)
    with solver(rf, tf, pf, br) as s:
        res = s.solve(rtol=0.0, maxit=k)
    assert res.iters == ref["iters"] == k and res.status == 1
    scale = np.abs(ref["x"]).max()
    tol = {1: 1e-14, 2: 1e-13}.get(k, 1e-11 if dims[0] * dims[1] >= 400 else 1e-9)
    assert np.abs(res.phi - ref["x"]).max() <= tol * scale


@pytest.mark.parametrize("k", [2, 3, 5])
def test_cg1_loopback_slabs(k):
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    _check(rf, tf, pf, c.br0(), k=k)


def test_cg1_ragged_and_zero_rhs():
    rf, tf, pf = synth.grid(4, 9, 65)
    _check(rf, tf, pf, synth.br0_map(tf, pf, lmax=4, seed=3))
    with solver(rf, tf, pf, np.zeros((65, 9))) as s:
        r = s.solve()
    assert r.iters == 0 and r.status == 0 and not np.asarray(r.phi).any()
