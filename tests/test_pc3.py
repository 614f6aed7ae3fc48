"""PC3 -- Chebyshev-accelerated Jacobi (the "vector-friendly"
preconditioner the paper calls for) -- against its oracle (oracle/
orc_cheb_apply: Saad Alg. 12.1 step by step, pinned by the closed form in
tests/test_oracle_pins.py).  The apply element-wise, full solves within +-1
iteration and 1e-9, several degrees and intervals."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
SS, CW = synth.SOURCE_SURFACE, synth.CLOSED_WALL


def solver(rf, tf, pf, br, poly=(4, 100.0), **kw):
    from paper_1709_01126_b200 import Pot3d

    return Pot3d(rf, tf, pf, br, pc=3, poly=poly, **kw)


@pytest.mark.parametrize("dims", [(3, 5, 7), (9, 23, 129), (21, 31, 61), (42, 62, 122)])
@pytest.mark.parametrize("poly", [(2, 100.0), (4, 100.0), (6, 30.0)])
def test_pc3_apply_matches_oracle(dims, poly):
    rf, tf, pf = synth.grid(*dims)
    x = synth.random_vector(int(np.prod(dims)), 2).reshape(dims[::-1])
    z_ref = oracle.precond(rf, tf, pf, x, pc=3, poly=poly)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0), poly=poly) as s:
        z = s.precond(x)
    assert np.abs(z - z_ref).max() <= 1e-12 * np.abs(z_ref).max()


@pytest.mark.parametrize("name,poly", [("tiny", (4, 100.0)), ("tiny", (6, 100.0)), ("small", (4, 100.0))])
def test_pc3_solve_matches_oracle(name, poly):
    c = synth.CONFIGS[name]
    rf, tf, pf = c.faces()
    ref = oracle.solve(rf, tf, pf, c.br0(), pc=3, poly=poly, rtol=1e-9)
    with solver(rf, tf, pf, c.br0(), poly=poly) as s:
        res = s.solve(rtol=1e-9)
        assert s.info()["pc"] == 3
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    rel = np.linalg.norm(res.phi - ref["x"]) / np.linalg.norm(ref["x"])
    assert rel <= 1e-9, rel
    assert res.true_rel_residual <= 1.5e-9


def test_pc3_closed_wall_and_fixed_iterations():
    rf, tf, pf = synth.grid(10, 17, 40)
    br = synth.br0_map(tf, pf, lmax=3, seed=2)
    ref = oracle.solve(rf, tf, pf, br, bc=synth.CLOSED_WALL, pc=3, rtol=1e-9)
    with solver(rf, tf, pf, br, bc=synth.CLOSED_WALL) as s:
        res = s.solve(rtol=1e-9)
        assert abs(res.iters - ref["iters"]) <= 1
        assert np.linalg.norm(res.phi - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
        for k in (1, 3):
            r = s.solve(rtol=0.0, maxit=k)
            o = oracle.solve(rf, tf, pf, br, bc=synth.CLOSED_WALL, pc=3, rtol=0.0, maxit=k)
            assert np.abs(r.phi - o["x"]).max() <= 1e-12 * np.abs(o["x"]).max()


def test_pc3_rejects_bad_parameters():
    from paper_1709_01126_b200.pot3d import Pot3dError

    c = synth.CONFIGS["tiny"]
    with pytest.raises(Pot3dError):
        solver(*c.faces(), c.br0(), variant=1)
    with pytest.raises(Pot3dError):
        solver(*c.faces(), c.br0(), poly=(1, 100.0))


@pytest.mark.parametrize("k,bc", [(2, SS), (3, SS), (2, CW)])
def test_pc3_loopback_slabs(k, bc):
    """PC3 across r-slabs (loopback groups: the ranks' exchange on one GPU, a halo of d
    between the Chebyshev steps, r.z through the mailboxes): the oracle's PC3 solve
    (the polynomial acts on the global operator, so the slabs do not change it)."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    br = c.br0()
    ref = oracle.solve(rf, tf, pf, br, bc=bc, pc=3, poly=(4, 100.0), rtol=1e-9)
    with solver(rf, tf, pf, br, bc=bc, loopback_slabs=k) as s:
        res = s.solve(rtol=1e-9)
        again = s.solve(rtol=1e-9)
    assert res.status == 0 and abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    assert np.linalg.norm(res.phi - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
    assert again.iters == res.iters and np.array_equal(again.phi, res.phi)
