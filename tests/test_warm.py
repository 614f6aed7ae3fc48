"""Warm start -- repeated solves (pot3d_solve_from; MAS
repeats equivalent PCG solves; A28): the same PCG from a given
x0 (r_0 = b - A x0, the stopping test still relative to ||b||, A9).

Parity: x0 = 0 through the warm path is the cold GPU solve bitwise (r_0 = b - A 0
= b exactly); a warm start from another map's solution matches the oracle's warm
start from the same x0 (orc_pcg flag X0, pinned in test_oracle_pins.py) within the
solve bars of DESIGN.md §6.2; warm=True (the context's last Phi, kept across
pot3d_set_br0) equals passing that Phi explicitly, bitwise; batches take one x0
per problem."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
SS, CW = synth.SOURCE_SURFACE, synth.CLOSED_WALL


def ctx(rf, tf, pf, br, **kw):
    from paper_1709_01126_b200 import Pot3d

    return Pot3d(rf, tf, pf, br, **kw)


@pytest.mark.parametrize("pc,variant", [(1, 0), (2, 0), (3, 0), (1, 1)])
def test_warm_from_zero_is_the_cold_solve(pc, variant):
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    br = c.br0()
    with ctx(rf, tf, pf, br, pc=pc, variant=variant) as s:
        cold = s.solve(rtol=1e-9)
        hc = s.history(cold.iters + 1)
        warm = s.solve(rtol=1e-9, x0=np.zeros_like(cold.phi))
        hw = s.history(warm.iters + 1)
    assert warm.iters == cold.iters and warm.rel_residual == cold.rel_residual
    assert np.array_equal(warm.phi, cold.phi) and np.array_equal(hw, hc)


@pytest.mark.parametrize("bc", [SS, CW])
def test_warm_time_series_against_oracle(bc):
    """Map a, then map b = a + a 2 % perturbation started from Phi(a): fewer
    iterations than b's cold solve, the oracle's warm start from the same x0
    within 1 iteration and 1e-9, and warm=True equal to x0 = Phi(a) bitwise."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = synth.grid(c.nr, c.nt, c.np)
    a = synth.br0_map(tf, pf, 6, 4)
    b = a + 0.02 * synth.br0_map(tf, pf, 6, 9)
    with ctx(rf, tf, pf, a, bc=bc) as s:
        ra = s.solve(rtol=1e-9)
        s.set_br0(b)
        rw = s.solve(rtol=1e-9, warm=True)      # from the context's Phi(a)
        h = s.history(rw.iters + 1)
        rc = s.solve(rtol=1e-9)                 # b cold
        rx = s.solve(rtol=1e-9, x0=ra.phi)      # b from Phi(a) passed explicitly
    assert rw.status == 0 and rw.iters < rc.iters
    assert rx.iters == rw.iters and np.array_equal(rx.phi, rw.phi)
    ow = oracle.solve(rf, tf, pf, b, bc=bc, rtol=1e-9, x0=ra.phi, history=True)
    assert abs(rw.iters - ow["iters"]) <= 1, (rw.iters, ow["iters"])
    assert np.linalg.norm(rw.phi - ow["x"]) <= 1e-9 * np.linalg.norm(ow["x"])
    assert abs(h[0] - ow["hist"][0]) <= 1e-12 * ow["hist"][0]   # ||b - A Phi(a)|| / ||b||
    assert rw.true_rel_residual <= 1.5e-9


def test_warm_converged_start_zero_map_and_states():
    """From its own converged Phi a map stops at 0 iterations with Phi unchanged;
    a zero map returns Phi = 0 from any x0; warm=True after a diagnostic
    apply is refused (the apply overwrote x)."""
    from paper_1709_01126_b200 import Pot3dError

    rf, tf, pf = synth.grid(16, 24, 40)
    br = synth.br0_map(tf, pf, 4, 2)
    with ctx(rf, tf, pf, br) as s:
        r0 = s.solve(rtol=1e-9)
        again = s.solve(rtol=1e-9, warm=True)
        assert again.iters == 0 and np.array_equal(again.phi, r0.phi)
        s.set_br0(np.zeros_like(br))
        z = s.solve(rtol=1e-9, x0=r0.phi)
        assert z.iters == 0 and not z.phi.any() and z.rel_residual == 0.0
        s.set_br0(br)
        s.apply(r0.phi)
        with pytest.raises(Pot3dError, match="state"):
            s.solve(rtol=1e-9, warm=True)
        assert s.solve(rtol=1e-9, x0=r0.phi).iters == 0


def test_warm_batch_per_problem_x0():
    """A batch started from k different x0 equals k single warm solves bitwise."""
    rf, tf, pf = synth.grid(21, 33, 64)
    br = np.stack([synth.br0_map(tf, pf, 4, s) for s in (3, 4, 5)])
    x0 = np.stack([np.zeros((64, 33, 21)), oracle.solve(rf, tf, pf, br[1] * 0.9, rtol=1e-6)["x"],
                   synth.random_vector(21 * 33 * 64, 8).reshape(64, 33, 21) * 1e-3])
    with ctx(rf, tf, pf, br, nrhs=3) as s:
        res = s.solve(rtol=1e-9, x0=x0)
        res2 = s.solve(rtol=1e-9, warm=True)
    assert res.status == 0 and (res2.iters == 0).all()
    for q in range(3):
        with ctx(rf, tf, pf, br[q]) as one:
            r1 = one.solve(rtol=1e-9, x0=x0[q])
        assert res.iters[q] == r1.iters and np.array_equal(res.phi[q], r1.phi), q
    assert res.iters[1] < res.iters[0]


@pytest.mark.parametrize("k,variant", [(2, 0), (3, 0), (2, 1)])
def test_warm_loopback_slabs(k, variant):
    """Warm starts across r-slabs (loopback groups run the ranks' exchange on one GPU):
    x0 = 0 is the cold solve bitwise; from the previous Phi the oracle's warm start."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    a = c.br0()
    b = a + 0.02 * synth.br0_map(tf, pf, 4, 9)
    with ctx(rf, tf, pf, a, loopback_slabs=k, variant=variant) as s:
        cold = s.solve(rtol=1e-9)
        zero = s.solve(rtol=1e-9, x0=np.zeros_like(cold.phi))
        s.set_br0(b)
        warm = s.solve(rtol=1e-9, warm=True)
    assert zero.iters == cold.iters and np.array_equal(zero.phi, cold.phi)
    ow = oracle.solve(rf, tf, pf, b, rtol=1e-9, variant=variant, x0=cold.phi)
    assert warm.status == 0 and abs(warm.iters - ow["iters"]) <= 1, (warm.iters, ow["iters"])
    assert np.linalg.norm(warm.phi - ow["x"]) <= 1e-9 * np.linalg.norm(ow["x"])
