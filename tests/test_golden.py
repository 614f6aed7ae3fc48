"""Pins of the oracle to the hand-worked values under tests/golden/.

Each fixture line is `name = expression = decimal`, worked out by hand from a
closed form of the paper or a SPEC example; the test first
re-evaluates the expression (a typo guard), then compares the oracle with the
decimal.  Nothing here comes from the CUDA path.  `not gpu`.
"""
import math
import pathlib

import numpy as np
import pytest

import synth

GOLDEN = pathlib.Path(__file__).parent / "golden"


def load(name):
    vals = {}
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, expr, dec = (s.strip() for s in line.split("="))
        v = float(dec)
        ev = eval(expr, {"__builtins__": {}}, {"sin": math.sin, "pi": math.pi})
        assert ev == pytest.approx(v, rel=1e-15, abs=1e-17), (name, key)
        vals[key] = v
    return vals


def test_dipole_golden_against_oracle(oracle_lib):
    """Eq.2 + source surface: the oracle's Phi on a 32x48x96 uniform
    grid matches (a r + b r^-2) cos(theta) with the hand-solved a, b to the
    discretisation error, and the fixture is self-consistent."""
    g = load("dipole_source_surface.txt")
    a, b = g["a"], g["b"]
    assert a - 2 * b == pytest.approx(1.0, rel=1e-15)        # dPhi/dr(r0)=1
    assert 2.5 * a + b / 6.25 == pytest.approx(0.0, abs=1e-16)  # Phi(r1)=0
    assert a + b == pytest.approx(g["phi_r0_over_cos"], rel=1e-15)
    assert 2 * a + b / 4 == pytest.approx(g["phi_r2"], rel=1e-14)
    rf, tf, pf = synth.grid(32, 48, 96, uniform=True)
    o = oracle_lib.solve(rf, tf, pf, synth.br0_map(tf, pf, 0), rtol=1e-12)
    assert o["status"] == 0
    rc, tc = synth.centres(rf), synth.centres(tf)
    ex = (a * rc + b * rc**-2)[None, None, :] * np.cos(tc)[None, :, None]
    err = np.sqrt(((o["x"] - ex) ** 2).mean() / (ex**2).mean())
    assert err < 2e-3, err


def test_coefficient_golden_against_oracle(oracle_lib):
    """radial face coefficient and the source-surface diagonal
    term of one cell of the uniform 4x4x8 grid, hand-evaluated."""
    g = load("coefficient_uniform_4x4x8.txt")
    rf, tf, pf = synth.grid(4, 4, 8, uniform=True)
    S = oracle_lib.System(rf, tf, pf)
    nr, nt = 4, 4
    m = 1 + nr * (2 + nt * 5)
    assert -S.bands[4, m] == pytest.approx(g["a_r_1_2_5"], rel=1e-14)
    mo = 3 + nr * (2 + nt * 5)                       # outer shell, no phi wrap at k=5
    offd = -(S.bands[:, mo].sum() - S.bands[3, mo])
    assert S.bands[3, mo] - offd == pytest.approx(g["s_outer_2_5"], rel=1e-12)
