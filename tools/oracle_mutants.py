"""Mutation check of the oracle pins (VERDICT r1 "Next round" 1: a wrong eps,
a wrong PC1 diagonal or trailing-remainder slabs must each fail a committed
test).  Builds deliberately broken copies of oracle/pot3d_oracle.c under /tmp,
runs the `not gpu` oracle tests against each (POT3D_ORACLE_LIB), and reports
which tests catch it.  Output: profiles/r02_oracle_mutants.log.
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = (ROOT / "oracle" / "pot3d_oracle.c").read_text()
TESTS = ["tests/test_oracle.py", "tests/test_oracle_pins.py", "tests/test_golden.py"]

MUTANTS = {
    "pc1_diag_of_next_cell": (
        "M->inv_diag[m] = 1.0 / bands[3 * N + m];",
        "M->inv_diag[m] = 1.0 / bands[3 * N + (m + 1) % N];"),
    "pc1_diag_without_theta_terms": (
        "M->inv_diag[m] = 1.0 / bands[3 * N + m];",
        "M->inv_diag[m] = 1.0 / (bands[3 * N + m] + bands[1 * N + m] + bands[5 * N + m]);"),
    "slabs_trailing_remainder": (
        "*i0 = b * base + (b < rem ? b : rem);\n  *i1 = *i0 + base + (b < rem ? 1 : 0);",
        "int lead = nblocks - rem;\n  *i0 = b * base + (b > lead ? b - lead : 0);\n"
        "  *i1 = *i0 + base + (b >= lead ? 1 : 0);"),
    "polar_eps_full_cell": (
        "(g.rc[i] * (g.tc[0] - tf[0]))", "(g.rc[i] * g.dt[0])"),
    "polar_eps_south_full_cell": (
        "(g.rc[i] * (tf[nt] - g.tc[nt - 1]))", "(g.rc[i] * g.dt[nt - 1])"),
    "polar_average_dropped": (
        "v = (X(i, 0, k) - poleN[i])", "v = (X(i, 0, k) - 0.0)"),
    "theta_face_sine_at_centre": (
        "return V * g->stf[j + 1] / (g->rc[i] * g->rc[i] * g->st[j] * g->dt[j] * g->dth[j]);",
        "return V * g->st[j] / (g->rc[i] * g->rc[i] * g->st[j] * g->dt[j] * g->dth[j]);"),
    "ilu0_no_update": (
        "if (pos[jj] >= 0) c->val[pos[jj]] -= lik * c->val[q];",
        "if (pos[jj] >= 0 && 0) c->val[pos[jj]] -= lik * c->val[q];"),
    "cg1_den_without_beta": (
        "double den = delta - beta * gamma_new / alpha;",
        "double den = delta - gamma_new / alpha;"),
    "pcg_beta_inverted": (
        "double beta = rho_new / rho;", "double beta = rho / rho_new;"),
    "warm_r0_ignores_x0": (
        "for (int64_t m = 0; m < N; m++) r[m] = b[m] - r[m];",
        "for (int64_t m = 0; m < N; m++) r[m] = b[m];"),
    "warm_norm_of_r0_not_b": (
        "const double bnorm = sqrt(dot(N, b, b));\n  int64_t k = 0;",
        "const double bnorm = sqrt(dot(N, r, r));\n  int64_t k = 0;"),
    "rhs_sign": (
        "= -c * br[j + (int64_t)nt * k] * dr1;", "= c * br[j + (int64_t)nt * k] * dr1;"),
}


def main():
    out = []
    env0 = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    for name, (a, b) in MUTANTS.items():
        assert SRC.count(a) == 1, (name, SRC.count(a))
        src = SRC.replace(a, b)
        c = Path(f"/tmp/oracle_mut_{name}.c")
        so = c.with_suffix(".so")
        c.write_text(src)
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                               "-std=c11", "-o", str(so), str(c), "-lm"])
        env = dict(env0, POT3D_ORACLE_LIB=str(so))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
        failed = sorted({l.split(" ")[1].split(" - ")[0] for l in r.stdout.splitlines()
                         if l.startswith("FAILED")})
        line = f"{name}: {'CAUGHT' if failed else 'NOT CAUGHT'} by {len(failed)} test(s)"
        out.append(line)
        out += [f"    {f}" for f in failed]
        print(line, flush=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider", *TESTS],
                       cwd=ROOT, env=env0, capture_output=True, text=True)
    out.append("unmutated oracle: " + r.stdout.strip().splitlines()[-1])
    (ROOT / "profiles" / "r02_oracle_mutants.log").write_text(
        "# tools/oracle_mutants.py: each mutant is a deliberately broken oracle build;\n"
        "# the listed `not gpu` tests fail on it.\n" + "\n".join(out) + "\n")
    print(out[-1])


if __name__ == "__main__":
    main()
