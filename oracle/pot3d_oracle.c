/*
 * pot3d_oracle.c -- plain, slow, obviously-correct CPU fp64 oracle for the POT3D
 * potential-field PCG solve of arXiv 1709.01126 ("From MPI to MPI+OpenACC ...").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA product path in
 * paper_1709_01126_b200/ and neither side includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (the paper's LaTeX);
 *            S:n = /root/reference/SPEC.md line n;
 *            A<n> = reading A<n> of SURVEY.md §8(c), restated in DESIGN.md.
 *
 * Structure follows the paper, not the GPU design:
 *   - unknowns Phi_{i,j,k} cell-centred (A2), stored r-fastest
 *     m = i + nr*(j + nt*k) like the Fortran x(i,j,k) of P:222-224;
 *   - the interior matrix A is stored in DIA format, 7 bands, with
 *     offsets [-nr*nt, -nr, -1, 0, +1, +nr, +nr*nt];
 *   - the boundary conditions are applied matrix-free: the periodic
 *     phi wrap through ghost values, the photospheric Br Neumann data
 *     (Eq.2) through the ghost fill x(1)=x(2)-vmask*br0*dr1
 *      which puts the inhomogeneous part into b, the outer
 *     source-surface / closed-wall condition folded into the diagonal,
 *     the polar average (Eq.3) whose face weight is sin(0)=0 (A5);
 *   - PCG exactly as the standard algorithm, PC1 = inverse
 *     of diag(A), PC2 = zero-fill ILU of each r-slab block with the
 *     generic IKJ algorithm on CSR (A11) and sequential
 *     forward/backward triangular solves ("standard algorithm ... not
 *     vectorizable").
 *
 * Each function names the passage it follows.  Parity is pinned by
 * tests/test_oracle_*.py (closed forms, symmetry, dense brute force, ILU0
 * defining property, SPEC worked examples, divergence identity).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_SOURCE_SURFACE 0
#define ORC_CLOSED_WALL 1

/* ------------------------------------------------------------------------ */
/* Mesh: cell-centred nonuniform spherical grid (A2).         */
/* ------------------------------------------------------------------------ */
typedef struct {
  int nr, nt, np;
  double *rf, *tf, *pf;   /* faces, n+1 */
  double *rc, *tc, *pc;   /* centres = face midpoints (A2) */
  double *dr, *dt, *dp;   /* main-mesh widths  Delta x_i = f_{i+1}-f_i            */
  double *drh, *dth, *dph;/* half-mesh widths  Delta x_{i+1/2} = c_{i+1}-c_i      */
  double *st;             /* sin(theta_j) at centres                               */
  double *stf;            /* sin(theta_{j-1/2}) at faces, exactly 0 at the poles   */
  double period;          /* pf[np]-pf[0] = 2 pi                                   */
} orc_mesh;

static void mesh_free(orc_mesh *g) {
  free(g->rc); free(g->tc); free(g->pc);
  free(g->dr); free(g->dt); free(g->dp);
  free(g->drh); free(g->dth); free(g->dph);
  free(g->st); free(g->stf);
}

static int mesh_build(orc_mesh *g, int nr, int nt, int np, const double *rf,
                      const double *tf, const double *pf) {
  if (nr < 2 || nt < 2 || np < 2) return -1;
  for (int i = 0; i < nr; i++) if (!(rf[i + 1] > rf[i])) return -1;
  for (int j = 0; j < nt; j++) if (!(tf[j + 1] > tf[j])) return -1;
  for (int k = 0; k < np; k++) if (!(pf[k + 1] > pf[k])) return -1;
  if (!(rf[0] > 0.0)) return -1;
  g->nr = nr; g->nt = nt; g->np = np;
  g->rf = (double *)rf; g->tf = (double *)tf; g->pf = (double *)pf;
  g->rc = malloc(sizeof(double) * nr); g->dr = malloc(sizeof(double) * nr);
  g->drh = malloc(sizeof(double) * nr);
  g->tc = malloc(sizeof(double) * nt); g->dt = malloc(sizeof(double) * nt);
  g->dth = malloc(sizeof(double) * nt);
  g->pc = malloc(sizeof(double) * np); g->dp = malloc(sizeof(double) * np);
  g->dph = malloc(sizeof(double) * np);
  g->st = malloc(sizeof(double) * nt); g->stf = malloc(sizeof(double) * (nt + 1));
  for (int i = 0; i < nr; i++) { g->rc[i] = 0.5 * (rf[i] + rf[i + 1]); g->dr[i] = rf[i + 1] - rf[i]; }
  for (int j = 0; j < nt; j++) { g->tc[j] = 0.5 * (tf[j] + tf[j + 1]); g->dt[j] = tf[j + 1] - tf[j]; }
  for (int k = 0; k < np; k++) { g->pc[k] = 0.5 * (pf[k] + pf[k + 1]); g->dp[k] = pf[k + 1] - pf[k]; }
  /* Delta x_{i+1/2} between consecutive centres; the last r/theta
   * entry is unused; phi wraps periodically. */
  for (int i = 0; i < nr - 1; i++) g->drh[i] = g->rc[i + 1] - g->rc[i];
  g->drh[nr - 1] = 0.0;
  for (int j = 0; j < nt - 1; j++) g->dth[j] = g->tc[j + 1] - g->tc[j];
  g->dth[nt - 1] = 0.0;
  g->period = pf[np] - pf[0];
  for (int k = 0; k < np - 1; k++) g->dph[k] = g->pc[k + 1] - g->pc[k];
  g->dph[np - 1] = g->pc[0] + g->period - g->pc[np - 1];
  for (int j = 0; j < nt; j++) g->st[j] = sin(g->tc[j]);
  /* sin(theta_{j-1/2}) at faces.  The faces at theta=0 and theta=pi ARE the
   * poles, where sin vanishes exactly (A5: the polar face has zero area). */
  for (int j = 0; j <= nt; j++) g->stf[j] = sin(tf[j]);
  g->stf[0] = 0.0;
  g->stf[nt] = 0.0;
  return 0;
}

/* Cell volume r_i^2 sin(theta_j) dr_i dtheta_j dphi_k: the row scaling that
 * makes A symmetric ("symmetric", A3). */
static double cell_volume(const orc_mesh *g, int i, int j, int k) {
  return g->rc[i] * g->rc[i] * g->st[j] * g->dr[i] * g->dt[j] * g->dp[k];
}

/* Volume-scaled coefficients of the flux-difference stencil of P:65-76 with
 * the full spherical metric (A1):
 *   lap = 1/(r^2 dr_i) [ r_{i+1/2}^2 (P_{i+1}-P_i)/dr_{i+1/2} - r_{i-1/2}^2 (P_i-P_{i-1})/dr_{i-1/2} ]
 *       + 1/(r^2 sin t_j dt_j) [ sin t_{j+1/2} (P_{j+1}-P_j)/dt_{j+1/2} - sin t_{j-1/2} (...) ]
 *       + 1/(r^2 sin^2 t_j dp_k) [ (P_{k+1}-P_k)/dp_{k+1/2} - (P_k-P_{k-1})/dp_{k-1/2} ]
 * A = -V * lap (A4), so each coefficient below is V times the factor in front
 * of (P_nbr - P_centre). */
static double coef_rp(const orc_mesh *g, int i, int j, int k, double drface) {
  double V = cell_volume(g, i, j, k);
  return V * g->rf[i + 1] * g->rf[i + 1] / (g->rc[i] * g->rc[i] * g->dr[i] * drface);
}
static double coef_rm(const orc_mesh *g, int i, int j, int k, double drface) {
  double V = cell_volume(g, i, j, k);
  return V * g->rf[i] * g->rf[i] / (g->rc[i] * g->rc[i] * g->dr[i] * drface);
}
static double coef_tp(const orc_mesh *g, int i, int j, int k) {
  double V = cell_volume(g, i, j, k);
  if (j == g->nt - 1) return 0.0; /* pole face (A5) */
  return V * g->stf[j + 1] / (g->rc[i] * g->rc[i] * g->st[j] * g->dt[j] * g->dth[j]);
}
static double coef_tm(const orc_mesh *g, int i, int j, int k) {
  double V = cell_volume(g, i, j, k);
  if (j == 0) return 0.0; /* pole face (A5) */
  return V * g->stf[j] / (g->rc[i] * g->rc[i] * g->st[j] * g->dt[j] * g->dth[j - 1]);
}
static double coef_pp(const orc_mesh *g, int i, int j, int k) {
  double V = cell_volume(g, i, j, k);
  return V / (g->rc[i] * g->rc[i] * g->st[j] * g->st[j] * g->dp[k] * g->dph[k]);
}
static double coef_pm(const orc_mesh *g, int i, int j, int k) {
  double V = cell_volume(g, i, j, k);
  int km = (k == 0) ? g->np - 1 : k - 1;
  return V / (g->rc[i] * g->rc[i] * g->st[j] * g->st[j] * g->dp[k] * g->dph[km]);
}

/* ------------------------------------------------------------------------ */
/* Operator assembly in DIA format.               */
/* bands: 7*N doubles, band d at row m = coefficient of column m+off[d].     */
/* wrap:  2*nr*nt doubles: [0] coupling of k=0 to its ghost k=-1 (= cell    */
/*        np-1), [1] coupling of k=np-1 to its ghost k=np (= cell 0).        */
/*        These are the matrix-free periodic BC couplings.      */
/* ------------------------------------------------------------------------ */
int orc_assemble(int nr, int nt, int np, const double *rf, const double *tf,
                 const double *pf, int bc, double *bands, double *wrap) {
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return -1;
  const int64_t N = (int64_t)nr * nt * np;
  memset(bands, 0, sizeof(double) * 7 * N);
#pragma omp parallel for schedule(static)
  for (int k = 0; k < np; k++)
    for (int j = 0; j < nt; j++)
      for (int i = 0; i < nr; i++) {
        int64_t m = i + (int64_t)nr * (j + (int64_t)nt * k);
        double diag = 0.0, c;
        /* r direction.  Inner face (i=0): homogeneous Neumann ghost
         * x(1)=x(2) (vmask=0, A6) contributes nothing; its inhomogeneous
         * part lives in b (orc_rhs).  Outer face (i=nr-1): source surface
         * Phi=0 on the face, ghost = -Phi (A7) -> 2*c on the diagonal; the
         * closed wall (Br=0) ghost = +Phi contributes nothing. */
        if (i < nr - 1) {
          c = coef_rp(&g, i, j, k, g.drh[i]);
          bands[4 * N + m] = -c; diag += c;
        } else if (bc == ORC_SOURCE_SURFACE) {
          c = coef_rp(&g, i, j, k, g.dr[nr - 1]); /* ghost centre mirrored: distance dr_{nr-1} */
          diag += 2.0 * c;
        }
        if (i > 0) {
          c = coef_rm(&g, i, j, k, g.drh[i - 1]);
          bands[2 * N + m] = -c; diag += c;
        }
        /* theta direction; pole faces carry sin(0)=0 weight (A5). */
        c = coef_tp(&g, i, j, k);
        if (j < nt - 1) bands[5 * N + m] = -c;
        diag += c;
        c = coef_tm(&g, i, j, k);
        if (j > 0) bands[1 * N + m] = -c;
        diag += c;
        /* phi direction, periodic: interior couplings in the bands,
         * the k=0 <-> k=np-1 coupling matrix-free through ghosts. */
        c = coef_pp(&g, i, j, k);
        if (k < np - 1) bands[6 * N + m] = -c;
        else wrap[1 * (int64_t)nr * nt + i + (int64_t)nr * j] = c;
        diag += c;
        c = coef_pm(&g, i, j, k);
        if (k > 0) bands[0 * N + m] = -c;
        else wrap[0 * (int64_t)nr * nt + i + (int64_t)nr * j] = c;
        diag += c;
        bands[3 * N + m] = diag;
      }
  mesh_free(&g);
  return 0;
}

/* y = A x : DIA product over the interior plus the matrix-free
 * periodic-phi ghost couplings.  r/theta boundary ghosts are
 * homogeneous in the Krylov operator (A6) and already folded in. */
void orc_apply(int nr, int nt, int np, const double *bands, const double *wrap,
               const double *x, double *y) {
  const int64_t N = (int64_t)nr * nt * np;
  const int64_t off[7] = {-(int64_t)nr * nt, -(int64_t)nr, -1, 0, 1, nr, (int64_t)nr * nt};
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < N; m++) {
    double s = 0.0;
    for (int d = 0; d < 7; d++) {
      int64_t c = m + off[d];
      if (c >= 0 && c < N) s += bands[d * N + m] * x[c];
    }
    y[m] = s;
  }
  /* phi ghosts: x(k=-1) = x(np-1), x(k=np) = x(0). */
  const int64_t plane = (int64_t)nr * nt;
#pragma omp parallel for schedule(static)
  for (int64_t ij = 0; ij < plane; ij++) {
    y[ij] -= wrap[ij] * x[ij + plane * (np - 1)];
    y[ij + plane * (np - 1)] -= wrap[plane + ij] * x[ij];
  }
}

/* Solvability for the closed wall (pure Neumann): subtract the area-weighted
 * mean, weights sin(t_j) dt_j dp_k (A8). */
static void enforce_solvability(const orc_mesh *g, double *br) {
  double sw = 0.0, swb = 0.0;
  for (int k = 0; k < g->np; k++)
    for (int j = 0; j < g->nt; j++) {
      double w = g->st[j] * g->dt[j] * g->dp[k];
      sw += w; swb += w * br[j + (int64_t)g->nt * k];
    }
  double mean = swb / sw;
  for (int64_t q = 0; q < (int64_t)g->nt * g->np; q++) br[q] -= mean;
}

/* b from the photospheric Neumann data (Eq.2): with the ghost fill
 * x(1,:,:) = x(2,:,:) - vmask*br0*dr1 (A6: dr1 = Delta r_{-1/2}
 * = dr_0 for the mirrored ghost), the row i=0 of -V*lap reads
 *   (A Phi)_0 + c_{r-}(i=0) * (Phi_0 - Phi_ghost) = 0,
 * so b_0 = -c_{r-}(i=0) * br0 * dr1 and b = 0 elsewhere.
 * br_adj (nt*np, may be NULL) receives the (solvability-adjusted) map. */
int orc_rhs(int nr, int nt, int np, const double *rf, const double *tf,
            const double *pf, int bc, const double *br0, double *b, double *br_adj) {
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return -1;
  const int64_t N = (int64_t)nr * nt * np;
  double *br = malloc(sizeof(double) * nt * np);
  memcpy(br, br0, sizeof(double) * nt * np);
  if (bc == ORC_CLOSED_WALL) enforce_solvability(&g, br);
  for (int64_t m = 0; m < N; m++) b[m] = 0.0;
  const double dr1 = g.dr[0];
  for (int k = 0; k < np; k++)
    for (int j = 0; j < nt; j++) {
      double c = coef_rm(&g, 0, j, k, dr1);
      b[(int64_t)nr * (j + (int64_t)nt * k)] = -c * br[j + (int64_t)nt * k] * dr1;
    }
  if (br_adj) memcpy(br_adj, br, sizeof(double) * nt * np);
  free(br);
  mesh_free(&g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* CSR, ILU0 (IKJ) and triangular solves: PC2.       */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t *rowptr;
  int64_t *col;
  double *val;
  int64_t *diagpos;
  double *a0;  /* ORC_ILU_DFORM only: A's values on the pattern */
} orc_csr;

static void csr_free(orc_csr *c) {
  free(c->rowptr); free(c->col); free(c->val); free(c->diagpos);
#ifdef ORC_ILU_DFORM
  free(c->a0);
#endif
}

/* dia_to_csr restricted to one r-slab block [i0,i1):
 * couplings leaving the block, and the periodic phi wrap (a matrix-free BC,
 * P:83), are dropped (truncation); the full diagonal is kept (A11).
 * Only structural couplings enter the pattern (A11).  Local ordering is the
 * global r-fastest ordering restricted to the block. */
static void block_csr(int nr, int nt, int np, const double *bands, int i0, int i1, orc_csr *c) {
  const int64_t N = (int64_t)nr * nt * np;
  const int nb = i1 - i0;
  const int64_t n = (int64_t)nb * nt * np;
  c->n = n;
  c->rowptr = malloc(sizeof(int64_t) * (n + 1));
  c->col = malloc(sizeof(int64_t) * n * 7);
  c->val = malloc(sizeof(double) * n * 7);
  c->a0 = NULL;
  c->diagpos = malloc(sizeof(int64_t) * n);
  int64_t nnz = 0;
  for (int k = 0; k < np; k++)
    for (int j = 0; j < nt; j++)
      for (int il = 0; il < nb; il++) {
        int i = i0 + il;
        int64_t m = i + (int64_t)nr * (j + (int64_t)nt * k);
        int64_t row = il + (int64_t)nb * (j + (int64_t)nt * k);
        c->rowptr[row] = nnz;
        /* columns in increasing local order: k-1, j-1, i-1, diag, i+1, j+1, k+1 */
        if (k > 0)      { c->col[nnz] = row - (int64_t)nb * nt; c->val[nnz++] = bands[0 * N + m]; }
        if (j > 0)      { c->col[nnz] = row - nb;               c->val[nnz++] = bands[1 * N + m]; }
        if (il > 0)     { c->col[nnz] = row - 1;                c->val[nnz++] = bands[2 * N + m]; }
        c->diagpos[row] = nnz;
        c->col[nnz] = row; c->val[nnz++] = bands[3 * N + m];
        if (il < nb - 1){ c->col[nnz] = row + 1;                c->val[nnz++] = bands[4 * N + m]; }
        if (j < nt - 1) { c->col[nnz] = row + nb;               c->val[nnz++] = bands[5 * N + m]; }
        if (k < np - 1) { c->col[nnz] = row + (int64_t)nb * nt; c->val[nnz++] = bands[6 * N + m]; }
      }
  c->rowptr[n] = nnz;
}

/* Zero-fill ILU, row-wise IKJ variant (Saad):
 *   for i: for k in row i, k < i: a_ik /= a_kk;
 *            for j in row i, j > k: a_ij -= a_ik * a_kj   (only if (k,j) in pattern)
 * L (unit lower) and U (upper incl. diagonal) overwrite val.  Returns -2 on a
 * pivot with |u_ii| < 1e-300 (breakdown). */
static int ilu0_ikj(orc_csr *c) {
  const int64_t n = c->n;
  int64_t *pos = malloc(sizeof(int64_t) * n);
  for (int64_t q = 0; q < n; q++) pos[q] = -1;
  int rc = 0;
  for (int64_t i = 0; i < n && rc == 0; i++) {
    for (int64_t p = c->rowptr[i]; p < c->rowptr[i + 1]; p++) pos[c->col[p]] = p;
    for (int64_t p = c->rowptr[i]; p < c->rowptr[i + 1]; p++) {
      int64_t k = c->col[p];
      if (k >= i) break;
      double ukk = c->val[c->diagpos[k]];
      double lik = c->val[p] / ukk;
      c->val[p] = lik;
      for (int64_t q = c->diagpos[k] + 1; q < c->rowptr[k + 1]; q++) {
        int64_t jj = c->col[q];
        if (pos[jj] >= 0) c->val[pos[jj]] -= lik * c->val[q];
      }
    }
    if (fabs(c->val[c->diagpos[i]]) < 1e-300) rc = -2;
    for (int64_t p = c->rowptr[i]; p < c->rowptr[i + 1]; p++) pos[c->col[p]] = -1;
  }
  free(pos);
  return rc;
}

/* z = U^{-1} L^{-1} r, sequential forward then backward substitution (P:97
 * "standard algorithm ... not vectorizable"). */
static void lusolve(const orc_csr *c, const double *r, double *z) {
  const int64_t n = c->n;
#ifdef ORC_ILU_DFORM
  /* the same (LU)^-1 in D-ILU form (tools/oracle_spread.py only): with L = I + A_L D^-1,
   * U = D + A_U, D = diag(U): w = D^-1 (r - A_L w), z = w - D^-1 A_U z -- an equally
   * valid evaluation order; a0 holds A's values on the pattern */
  for (int64_t i = 0; i < n; i++) {
    double s = r[i];
    for (int64_t p = c->rowptr[i]; p < c->diagpos[i]; p++) s -= c->a0[p] * z[c->col[p]];
    z[i] = s * (1.0 / c->val[c->diagpos[i]]);
  }
  for (int64_t i = n - 1; i >= 0; i--) {
    double s = 0.0;
    for (int64_t p = c->diagpos[i] + 1; p < c->rowptr[i + 1]; p++) s += c->a0[p] * z[c->col[p]];
    z[i] -= (1.0 / c->val[c->diagpos[i]]) * s;
  }
  return;
#endif
  for (int64_t i = 0; i < n; i++) {
    double s = r[i];
    for (int64_t p = c->rowptr[i]; p < c->diagpos[i]; p++) s -= c->val[p] * z[c->col[p]];
    z[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; i--) {
    double s = z[i];
    for (int64_t p = c->diagpos[i] + 1; p < c->rowptr[i + 1]; p++) s -= c->val[p] * z[c->col[p]];
    z[i] = s / c->val[c->diagpos[i]];
  }
}

/* Slab partition along r (S:392 leading-remainder rule, A11/§8(c)-6):
 * block b gets nr/B + (b < nr%B) shells. */
static void slab_bounds(int nr, int nblocks, int b, int *i0, int *i1) {
  int base = nr / nblocks, rem = nr % nblocks;
  *i0 = b * base + (b < rem ? b : rem);
  *i1 = *i0 + base + (b < rem ? 1 : 0);
}

typedef struct {
  int pc, nblocks, nr, nt, np;
  double *inv_diag;      /* PC1, PC3 */
  int poly_m;            /* PC3: Chebyshev steps (the degree of the residual polynomial) */
  double poly_a, poly_b; /* PC3: eigenvalue interval of D^-1 A the polynomial targets */
  const double *wrap;    /* PC3: the operator's periodic couplings (set by the caller) */
  orc_csr *blocks;       /* PC2 */
  double *rb, *zb;       /* PC2 scratch */
} orc_pc;

/* ------------------------------------------------------------------------ */
/* PC3 (the "vector-friendly" preconditioner the paper    */
/* calls for; not in the paper): Chebyshev acceleration of Jacobi,    */
/* Saad, Iterative Methods 2nd ed., Alg. 12.1, applied to A z = r from       */
/* z_0 = 0 with the preconditioned residual D^-1 r, m steps:                 */
/*   theta = (b+a)/2, delta = (b-a)/2, sigma1 = theta/delta, rho0 = 1/sigma1 */
/*   res_0 = D^-1 r;  d_0 = res_0 / theta;  z_1 = d_0                        */
/*   k = 1..m-1: res_k = res_{k-1} - D^-1 A d_{k-1}                          */
/*               rho_k = 1 / (2 sigma1 - rho_{k-1})                          */
/*               d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) res_k     */
/*               z_{k+1} = z_k + d_k                                         */
/* so z_m = (I - R_m(D^-1 A)) A^-1 r with R_m(t) = T_m((b+a-2t)/(b-a)) /     */
/* T_m((b+a)/(b-a)): a fixed SPD operator when the spectrum of D^-1 A lies   */
/* in (0, b].  b = 2 bounds it (Gershgorin: A is diagonally dominant).       */
/* ------------------------------------------------------------------------ */
typedef void (*orc_linop)(void *ctx, const double *x, double *y);

void orc_cheb_apply(int64_t N, orc_linop A, void *actx, const double *inv_d, int m, double a,
                    double b, const double *r, double *z) {
  double *res = malloc(sizeof(double) * N), *d = malloc(sizeof(double) * N);
  double *q = malloc(sizeof(double) * N);
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma1 = theta / delta;
  double rho = 1.0 / sigma1;
  for (int64_t i = 0; i < N; i++) {
    res[i] = inv_d[i] * r[i];
    d[i] = res[i] / theta;
    z[i] = d[i];
  }
  for (int k = 1; k < m; k++) {
    A(actx, d, q);
    const double rho_new = 1.0 / (2.0 * sigma1 - rho);
    const double c1 = rho_new * rho, c2 = 2.0 * rho_new / delta;
    for (int64_t i = 0; i < N; i++) {
      res[i] -= inv_d[i] * q[i];
      d[i] = c1 * d[i] + c2 * res[i];
      z[i] += d[i];
    }
    rho = rho_new;
  }
  free(res); free(d); free(q);
}

typedef struct { int nr, nt, np; const double *bands, *wrap; } orc_sys;
static void sys_apply(void *ctx, const double *x, double *y) {
  const orc_sys *S = (const orc_sys *)ctx;
  orc_apply(S->nr, S->nt, S->np, S->bands, S->wrap, x, y);
}

/* PC3 parameters (degree m, interval ratio b/a); orc_set_poly changes them for
 * the following builds of the preconditioner. */
static int g_poly_m = 4;
static double g_poly_ratio = 100.0;
void orc_set_poly(int m, double ratio) {
  g_poly_m = m;
  g_poly_ratio = ratio;
}

/* PC1: inverse of the diagonal of A. */
static void pc_apply(const orc_pc *M, const double *bands, const double *r, double *z) {
  const int64_t N = (int64_t)M->nr * M->nt * M->np;
  if (M->pc == 3) {
    orc_sys op = {M->nr, M->nt, M->np, bands, M->wrap};
    orc_cheb_apply(N, sys_apply, &op, M->inv_diag, M->poly_m, M->poly_a, M->poly_b, r, z);
    return;
  }
  if (M->pc == 1) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < N; m++) z[m] = M->inv_diag[m] * r[m];
    return;
  }
  /* PC2: each block solved independently, no communication. */
  for (int b = 0; b < M->nblocks; b++) {
    int i0, i1;
    slab_bounds(M->nr, M->nblocks, b, &i0, &i1);
    int nb = i1 - i0;
    for (int k = 0; k < M->np; k++)
      for (int j = 0; j < M->nt; j++)
        for (int il = 0; il < nb; il++)
          M->rb[il + (int64_t)nb * (j + (int64_t)M->nt * k)] =
              r[i0 + il + (int64_t)M->nr * (j + (int64_t)M->nt * k)];
    lusolve(&M->blocks[b], M->rb, M->zb);
    for (int k = 0; k < M->np; k++)
      for (int j = 0; j < M->nt; j++)
        for (int il = 0; il < nb; il++)
          z[i0 + il + (int64_t)M->nr * (j + (int64_t)M->nt * k)] =
              M->zb[il + (int64_t)nb * (j + (int64_t)M->nt * k)];
  }
}

static int pc_build(orc_pc *M, int pc, int nblocks, int nr, int nt, int np, const double *bands) {
  const int64_t N = (int64_t)nr * nt * np;
  memset(M, 0, sizeof(*M));
  M->pc = pc; M->nblocks = nblocks < 1 ? 1 : nblocks; M->nr = nr; M->nt = nt; M->np = np;
  if (pc == 3) {
    if (g_poly_m < 1 || !(g_poly_ratio > 1.0)) return -1;
    M->poly_m = g_poly_m;
    M->poly_b = 2.0;
    M->poly_a = 2.0 / g_poly_ratio;
  }
  if (pc == 1 || pc == 3) {
    M->inv_diag = malloc(sizeof(double) * N);
    for (int64_t m = 0; m < N; m++) {
      if (bands[3 * N + m] == 0.0) return -1;
      M->inv_diag[m] = 1.0 / bands[3 * N + m];
    }
    return 0;
  }
  if (M->nblocks > nr) return -1;
  M->blocks = calloc(M->nblocks, sizeof(orc_csr));
  int64_t maxn = 0;
  for (int b = 0; b < M->nblocks; b++) {
    int i0, i1;
    slab_bounds(nr, M->nblocks, b, &i0, &i1);
    block_csr(nr, nt, np, bands, i0, i1, &M->blocks[b]);
#ifdef ORC_ILU_DFORM
    {
      const int64_t nnz = M->blocks[b].rowptr[M->blocks[b].n];
      M->blocks[b].a0 = malloc(sizeof(double) * nnz);
      memcpy(M->blocks[b].a0, M->blocks[b].val, sizeof(double) * nnz);
    }
#endif
    if (ilu0_ikj(&M->blocks[b])) return -2;
    if (M->blocks[b].n > maxn) maxn = M->blocks[b].n;
  }
  M->rb = malloc(sizeof(double) * maxn);
  M->zb = malloc(sizeof(double) * maxn);
  return 0;
}

static void pc_free(orc_pc *M) {
  free(M->inv_diag);
  if (M->blocks) { for (int b = 0; b < M->nblocks; b++) csr_free(&M->blocks[b]); free(M->blocks); }
  free(M->rb); free(M->zb);
}

/* Wall time of the last orc_solve PCG loop (instrumentation for the timed
 * cpu_baseline; not part of the method). */
static double g_loop_seconds = 0.0;
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* Plain sequential inner product in index order. */
static double dot(int64_t n, const double *x, const double *y) {
  double s = 0.0;
#ifdef ORC_DOT_REVERSE
  /* an equally valid summation order (tools/oracle_spread.py only): measures how
   * far the iteration count at rtol moves under a rounding-order change alone */
  for (int64_t m = n - 1; m >= 0; m--) s += x[m] * y[m];
#else
  for (int64_t m = 0; m < n; m++) s += x[m] * y[m];
#endif
  return s;
}

/* ------------------------------------------------------------------------ */
/* PCG on an abstract SPD operator (A9).  A and M^-1 are */
/* callbacks y = op(ctx, x), so the same loop runs the POT3D system         */
/* (orc_solve) and the SPEC worked examples / random SPD matrices    */
/* in the tests.                                                     */
/*                                                                           */
/* variant ORC_PCG_STANDARD (0) -- the standard two-reduction PCG:   */
/*   x0 = 0, r = b, z = M^-1 r, p = z, rho = r.z                             */
/*   loop: q = A p; sigma = p.q (<=0 -> indefinite); alpha = rho/sigma;      */
/*         x += alpha p; r -= alpha q; k++;                                  */
/*         stop if ||r|| <= rtol ||b|| or k == maxit;                        */
/*         z = M^-1 r; rho' = r.z; p = z + (rho'/rho) p; rho = rho'.         */
/*                                                                           */
/* variant ORC_PCG_CG1 (1) -- single-reduction PCG of Chronopoulos & Gear    */
/* (1989), in the form of Ghysels & Vanroose (2014) Alg. 2.       */
/* §8(f)-1: the paper names the inner products' "collective/synchronous     */
/* nature" as the scaling limiter; this variant gathers the    */
/* three inner products of an iteration into one reduction.  Not in the      */
/* paper, so it follows the cited algorithm step by step:                    */
/*   x0 = 0, r = b, u = M^-1 r, w = A u,                                     */
/*   gamma = r.u, delta = w.u (<=0 -> indefinite), alpha = gamma/delta,      */
/*   beta = 0;                                                               */
/*   loop: p = u + beta p; s = w + beta s;  (k = 0: p = u, s = w)            */
/*         x += alpha p; r -= alpha s; k++;                                  */
/*         u = M^-1 r; w = A u; gamma' = r.u; delta = w.u; rr = r.r          */
/*           (ONE reduction of three inner products);                        */
/*         stop if sqrt(rr) <= rtol ||b|| or k == maxit;                     */
/*         beta = gamma'/gamma; den = delta - beta gamma'/alpha              */
/*           (= p.Ap in exact arithmetic; <=0 -> indefinite);                */
/*         alpha = gamma'/den; gamma = gamma'.                               */
/* In exact arithmetic both variants produce the same iterates.              */
/*                                                                           */
/* Flag ORC_PCG_X0 (or-ed into variant) -- warm start, the "repeated solves" */
/* of SURVEY.md §8(f)-3 (MAS repeats equivalent PCG solves; DESIGN.md  */
/* reading A28): x holds x0 on entry and the loop starts from r = b - A x0   */
/* instead of x0 = 0, r = b; everything after that line is unchanged (the    */
/* stopping test stays ||r|| <= rtol ||b||).  If x0 already meets it the     */
/* solve stops with iters = 0; b = 0 still returns x = 0.            */
/*                                                                           */
/* status: 0 converged, 1 maxit reached, -4 indefinite.                      */
/* hist (nullable, maxit+1 doubles): ||r_k||/||b|| for k = 0..iters.          */
/* ------------------------------------------------------------------------ */
#define ORC_PCG_STANDARD 0
#define ORC_PCG_CG1 1
#define ORC_PCG_X0 16

int orc_pcg(int64_t N, orc_linop A, void *actx, orc_linop Minv, void *mctx, const double *b,
            double rtol, int64_t maxit, int variant, double *x, int64_t *iters,
            double *rel_res, double *hist) {
  const int warm = (variant & ORC_PCG_X0) != 0;
  variant &= ~ORC_PCG_X0;
  double *r = malloc(sizeof(double) * N);
  double *z = malloc(sizeof(double) * N);  /* z (standard) / u (CG1) */
  double *p = malloc(sizeof(double) * N);
  double *q = malloc(sizeof(double) * N);  /* q = A p (standard) / w = A u (CG1) */
  double *s = variant == ORC_PCG_CG1 ? malloc(sizeof(double) * N) : NULL;
  int status = 0, conv = 0;
  if (warm) {                        /* r = b - A x0 */
    A(actx, x, r);
    for (int64_t m = 0; m < N; m++) r[m] = b[m] - r[m];
  } else {
    for (int64_t m = 0; m < N; m++) { x[m] = 0.0; r[m] = b[m]; }
  }
  const double bnorm = sqrt(dot(N, b, b));
  int64_t k = 0;
  double rnorm = warm ? sqrt(dot(N, r, r)) : bnorm;
  if (hist) hist[0] = bnorm > 0 ? rnorm / bnorm : 0.0;
  if (bnorm == 0.0) { /* b = 0 -> Phi = 0 */
    for (int64_t m = 0; m < N; m++) x[m] = 0.0;
    *iters = 0; *rel_res = 0.0;
    goto done;
  }
  if (warm && rnorm <= rtol * bnorm) { /* x0 already meets the test */
    *iters = 0; *rel_res = rnorm / bnorm;
    goto done;
  }
  const double t_loop = now_s();
  if (variant == ORC_PCG_STANDARD) {
    Minv(mctx, r, z);
    for (int64_t m = 0; m < N; m++) p[m] = z[m];
    double rho = dot(N, r, z);
    while (1) {
      A(actx, p, q);
      double sigma = dot(N, p, q);
      if (!(sigma > 0.0)) { status = -4; break; }
      double alpha = rho / sigma;
#pragma omp parallel for schedule(static)
      for (int64_t m = 0; m < N; m++) { x[m] += alpha * p[m]; r[m] -= alpha * q[m]; }
      k++;
      rnorm = sqrt(dot(N, r, r));
      if (hist) hist[k] = rnorm / bnorm;
      if (rnorm <= rtol * bnorm) { conv = 1; break; }
      if (k >= maxit) break;
      Minv(mctx, r, z);
      double rho_new = dot(N, r, z);
      double beta = rho_new / rho;
#pragma omp parallel for schedule(static)
      for (int64_t m = 0; m < N; m++) p[m] = z[m] + beta * p[m];
      rho = rho_new;
    }
  } else {
    Minv(mctx, r, z);          /* u */
    A(actx, z, q);             /* w = A u */
    double gamma = dot(N, r, z), delta = dot(N, q, z);
    if (!(delta > 0.0)) { status = -4; goto stop; }
    double alpha = gamma / delta, beta = 0.0;
    while (1) {
#pragma omp parallel for schedule(static)
      for (int64_t m = 0; m < N; m++) {
        p[m] = (k == 0) ? z[m] : z[m] + beta * p[m];
        s[m] = (k == 0) ? q[m] : q[m] + beta * s[m];
        x[m] += alpha * p[m];
        r[m] -= alpha * s[m];
      }
      k++;
      Minv(mctx, r, z);
      A(actx, z, q);
      double gamma_new = dot(N, r, z);
      delta = dot(N, q, z);
      rnorm = sqrt(dot(N, r, r));
      if (hist) hist[k] = rnorm / bnorm;
      if (rnorm <= rtol * bnorm) { conv = 1; break; }
      if (k >= maxit) break;
      beta = gamma_new / gamma;
      double den = delta - beta * gamma_new / alpha;
      if (!(den > 0.0)) { status = -4; break; }
      alpha = gamma_new / den;
      gamma = gamma_new;
    }
  }
stop:
  g_loop_seconds = now_s() - t_loop;
  if (status == 0 && !conv) status = 1;
  *iters = k;
  *rel_res = rnorm / bnorm;
done:
  free(r); free(z); free(p); free(q); free(s);
  return status;
}

/* The POT3D preconditioners as orc_pcg callbacks. */
typedef struct { const orc_pc *M; const double *bands; } orc_pcctx;
static void pc_cb(void *ctx, const double *r, double *z) {
  const orc_pcctx *C = (const orc_pcctx *)ctx;
  pc_apply(C->M, C->bands, r, z);
}

/* ------------------------------------------------------------------------ */
/* The POT3D solve: assemble A (DIA), b (Eq.2),       */
/* build PC1/PC2, run orc_pcg, closed-wall gauge (A8).         */
/* status: 0 converged, 1 maxit reached, 2 PC2 fell back to PC1 (converged  */
/* or not), -1 bad input, -4 indefinite.                                     */
/* ------------------------------------------------------------------------ */
int orc_solve_v(int nr, int nt, int np, const double *rf, const double *tf,
                const double *pf, int bc, int pc, int pc2_blocks, const double *br0,
                double rtol, int64_t maxit, int variant, double *x, int64_t *iters,
                double *rel_res, double *true_rel_res, double *hist) {
  const int64_t N = (int64_t)nr * nt * np;
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return -1;
  double *bands = malloc(sizeof(double) * 7 * N);
  double *wrap = malloc(sizeof(double) * 2 * nr * nt);
  double *b = malloc(sizeof(double) * N);
  int status = 0, fell_back = 0;
  orc_assemble(nr, nt, np, rf, tf, pf, bc, bands, wrap);
  orc_rhs(nr, nt, np, rf, tf, pf, bc, br0, b, NULL);
  orc_pc M;
  int prc = pc_build(&M, pc, pc2_blocks, nr, nt, np, bands);
  M.wrap = wrap;
  if (prc == -2) { /* ILU breakdown: fall back to PC1 */
    pc_free(&M);
    pc_build(&M, 1, 1, nr, nt, np, bands);
    fell_back = 1;
  } else if (prc) { status = -1; goto done; }
  orc_sys sys = {nr, nt, np, bands, wrap};
  orc_pcctx pcc = {&M, bands};
  status = orc_pcg(N, sys_apply, &sys, pc_cb, &pcc, b, rtol, maxit, variant, x, iters, rel_res,
                   hist);
  if (status == 0 && fell_back) status = 2;
  const double bnorm = sqrt(dot(N, b, b));
  if (bnorm == 0.0) { if (true_rel_res) *true_rel_res = 0.0; goto done; }
  if (bc == ORC_CLOSED_WALL) {
    double sv = 0.0, svx = 0.0;
    for (int kk = 0; kk < np; kk++)
      for (int j = 0; j < nt; j++)
        for (int i = 0; i < nr; i++) {
          double V = cell_volume(&g, i, j, kk);
          sv += V; svx += V * x[i + (int64_t)nr * (j + (int64_t)nt * kk)];
        }
    double mean = svx / sv;
    for (int64_t m = 0; m < N; m++) x[m] -= mean;
  }
  if (true_rel_res) {
    double *q = malloc(sizeof(double) * N);
    orc_apply(nr, nt, np, bands, wrap, x, q);
    for (int64_t m = 0; m < N; m++) q[m] = b[m] - q[m];
    *true_rel_res = sqrt(dot(N, q, q)) / bnorm;
    free(q);
  }
done:
  pc_free(&M);
  free(bands); free(wrap); free(b);
  mesh_free(&g);
  return status;
}

int orc_solve(int nr, int nt, int np, const double *rf, const double *tf,
              const double *pf, int bc, int pc, int pc2_blocks, const double *br0,
              double rtol, int64_t maxit, double *x, int64_t *iters,
              double *rel_res, double *true_rel_res, double *hist) {
  return orc_solve_v(nr, nt, np, rf, tf, pf, bc, pc, pc2_blocks, br0, rtol, maxit,
                     ORC_PCG_STANDARD, x, iters, rel_res, true_rel_res, hist);
}

/* Slab partition exported for the tests. */
void orc_slab_bounds(int nr, int nblocks, int b, int *i0, int *i1) {
  slab_bounds(nr, nblocks, b, i0, i1);
}

/* Preconditioner apply on its own (for tests): z = M^-1 r. */
int orc_precond(int nr, int nt, int np, const double *rf, const double *tf,
                const double *pf, int bc, int pc, int pc2_blocks, const double *r, double *z) {
  const int64_t N = (int64_t)nr * nt * np;
  double *bands = malloc(sizeof(double) * 7 * N);
  double *wrap = malloc(sizeof(double) * 2 * nr * nt);
  orc_assemble(nr, nt, np, rf, tf, pf, bc, bands, wrap);
  orc_pc M;
  int rc = pc_build(&M, pc, pc2_blocks, nr, nt, np, bands);
  M.wrap = wrap;
  if (rc == 0) pc_apply(&M, bands, r, z);
  pc_free(&M);
  free(bands); free(wrap);
  return rc;
}

/* ILU0 of one block, exported for the defining-property test:
 * fills CSR arrays (rowptr n+1, col/val up to 7n, A values in aval). */
int orc_block_ilu0(int nr, int nt, int np, const double *rf, const double *tf,
                   const double *pf, int bc, int i0, int i1, int64_t *rowptr,
                   int64_t *col, double *aval, double *luval) {
  const int64_t N = (int64_t)nr * nt * np;
  double *bands = malloc(sizeof(double) * 7 * N);
  double *wrap = malloc(sizeof(double) * 2 * nr * nt);
  orc_assemble(nr, nt, np, rf, tf, pf, bc, bands, wrap);
  orc_csr c;
  block_csr(nr, nt, np, bands, i0, i1, &c);
  memcpy(rowptr, c.rowptr, sizeof(int64_t) * (c.n + 1));
  memcpy(col, c.col, sizeof(int64_t) * c.rowptr[c.n]);
  memcpy(aval, c.val, sizeof(double) * c.rowptr[c.n]);
  int rc = ilu0_ikj(&c);
  memcpy(luval, c.val, sizeof(double) * c.rowptr[c.n]);
  csr_free(&c);
  free(bands); free(wrap);
  return rc;
}

/* Generic ILU0 on a caller CSR matrix (for the SPEC worked examples). */
int orc_ilu0_csr(int64_t n, const int64_t *rowptr, const int64_t *col, double *val) {
  orc_csr c;
  c.n = n;
  c.rowptr = (int64_t *)rowptr; c.col = (int64_t *)col; c.val = val;
  c.a0 = NULL;
  c.diagpos = malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; i++) {
    c.diagpos[i] = -1;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; p++) if (col[p] == i) c.diagpos[i] = p;
    if (c.diagpos[i] < 0) { free(c.diagpos); return -1; }
  }
  int rc = ilu0_ikj(&c);
  free(c.diagpos);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Polar ring average, Eq.3: Phi_pole(i) = (1/2pi) sum_k dphi_k   */
/* Phi(i, j_adj, k), the ring at eps = half a cell from the pole.*/
/* ------------------------------------------------------------------------ */
void orc_polar_average(int nr, int nt, int np, const double *pf, const double *x,
                       int south, double *avg) {
  double period = pf[np] - pf[0];
  int j = south ? nt - 1 : 0;
  for (int i = 0; i < nr; i++) {
    double s = 0.0;
    for (int k = 0; k < np; k++) s += (pf[k + 1] - pf[k]) * x[i + (int64_t)nr * (j + (int64_t)nt * k)];
    avg[i] = s / period;
  }
}

/* ------------------------------------------------------------------------ */
/* Field B = grad Phi on staggered faces (A16), from the ghost  */
/* fill with vmask = 1 (A6):                                      */
/*   Br : (nr+1) x nt x np  at r faces,   index ir + (nr+1)(j + nt k)        */
/*   Bt : nr x (nt+1) x np  at t faces,   index i + nr(jf + (nt+1) k)        */
/*   Bp : nr x nt x np      at p faces k+1/2 (periodic), index i + nr(j+nt k)*/
/* br0 is the (solvability-adjusted for the closed wall) boundary map.       */
/* ------------------------------------------------------------------------ */
int orc_field(int nr, int nt, int np, const double *rf, const double *tf,
              const double *pf, int bc, const double *br0, const double *x,
              double *br, double *bt, double *bp) {
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return -1;
  double *br_adj = malloc(sizeof(double) * nt * np);
  memcpy(br_adj, br0, sizeof(double) * nt * np);
  if (bc == ORC_CLOSED_WALL) enforce_solvability(&g, br_adj);
  double *poleN = malloc(sizeof(double) * nr), *poleS = malloc(sizeof(double) * nr);
  orc_polar_average(nr, nt, np, pf, x, 0, poleN);
  orc_polar_average(nr, nt, np, pf, x, 1, poleS);
#define X(i, j, k) x[(i) + (int64_t)nr * ((j) + (int64_t)nt * (k))]
  for (int k = 0; k < np; k++)
    for (int j = 0; j < nt; j++) {
      /* r faces.  Ghost at r0: x(1)=x(2)-br0*dr1 (vmask=1); at r1: -x for the
       * source surface (Phi=0), +x for the closed wall (Br=0) (A7). */
      double ghost_in = X(0, j, k) - br_adj[j + (int64_t)nt * k] * g.dr[0];
      double ghost_out = (bc == ORC_SOURCE_SURFACE) ? -X(nr - 1, j, k) : X(nr - 1, j, k);
      for (int ir = 0; ir <= nr; ir++) {
        double v;
        if (ir == 0) v = (X(0, j, k) - ghost_in) / g.dr[0];
        else if (ir == nr) v = (ghost_out - X(nr - 1, j, k)) / g.dr[nr - 1];
        else v = (X(ir, j, k) - X(ir - 1, j, k)) / g.drh[ir - 1];
        br[ir + (int64_t)(nr + 1) * (j + (int64_t)nt * k)] = v;
      }
    }
  for (int k = 0; k < np; k++)
    for (int jf = 0; jf <= nt; jf++)
      for (int i = 0; i < nr; i++) {
        double v;
        /* theta faces; at the poles the ghost is the Eq.3 average placed on
         * the pole itself, eps = tc_0 - 0 away from the first ring. */
        if (jf == 0) v = (X(i, 0, k) - poleN[i]) / (g.rc[i] * (g.tc[0] - tf[0]));
        else if (jf == nt) v = (poleS[i] - X(i, nt - 1, k)) / (g.rc[i] * (tf[nt] - g.tc[nt - 1]));
        else v = (X(i, jf, k) - X(i, jf - 1, k)) / (g.rc[i] * g.dth[jf - 1]);
        bt[i + (int64_t)nr * (jf + (int64_t)(nt + 1) * k)] = v;
      }
  for (int k = 0; k < np; k++) {
    int kp = (k + 1) % np;
    for (int j = 0; j < nt; j++)
      for (int i = 0; i < nr; i++)
        bp[i + (int64_t)nr * (j + (int64_t)nt * k)] =
            (X(i, j, kp) - X(i, j, k)) / (g.rc[i] * g.st[j] * g.dph[k]);
  }
#undef X
  free(br_adj); free(poleN); free(poleS);
  mesh_free(&g);
  return 0;
}

/* Cell volumes (for the closed-wall gauge and the divergence identity test). */
int orc_volumes(int nr, int nt, int np, const double *rf, const double *tf,
                const double *pf, double *vol) {
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return -1;
  for (int k = 0; k < np; k++)
    for (int j = 0; j < nt; j++)
      for (int i = 0; i < nr; i++)
        vol[i + (int64_t)nr * (j + (int64_t)nt * k)] = cell_volume(&g, i, j, k);
  mesh_free(&g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Timing harness for bench.py's cpu_baseline / --impl reference legs (not   */
/* part of the method): the system (DIA bands, b, PC1/PC2) is assembled once */
/* per session, then every orc_session_solve runs the unchanged orc_pcg from */
/* x0 = 0 and reports the PCG loop's wall time.                              */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t N;
  double *bands, *wrap, *b;
  orc_pc M;
  orc_sys sys;
  orc_pcctx pcc;
} orc_session;

void *orc_session_create(int nr, int nt, int np, const double *rf, const double *tf,
                         const double *pf, int bc, int pc, int pc2_blocks, const double *br0) {
  orc_mesh g;
  if (mesh_build(&g, nr, nt, np, rf, tf, pf)) return NULL;
  mesh_free(&g);
  orc_session *S = calloc(1, sizeof(orc_session));
  S->N = (int64_t)nr * nt * np;
  S->bands = malloc(sizeof(double) * 7 * S->N);
  S->wrap = malloc(sizeof(double) * 2 * nr * nt);
  S->b = malloc(sizeof(double) * S->N);
  orc_assemble(nr, nt, np, rf, tf, pf, bc, S->bands, S->wrap);
  orc_rhs(nr, nt, np, rf, tf, pf, bc, br0, S->b, NULL);
  if (pc_build(&S->M, pc, pc2_blocks, nr, nt, np, S->bands)) {
    pc_free(&S->M);
    pc_build(&S->M, 1, 1, nr, nt, np, S->bands);
  }
  S->M.wrap = S->wrap;
  S->sys = (orc_sys){nr, nt, np, S->bands, S->wrap};
  S->pcc = (orc_pcctx){&S->M, S->bands};
  return S;
}

int orc_session_solve(void *sp, double rtol, int64_t maxit, int variant, double *x,
                      int64_t *iters, double *rel_res, double *loop_seconds) {
  orc_session *S = (orc_session *)sp;
  int st = orc_pcg(S->N, sys_apply, &S->sys, pc_cb, &S->pcc, S->b, rtol, maxit, variant, x, iters,
                   rel_res, NULL);
  if (loop_seconds) *loop_seconds = g_loop_seconds;
  return st;
}

void orc_session_free(void *sp) {
  orc_session *S = (orc_session *)sp;
  if (!S) return;
  pc_free(&S->M);
  free(S->bands); free(S->wrap); free(S->b);
  free(S);
}

/* Threads the element-wise loops use (reported as cpu_baseline.cores). */
int orc_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* A fixed number of PCG iterations on a prebuilt system, for the timed
 * cpu_baseline leg: identical arithmetic to orc_solve (it IS orc_solve with
 * maxit = iters and rtol = 0), exposed separately only to report time. */
int orc_solve_fixed(int nr, int nt, int np, const double *rf, const double *tf,
                    const double *pf, int bc, int pc, int pc2_blocks, const double *br0,
                    int64_t iters, double *x, double *rel_res, double *loop_seconds) {
  int64_t it = 0;
  int st = orc_solve(nr, nt, np, rf, tf, pf, bc, pc, pc2_blocks, br0, 0.0, iters, x, &it,
                     rel_res, NULL, NULL);
  if (loop_seconds) *loop_seconds = g_loop_seconds;
  return st;
}
