// kernels.cu -- sm_100a kernels of the fp64 PCG hot path.
//
//   k_metrics        a1  1-D metric factors from the faces (A1-A7)
//   k_rhs            a2  b on the photosphere shell (Eq.2)
//   k_pass_a         a3  p = z + beta p_old (z = D^-1 r on the fly, PC1 P:88),
//                        q = A p, partial p.q, lazy x += alpha_prev p_old
//   k_pass_b         a7  q = A p (recomputed), r -= alpha q, z = D^-1 r,
//                        partials r.z and r.r
//   k_init_dots      a10 rho_0 = b.D^-1 b, ||b||
//   finalize_*       a6/a10 deterministic second-level reduction, alpha, beta,
//                        convergence test, on the device
//   k_apply          unfused 7-point apply (diagnostics, true residual)
//   k_finish         a11 x += alpha_last p_last
//   k_field_*        a11 B = grad Phi on staggered faces (A16)
//   k_transpose      user layout (r fastest) <-> device layout (phi fastest)
//
// The two fused passes march along r through a theta x phi tile (2.5-D
// blocking): each thread owns two phi-adjacent cells
// (one 128-bit fp64 load per array), the current plane of p is staged in a
// 3-slot shared-memory ring for the theta/phi neighbours, the r neighbours
// stay in registers, and the next plane is prefetched into registers while
// the stencil of the current plane runs.
#include "pot3d_internal.cuh"

namespace pot3d {
#ifndef PASS_MINB
#define PASS_MINB 2
#endif

// ---------------------------------------------------------------------------
// a1: metric factors.  One thread per entry; faces are device arrays.
// ---------------------------------------------------------------------------
__global__ void k_metrics(int nr, int nt, int np, int bc, const double *rf, const double *tf,
                          const double *pf, double *arp, double *arm, double *dr, double *ss,
                          double *g, double *atp, double *atm, double *q, double *dp, double *app,
                          double *apm, double *rc, double *drh, double *tc, double *dth,
                          double *st, double *dph, double *vr) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  const double period = pf[np] - pf[0];
  if (t < nr) {
    int i = t;
    double rci = 0.5 * (rf[i] + rf[i + 1]);
    rc[i] = rci;
    dr[i] = rf[i + 1] - rf[i];
    vr[i] = rci * rci * (rf[i + 1] - rf[i]);  // r_i^2 dr_i (cell-volume factor, A3)
    if (i < nr - 1) {
      double rcn = 0.5 * (rf[i + 1] + rf[i + 2]);
      drh[i] = rcn - rci;
      arp[i] = rf[i + 1] * rf[i + 1] / (rcn - rci);
    } else {
      drh[i] = 0.0;
      arp[i] = 0.0;
    }
    if (i > 0) {
      double rcp = 0.5 * (rf[i - 1] + rf[i]);
      arm[i] = rf[i] * rf[i] / (rci - rcp);
    } else {
      arm[i] = 0.0;  // homogeneous Neumann at r0 (A6): Br0 lives in b
    }
    // source surface: odd ghost through Phi=0 on the r1 face (A7)
    ss[i] = (i == nr - 1 && bc == 0) ? 2.0 * rf[nr] * rf[nr] / (rf[nr] - rf[nr - 1]) : 0.0;
  }
  if (t < nt) {
    int j = t;
    double tcj = 0.5 * (tf[j] + tf[j + 1]);
    double dtj = tf[j + 1] - tf[j];
    double s = sin(tcj);
    tc[j] = tcj;
    st[j] = s;
    g[j] = s * dtj;
    q[j] = dtj / s;
    if (j < nt - 1) {
      double tcn = 0.5 * (tf[j + 1] + tf[j + 2]);
      dth[j] = tcn - tcj;
      atp[j] = sin(tf[j + 1]) / (tcn - tcj);
    } else {
      dth[j] = 0.0;
      atp[j] = 0.0;  // pole face: sin(pi) area = 0 (A5)
    }
    if (j > 0) {
      double tcp = 0.5 * (tf[j - 1] + tf[j]);
      atm[j] = sin(tf[j]) / (tcj - tcp);
    } else {
      atm[j] = 0.0;  // pole face: sin(0) = 0 (A5)
    }
  }
  if (t < np) {
    int k = t;
    double pck = 0.5 * (pf[k] + pf[k + 1]);
    dp[k] = pf[k + 1] - pf[k];
    double pcn = (k < np - 1) ? 0.5 * (pf[k + 1] + pf[k + 2]) : 0.5 * (pf[0] + pf[1]) + period;
    double pcp = (k > 0) ? 0.5 * (pf[k - 1] + pf[k]) : 0.5 * (pf[np - 1] + pf[np]) - period;
    dph[k] = pcn - pck;
    app[k] = 1.0 / (pcn - pck);
    apm[k] = 1.0 / (pck - pcp);
  }
}

// ---------------------------------------------------------------------------
// Deterministic reductions (a6).  Level 1: warp shuffle tree + fixed-order
// combine of the warps of a block.  Level 2: the last block to finish sums
// the per-block partials in index order (threads stride, then a fixed tree),
// so the result does not depend on which block finishes last.
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void warp_sum(double (&v)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int n = 0; n < N; n++) v[n] += __shfl_xor_sync(0xffffffffu, v[n], o);
}

// Reduces v over the block; the result is valid in thread 0.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double *sred) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  warp_sum<N>(v);
  __syncthreads();  // sred may still be read by a previous use
  if (lane == 0)
#pragma unroll
    for (int n = 0; n < N; n++) sred[w * N + n] = v[n];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int n = 0; n < N; n++) v[n] = (lane < nw) ? sred[lane * N + n] : 0.0;
    warp_sum<N>(v);
  }
}

// Writes this block's partial, and returns true in the (single) last block,
// where `tot` then holds the grid total in every thread 0.
template <int N>
__device__ bool grid_sum(double (&v)[N], double *partials, unsigned int *counter, double *sred,
                         double (&tot)[N]) {
  __shared__ bool s_last;
  const int nb = gridDim.x * gridDim.y;
  const int bid = blockIdx.x + gridDim.x * blockIdx.y;
  block_sum<N>(v, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < N; n++) partials[(size_t)n * nb + bid] = v[n];
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    s_last = (t == (unsigned)nb - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double a[N];
#pragma unroll
  for (int n = 0; n < N; n++) a[n] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
    for (int n = 0; n < N; n++) a[n] += __ldcg(partials + (size_t)n * nb + b);
  block_sum<N>(a, sred);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < N; n++) tot[n] = a[n];
    *counter = 0u;
  }
  return true;
}

// After pass A: alpha = rho / p.Ap; p.Ap <= 0 -> indefinite.
__device__ void finalize_alpha(Scalars *S, double sigma) {
  S->sigma = sigma;
  if (!(sigma > 0.0)) {
    S->status = -4;
    S->stop = 1;
    return;
  }
  S->alpha = S->rho / sigma;
}

// After pass B: iteration count, convergence test ||r|| <= rtol ||b|| on the
// recurrence residual (A9), beta = rho'/rho.
__device__ void finalize_beta(Scalars *S, double rz, double rr, double *hist) {
  long long it = S->iter + 1;
  S->iter = it;
  S->rr = rr;
  double rn = sqrt(rr);
  if (hist) hist[it] = rn / S->bnorm;
  S->alpha_prev = S->alpha;
  if (rn <= S->rtol * S->bnorm) {
    S->stop = 1;
    S->status = 0;
    return;
  }
  if (it >= S->maxit) {
    S->stop = 1;
    S->status = 1;
    return;
  }
  S->beta = rz / S->rho;
  S->rho = rz;
}

// PC2 split of finalize_beta: ||r|| test after pass B, rho/beta after the sweeps.
__device__ void finalize_rr(Scalars *S, double rr, double *hist) {
  long long it = S->iter + 1;
  S->iter = it;
  S->rr = rr;
  double rn = sqrt(rr);
  if (hist) hist[it] = rn / S->bnorm;
  S->alpha_prev = S->alpha;
  if (rn <= S->rtol * S->bnorm) {
    S->stop = 1;
    S->status = 0;
  } else if (it >= S->maxit) {
    S->stop = 1;
    S->status = 1;
  }
}
__device__ void finalize_rho(Scalars *S, double rz) {
  S->beta = rz / S->rho;
  S->rho = rz;
}
// ---------------------------------------------------------------------------
// Per-cell helpers.
// ---------------------------------------------------------------------------
struct RowC {  // theta factors of one row
  double g, atp, atm, q;
};
struct PlaneC {  // r factors of one shell
  double arp, arm, dr, ss;
};

__device__ __forceinline__ RowC row_c(const Metrics &M, int j) {
  RowC c;
  c.g = __ldg(M.g + j);
  c.atp = __ldg(M.atp + j);
  c.atm = __ldg(M.atm + j);
  c.q = __ldg(M.q + j);
  return c;
}
__device__ __forceinline__ PlaneC plane_c(const Metrics &M, int ig) {
  PlaneC c;
  c.arp = __ldg(M.arp + ig);
  c.arm = __ldg(M.arm + ig);
  c.dr = __ldg(M.dr + ig);
  c.ss = __ldg(M.ss + ig);
  return c;
}
// diag(A) = dp_k [g_j (arp_i + arm_i + ss_i) + dr_i (atp_j + atm_j)] + dr_i q_j (app_k + apm_k)
struct DiagRow {  // diag = dp_k * a + b * sk
  double a, b;
};
__device__ __forceinline__ DiagRow diag_row(const PlaneC &P, const RowC &R) {
  DiagRow d;
  d.a = R.g * (P.arp + P.arm + P.ss) + P.dr * (R.atp + R.atm);
  d.b = P.dr * R.q;
  return d;
}

// ---------------------------------------------------------------------------
// Fused pass kernels.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void chunk_bounds(const Grid &G, int c, int &c0, int &c1) {
  int base = G.nr_loc / G.nchunks, rem = G.nr_loc % G.nchunks;
  c0 = c * base + (c < rem ? c : rem);
  c1 = c0 + base + (c < rem ? 1 : 0);
}

// Loaded data of one plane for one thread (own item + halo duties).
struct LoadA {
  double2 r, p, x;     // own item
  double2 hr, hp;      // halo row item (warps 0 / TJ-1)
  double cr, cp;       // halo column (lanes 0 / 31)
};

template <bool PASS_A, bool USE_Z>
__device__ __forceinline__ void pass_body(const PassArgs &A) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  if (S->stop) return;

  __shared__ __align__(16) double sm[3][SROWS][SROW];
  __shared__ double sred[(NTHREADS / 32) * 2];

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int tj = tile % G.ntj, tk = tile / G.ntj;
  const int j0 = tj * TJ, k0 = tk * TK;
  int c0, c1;
  chunk_bounds(G, blockIdx.y, c0, c1);

  const int j = j0 + w;                 // own row
  const bool jv = j < G.nt;
  const int k = k0 + 2 * lane;          // own columns k, k+1
  const bool kv0 = k < G.np, kv1 = (k + 1) < G.np;
  const bool lv = jv && kv0;            // own item loads/stores
  // halo duties
  const int hrow = (w == 0) ? j0 - 1 : ((w == TJ - 1) ? j0 + TJ : -2);  // -2: none
  const bool hv = (hrow >= 0) && (hrow < G.nt) && (w == 0 || w == TJ - 1);
  const int hslot = (w == 0) ? 0 : TJ + 1;
  // halo columns: lane 0 -> left neighbour of k0, lane 31 -> right neighbour of the last column
  const int kend = min(k0 + TK, G.np);
  const int hcol = (lane == 0) ? (k0 == 0 ? G.np - 1 : k0 - 1) : (kend == G.np ? 0 : kend);
  const int hs = (lane == 0) ? 1 : (kend - k0 + 2);
  const bool cv = jv && (lane == 0 || lane == 31);

  // per-column and per-row constant factors
  const int ka = min(k, G.np - 1), kb = min(k + 1, G.np - 1);
  const double dp0 = __ldg(M.dp + ka), dp1 = __ldg(M.dp + kb);
  const double app0 = __ldg(M.app + ka), app1 = __ldg(M.app + kb);
  const double apm0 = __ldg(M.apm + ka), apm1 = __ldg(M.apm + kb);
  const double sk0 = app0 + apm0, sk1 = app1 + apm1;
  const RowC rw = row_c(M, jv ? j : 0);
  const double beta = PASS_A ? S->beta : 0.0;
  const double alpha_prev = PASS_A ? S->alpha_prev : 0.0;
  const double alpha = PASS_A ? 0.0 : S->alpha;

  const double *src_r = PASS_A ? (USE_Z ? A.z : A.r) : nullptr;

  // ---- load one plane (il in [c0-1, c1]) into registers ----
  // PASS_A: own item r/z, p_old, x (x only for owned planes); halo row r/z, p_old; halo col r/z, p_old.
  //         On ghost planes (il < 0 or il >= nr_loc) p_new is final (halo exchange): load p_new.
  // PASS_B: own item p_new, plus r of plane il-1 (consumed by the stencil of il-1);
  //         halo row / col p_new.
  auto load = [&](int il, LoadA &L) {
    const bool ghost = (il < 0) || (il >= G.nr_loc);
    const long long rowbase = cidx(G, il, jv ? j : 0, 0);
    const double2 Z2 = make_double2(0.0, 0.0);
    if (PASS_A) {
      if (ghost) {
        L.r = lv ? *reinterpret_cast<const double2 *>(A.p_new + rowbase + k) : Z2;
        L.p = Z2;
      } else {
        L.r = lv ? __ldcs(reinterpret_cast<const double2 *>(src_r + rowbase + k)) : Z2;
        L.p = lv ? __ldcs(reinterpret_cast<const double2 *>(A.p_old + rowbase + k)) : Z2;
      }
      const bool own = (il >= c0) && (il < c1);
      L.x = (lv && own) ? __ldcs(reinterpret_cast<const double2 *>(A.x + rowbase + k)) : Z2;
      if (hv) {
        const long long hb = cidx(G, il, hrow, 0);
        if (ghost) {
          L.hr = kv0 ? *reinterpret_cast<const double2 *>(A.p_new + hb + k) : Z2;
          L.hp = Z2;
        } else {
          L.hr = kv0 ? *reinterpret_cast<const double2 *>(src_r + hb + k) : Z2;
          L.hp = kv0 ? *reinterpret_cast<const double2 *>(A.p_old + hb + k) : Z2;
        }
      }
      if (cv) {
        const long long cb = rowbase + hcol;
        if (ghost) {
          L.cr = A.p_new[cb];
          L.cp = 0.0;
        } else {
          L.cr = src_r[cb];
          L.cp = A.p_old[cb];
        }
      }
    } else {
      L.p = lv ? *reinterpret_cast<const double2 *>(A.p_new + rowbase + k) : Z2;
      const int ir = il - 1;
      const bool own = (ir >= c0) && (ir < c1);
      L.r = (lv && own) ? __ldcs(reinterpret_cast<const double2 *>(A.r + cidx(G, ir, j, k))) : Z2;
      if (hv) L.hp = kv0 ? *reinterpret_cast<const double2 *>(A.p_new + cidx(G, il, hrow, k)) : Z2;
      if (cv) L.cp = A.p_new[rowbase + hcol];
    }
  };

  // ---- transform a loaded plane: p_new values to registers (own) and smem ----
  // The own item is written to smem first; after __syncwarp the halo column
  // may overwrite the padding slot that follows the last phi column (the
  // periodic wrap neighbour lives there on the last tile).
  auto transform = [&](int il, const LoadA &L, double2 &pn, int slot, bool to_smem) {
    const bool ghost = (il < 0) || (il >= G.nr_loc);
    const double2 Z2 = make_double2(0.0, 0.0);
    double2 h = Z2;  // halo-row value
    double cvv = 0.0; // halo-column value
    if (PASS_A) {
      if (ghost) {
        pn = L.r;  // loaded p_new (already final on ghost shells)
        h = L.hr;
        cvv = L.cr;
      } else {
        const PlaneC pc = plane_c(M, G.i0 + il);
        if (lv) {
          if (USE_Z) {
            pn.x = L.r.x + beta * L.p.x;
            pn.y = L.r.y + beta * L.p.y;
          } else {
            const DiagRow d = diag_row(pc, rw);
            pn.x = L.r.x / (dp0 * d.a + d.b * sk0) + beta * L.p.x;
            pn.y = L.r.y / (dp1 * d.a + d.b * sk1) + beta * L.p.y;
          }
          if (!kv1) pn.y = 0.0;
        } else {
          pn = Z2;
        }
        const bool own = (il >= c0) && (il < c1);
        if (own && lv) {
          const long long o = cidx(G, il, j, k);
          if (kv1) {
            *reinterpret_cast<double2 *>(A.p_new + o) = pn;
            double2 xv = L.x;
            xv.x += alpha_prev * L.p.x;
            xv.y += alpha_prev * L.p.y;
            __stcs(reinterpret_cast<double2 *>(A.x + o), xv);
          } else {
            A.p_new[o] = pn.x;
            A.x[o] = L.x.x + alpha_prev * L.p.x;
          }
        }
        if (to_smem) {
          if (hv && kv0) {
            const RowC hrw = row_c(M, hrow);
            if (USE_Z) {
              h.x = L.hr.x + beta * L.hp.x;
              h.y = L.hr.y + beta * L.hp.y;
            } else {
              const DiagRow d = diag_row(pc, hrw);
              h.x = L.hr.x / (dp0 * d.a + d.b * sk0) + beta * L.hp.x;
              h.y = L.hr.y / (dp1 * d.a + d.b * sk1) + beta * L.hp.y;
            }
            if (!kv1) h.y = 0.0;
          }
          if (cv) {
            if (USE_Z) {
              cvv = L.cr + beta * L.cp;
            } else {
              const DiagRow d = diag_row(pc, rw);
              const double dpc = __ldg(M.dp + hcol);
              const double skc = __ldg(M.app + hcol) + __ldg(M.apm + hcol);
              cvv = L.cr / (dpc * d.a + d.b * skc) + beta * L.cp;
            }
          }
        }
      }
    } else {
      pn = L.p;
      h = L.hp;
      cvv = L.cp;
    }
    if (to_smem) {
      *reinterpret_cast<double2 *>(&sm[slot][w + 1][2 + 2 * lane]) = pn;
      // halo rows: neighbours above/below the tile; rows outside the grid
      // (beyond a pole) read as 0 and carry zero coupling (A5)
      if (w == 0 || w == TJ - 1)
        *reinterpret_cast<double2 *>(&sm[slot][hslot][2 + 2 * lane]) = hv ? h : Z2;
      __syncwarp();
      if (cv) sm[slot][w + 1][hs] = cvv;
    }
  };

  double acc0 = 0.0, acc1 = 0.0;  // A: p.q      B: r.z, r.r
  double2 pm, pc, pn;
  LoadA L;
  // prologue: planes c0-1 and c0
  load(c0 - 1, L);
  transform(c0 - 1, L, pm, 2, false);
  load(c0, L);
  transform(c0, L, pc, c0 % 3, true);
  if (c0 + 1 <= c1) load(c0 + 1, L);

  for (int il = c0; il < c1; il++) {
    const int slot_n = (il + 1) % 3, slot_c = il % 3;
    transform(il + 1, L, pn, slot_n, il + 1 < c1);
    // In pass B, r of plane il arrived with the load of plane il+1.
    const double2 rcur = L.r;
    if (il + 2 <= c1) load(il + 2, L);
    __syncthreads();
    if (jv) {
      const PlaneC P = plane_c(M, G.i0 + il);
      const double2 up = *reinterpret_cast<const double2 *>(&sm[slot_c][w][2 + 2 * lane]);
      const double2 dn = *reinterpret_cast<const double2 *>(&sm[slot_c][w + 2][2 + 2 * lane]);
      const double lf = sm[slot_c][w + 1][1 + 2 * lane];
      const double rt = sm[slot_c][w + 1][4 + 2 * lane];
      // element 0: left = lf, right = pc.y (or the wrap halo if element 1 is
      // padding); element 1: left = pc.x, right = rt
      const double c0v = pc.x, c1v = pc.y;
      const double r0n = kv1 ? c1v : sm[slot_c][w + 1][3 + 2 * lane];
      double q0 = dp0 * (rw.g * (P.arp * (c0v - pn.x) + P.arm * (c0v - pm.x) + P.ss * c0v) +
                         P.dr * (rw.atp * (c0v - dn.x) + rw.atm * (c0v - up.x))) +
                  P.dr * rw.q * (app0 * (c0v - r0n) + apm0 * (c0v - lf));
      double q1 = dp1 * (rw.g * (P.arp * (c1v - pn.y) + P.arm * (c1v - pm.y) + P.ss * c1v) +
                         P.dr * (rw.atp * (c1v - dn.y) + rw.atm * (c1v - up.y))) +
                  P.dr * rw.q * (app1 * (c1v - rt) + apm1 * (c1v - c0v));
      if (PASS_A) {
        if (kv0) acc0 += c0v * q0;
        if (kv1) acc0 += c1v * q1;
      } else {
        const long long o = cidx(G, il, j, k);
        double2 rn;
        rn.x = rcur.x - alpha * q0;
        rn.y = rcur.y - alpha * q1;
        if (USE_Z) {  // PC2: z is formed by the sweeps; only ||r||^2 here
          if (kv0) acc1 += rn.x * rn.x;
          if (kv1) acc1 += rn.y * rn.y;
        } else {
          const DiagRow d = diag_row(P, rw);
          const double z0 = rn.x / (dp0 * d.a + d.b * sk0);
          const double z1 = rn.y / (dp1 * d.a + d.b * sk1);
          if (kv0) {
            acc0 += rn.x * z0;
            acc1 += rn.x * rn.x;
          }
          if (kv1) {
            acc0 += rn.y * z1;
            acc1 += rn.y * rn.y;
          }
        }
        if (kv1) {
          __stcs(reinterpret_cast<double2 *>(A.r_out + o), rn);
        } else if (kv0) {
          A.r_out[o] = rn.x;
        }
      }
    }
    pm = pc;
    pc = pn;
  }

  // ---- reductions ----
  if (PASS_A) {
    double v[1] = {acc0}, tot[1];
    if (grid_sum<1>(v, A.partials, &S->counter[0], sred, tot) && threadIdx.x == 0) {
      if (A.finalize)
        finalize_alpha(S, tot[0]);
      else
        A.local_sum[0] = tot[0];
    }
  } else {
    double v[2] = {acc0, acc1}, tot[2];
    if (grid_sum<2>(v, A.partials, &S->counter[1], sred, tot) && threadIdx.x == 0) {
      if (A.finalize) {
        if (USE_Z) {
          finalize_rr(S, tot[1], A.hist);  // PC2: rho' comes from the sweeps
        } else {
          finalize_beta(S, tot[0], tot[1], A.hist);
        }
      } else {
        A.local_sum[0] = tot[0];
        A.local_sum[1] = tot[1];
      }
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, PASS_MINB) k_pass_a_pc1(PassArgs A) { pass_body<true, false>(A); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB) k_pass_a_pc2(PassArgs A) { pass_body<true, true>(A); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB) k_pass_b_pc1(PassArgs A) { pass_body<false, false>(A); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB) k_pass_b_pc2(PassArgs A) { pass_body<false, true>(A); }

// ---------------------------------------------------------------------------
// Multi-rank scalar finalisation: sum the all-gathered per-rank sums in rank
// order (bit-identical on every rank), then the same updates.
// ---------------------------------------------------------------------------
__global__ void k_finalize_alpha(Scalars *S, const double *gathered, int nranks) {
  if (S->stop) return;
  double s = 0.0;
  for (int r = 0; r < nranks; r++) s += gathered[r * 2 + 0];
  finalize_alpha(S, s);
}
__global__ void k_finalize_beta(Scalars *S, const double *gathered, int nranks, double *hist) {
  if (S->stop) return;
  double rz = 0.0, rr = 0.0;
  for (int r = 0; r < nranks; r++) {
    rz += gathered[r * 2 + 0];
    rr += gathered[r * 2 + 1];
  }
  finalize_beta(S, rz, rr, hist);
}

__global__ void k_finalize_rr(Scalars *S, const double *gathered, int nranks, double *hist) {
  if (S->stop) return;
  double rr = 0.0;
  for (int r = 0; r < nranks; r++) rr += gathered[r * 2 + 1];
  finalize_rr(S, rr, hist);
}
__global__ void k_finalize_rho(Scalars *S, const double *gathered, int nranks) {
  if (S->stop) return;
  double rz = 0.0;
  for (int r = 0; r < nranks; r++) rz += gathered[r * 2 + 0];
  finalize_rho(S, rz);
}

// ---------------------------------------------------------------------------
// Edge shells / whole-slab PC1 apply (see pot3d_internal.cuh for the modes).
// ---------------------------------------------------------------------------
__global__ void k_edge_p(Grid G, Metrics M, Scalars *S, const double *src, const double *p_old,
                         double *p_new, int mode) {
  if (mode >= 0 && S->stop) return;
  const double beta = (mode >= 0) ? S->beta : 0.0;
  const long long per = (long long)G.nt * G.np;
  const long long n = (mode < 0) ? per * G.nr_loc : 2 * per;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    long long t = c % per;
    int sidx = (int)(c / per);
    int il = (mode < 0) ? sidx : (sidx == 0 ? 0 : G.nr_loc - 1);
    int k = (int)(t % G.np), j = (int)(t / G.np);
    const long long o = cidx(G, il, j, k);
    double zv;
    if (mode == 1) {
      zv = src[o];
    } else {
      const PlaneC P = plane_c(M, G.i0 + il);
      const RowC R = row_c(M, j);
      const DiagRow d = diag_row(P, R);
      zv = src[o] / (__ldg(M.dp + k) * d.a + d.b * (__ldg(M.app + k) + __ldg(M.apm + k)));
    }
    p_new[o] = (mode < 0) ? zv : zv + beta * p_old[o];
  }
}

// ---------------------------------------------------------------------------
// Init: rho_0 = b . D^-1 b (PC1) and ||b||^2 over this rank's cells.
// r already holds b.  Grid-stride over cells.
// ---------------------------------------------------------------------------
__global__ void k_init_dots(Grid G, Metrics M, Scalars *S, const double *r, double *partials,
                            int finalize, double *local_sum, int use_z, const double *z) {
  __shared__ double sred[64];
  double a0 = 0.0, a1 = 0.0;
  const long long ncell = (long long)G.nr_loc * G.nt * G.np;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncell;
       c += (long long)gridDim.x * blockDim.x) {
    int k = (int)(c % G.np);
    long long t = c / G.np;
    int j = (int)(t % G.nt);
    int il = (int)(t / G.nt);
    const long long o = cidx(G, il, j, k);
    double rv = r[o];
    double zv;
    if (use_z) {
      zv = z[o];
    } else {
      const PlaneC P = plane_c(M, G.i0 + il);
      const RowC R = row_c(M, j);
      const DiagRow d = diag_row(P, R);
      zv = rv / (__ldg(M.dp + k) * d.a + d.b * (__ldg(M.app + k) + __ldg(M.apm + k)));
    }
    a0 += rv * zv;
    a1 += rv * rv;
  }
  double v[2] = {a0, a1}, tot[2];
  if (grid_sum<2>(v, partials, &S->counter[2], sred, tot) && threadIdx.x == 0) {
    if (finalize) {
      S->rho = tot[0];
      S->bnorm = sqrt(tot[1]);
      S->rr = tot[1];
      S->iter = 0;
      S->beta = 0.0;
      S->alpha = 0.0;
      S->alpha_prev = 0.0;
      S->status = 0;
      S->stop = (tot[1] == 0.0) ? 1 : 0;
    } else {
      local_sum[0] = tot[0];
      local_sum[1] = tot[1];
    }
  }
}

__global__ void k_init_finalize(Scalars *S, const double *gathered, int nranks) {
  double rz = 0.0, bb = 0.0;
  for (int r = 0; r < nranks; r++) {
    rz += gathered[r * 2 + 0];
    bb += gathered[r * 2 + 1];
  }
  S->rho = rz;
  S->bnorm = sqrt(bb);
  S->rr = bb;
  S->iter = 0;
  S->beta = 0.0;
  S->alpha = 0.0;
  S->alpha_prev = 0.0;
  S->status = 0;
  S->stop = (bb == 0.0) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Plain 7-point apply y = A x over this rank's cells (x has valid ghost
// shells).  One thread per cell; used for diagnostics and the true residual.
// mode 0: y = A x;  mode 1: y = b - A x restricted (b on shell il0 = bshell)
// and accumulate ||y||^2.
// ---------------------------------------------------------------------------
__global__ void k_apply(Grid G, Metrics M, const double *x, double *y, const double *bshell,
                        int b_il, Scalars *S, double *partials, double *local_sum) {
  __shared__ double sred[64];
  double acc = 0.0;
  const long long ncell = (long long)G.nr_loc * G.nt * G.np;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncell;
       c += (long long)gridDim.x * blockDim.x) {
    int k = (int)(c % G.np);
    long long t = c / G.np;
    int j = (int)(t % G.nt);
    int il = (int)(t / G.nt);
    const long long o = cidx(G, il, j, k);
    const PlaneC P = plane_c(M, G.i0 + il);
    const RowC R = row_c(M, j);
    const double dpk = __ldg(M.dp + k), appk = __ldg(M.app + k), apmk = __ldg(M.apm + k);
    const int kp = (k == G.np - 1) ? 0 : k + 1, km = (k == 0) ? G.np - 1 : k - 1;
    const double c0 = x[o];
    const double xip = x[o + G.plane], xim = x[o - G.plane];
    const double xjp = (j < G.nt - 1) ? x[o + G.PK] : 0.0;
    const double xjm = (j > 0) ? x[o - G.PK] : 0.0;
    const double xkp = x[o - k + kp], xkm = x[o - k + km];
    double q = dpk * (R.g * (P.arp * (c0 - xip) + P.arm * (c0 - xim) + P.ss * c0) +
                      P.dr * (R.atp * (c0 - xjp) + R.atm * (c0 - xjm))) +
               P.dr * R.q * (appk * (c0 - xkp) + apmk * (c0 - xkm));
    if (bshell) {
      double bv = (il == b_il) ? bshell[(long long)j * G.PK + k] : 0.0;
      q = bv - q;
      acc += q * q;
    }
    if (y) y[o] = q;
  }
  if (partials) {
    double v[1] = {acc}, tot[1];
    if (grid_sum<1>(v, partials, &S->counter[3], sred, tot) && threadIdx.x == 0) local_sum[0] = tot[0];
  }
}

// ---------------------------------------------------------------------------
// a2: RHS on the photosphere shell (rank owning global shell 0):
//   b_{0,j,k} = -r0^2 g_j dp_k (Br0_{j,k} - mean)   (Eq.2, A6)
// mean = area-weighted mean for the closed wall (A8), else 0.
// br is the device-layout map [j][k] with pitch PK.
// ---------------------------------------------------------------------------
__global__ void k_br_mean(Grid G, Metrics M, const double *br, double *out2) {
  // single block, deterministic: sum_w br w and sum_w w with w = g_j dp_k
  __shared__ double sred[64];
  double a0 = 0.0, a1 = 0.0;
  for (long long c = threadIdx.x; c < (long long)G.nt * G.np; c += blockDim.x) {
    int k = (int)(c % G.np), j = (int)(c / G.np);
    double wgt = __ldg(M.g + j) * __ldg(M.dp + k);
    a0 += wgt * br[(long long)j * G.PK + k];
    a1 += wgt;
  }
  double v[2] = {a0, a1};
  block_sum<2>(v, sred);
  if (threadIdx.x == 0) {
    out2[0] = v[0];
    out2[1] = v[1];
  }
}

__global__ void k_rhs(Grid G, Metrics M, double r0, const double *br, const double *mean2,
                      double *bshell) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)G.nt * G.np) return;
  int k = (int)(c % G.np), j = (int)(c / G.np);
  double mean = mean2 ? mean2[0] / mean2[1] : 0.0;
  long long o = (long long)j * G.PK + k;
  bshell[o] = -r0 * r0 * __ldg(M.g + j) * __ldg(M.dp + k) * (br[o] - mean);
}

// ---------------------------------------------------------------------------
// a11 finish: x += alpha_prev * p_last over owned cells (vectorised rows).
// ---------------------------------------------------------------------------
__global__ void k_axpy_cells(Grid G, double *x, const double *p, const Scalars *S) {
  const double a = S->alpha_prev;
  const long long n = (long long)G.nr_loc * G.plane;
  double *xo = x + G.plane;
  const double *po = p + G.plane;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x)
    xo[c] += a * po[c];
}

// Closed-wall gauge: sums of V x and V over this rank (V = vr_i g_j dp_k).
__global__ void k_gauge_sums(Grid G, Metrics M, const double *vr, const double *x, Scalars *S,
                             double *partials, double *local_sum) {
  __shared__ double sred[64];
  double a0 = 0.0, a1 = 0.0;
  const long long ncell = (long long)G.nr_loc * G.nt * G.np;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncell;
       c += (long long)gridDim.x * blockDim.x) {
    int k = (int)(c % G.np);
    long long t = c / G.np;
    int j = (int)(t % G.nt);
    int il = (int)(t / G.nt);
    double V = __ldg(vr + G.i0 + il) * __ldg(M.g + j) * __ldg(M.dp + k);
    a0 += V * x[cidx(G, il, j, k)];
    a1 += V;
  }
  double v[2] = {a0, a1}, tot[2];
  if (grid_sum<2>(v, partials, &S->counter[3], sred, tot) && threadIdx.x == 0) {
    local_sum[0] = tot[0];
    local_sum[1] = tot[1];
  }
}

__global__ void k_gauge_shift(Grid G, double *x, const double *gathered, int nranks) {
  double sx = 0.0, sv = 0.0;
  for (int r = 0; r < nranks; r++) {
    sx += gathered[2 * r];
    sv += gathered[2 * r + 1];
  }
  const double mean = sx / sv;
  const long long ncell = (long long)G.nr_loc * G.nt * G.np;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncell;
       c += (long long)gridDim.x * blockDim.x) {
    int k = (int)(c % G.np);
    long long t = c / G.np;
    int j = (int)(t % G.nt);
    int il = (int)(t / G.nt);
    x[cidx(G, il, j, k)] -= mean;
  }
}

// ---------------------------------------------------------------------------
// Transposes between the user layout a[i + n_i*(j + nt*k)] (r fastest) and
// the device layout d[i*stride_i + j*PK + k] (phi fastest), tiled 32x32 over
// (i, k) at fixed j.  to_dev: user -> device.
// ---------------------------------------------------------------------------
__global__ void k_transpose(int ni, int nt, int np, long long stride_i, int PK, const double *src,
                            double *dst, int to_dev) {
  __shared__ double tile[32][33];
  const int j = blockIdx.z;
  const int i_b = blockIdx.y * 32, k_b = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (to_dev) {
    // read user: contiguous in i
    for (int kk = ty; kk < 32; kk += 8) {
      int k = k_b + kk, i = i_b + tx;
      if (k < np && i < ni) tile[kk][tx] = src[i + (long long)ni * (j + (long long)nt * k)];
    }
    __syncthreads();
    for (int ii = ty; ii < 32; ii += 8) {
      int i = i_b + ii, k = k_b + tx;
      if (k < np && i < ni) dst[i * stride_i + (long long)j * PK + k] = tile[tx][ii];
    }
  } else {
    for (int ii = ty; ii < 32; ii += 8) {
      int i = i_b + ii, k = k_b + tx;
      if (k < np && i < ni) tile[tx][ii] = src[i * stride_i + (long long)j * PK + k];
    }
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {
      int k = k_b + kk, i = i_b + tx;
      if (k < np && i < ni) dst[i + (long long)ni * (j + (long long)nt * k)] = tile[kk][tx];
    }
  }
}

// ---------------------------------------------------------------------------
// a11 field: B = grad Phi on staggered faces (A16) in the device layout.
// x has valid ghost shells (halo-exchanged on multi-rank runs).
// ---------------------------------------------------------------------------

__global__ void k_field_r(FieldArgs F) {
  const Grid &G = F.G;
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)F.nbr * G.nt * G.np) return;
  int k = (int)(c % G.np);
  long long t = c / G.np;
  int j = (int)(t % G.nt);
  int fl = (int)(t / G.nt);
  int I = G.i0 + fl;  // global face index: between cells I-1 and I
  double v;
  if (I == 0) {
    // ghost x(1) = x(2) - vmask*br0*dr1, vmask = 1 (A6)
    double mean = F.mean2 ? F.mean2[0] / F.mean2[1] : 0.0;
    double x0 = F.x[cidx(G, 0, j, k)];
    double ghost = x0 - (F.br[(long long)j * G.PK + k] - mean) * F.dr[0];
    v = (x0 - ghost) / F.dr[0];
  } else if (I == G.nr) {
    double xl = F.x[cidx(G, fl - 1, j, k)];
    double ghost = (F.bc == 0) ? -xl : xl;  // source surface / closed wall (A7)
    v = (ghost - xl) / F.dr[G.nr - 1];
  } else {
    v = (F.x[cidx(G, fl, j, k)] - F.x[cidx(G, fl - 1, j, k)]) / F.drh[I - 1];
  }
  F.Br[(long long)fl * G.plane + (long long)j * G.PK + k] = v;
}

// per-shell polar ring averages, Eq.3; one block per (shell, pole)
__global__ void k_pole_avg(Grid G, const double *x, const double *dp, double period, double *poleN,
                           double *poleS) {
  __shared__ double sred[64];
  const int il = blockIdx.x;
  const int south = blockIdx.y;
  const int j = south ? G.nt - 1 : 0;
  double a = 0.0;
  for (int k = threadIdx.x; k < G.np; k += blockDim.x) a += dp[k] * x[cidx(G, il, j, k)];
  double v[1] = {a};
  block_sum<1>(v, sred);
  if (threadIdx.x == 0) (south ? poleS : poleN)[il] = v[0] / period;
}

__global__ void k_field_t(FieldArgs F) {
  const Grid &G = F.G;
  const int ntf = G.nt + 1;
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)G.nr_loc * ntf * G.np) return;
  int k = (int)(c % G.np);
  long long t = c / G.np;
  int jf = (int)(t % ntf);
  int il = (int)(t / ntf);
  const double rci = F.rc[G.i0 + il];
  double v;
  if (jf == 0) {
    v = (F.x[cidx(G, il, 0, k)] - F.poleN[il]) / (rci * (F.tc[0] - F.tf[0]));
  } else if (jf == G.nt) {
    v = (F.poleS[il] - F.x[cidx(G, il, G.nt - 1, k)]) / (rci * (F.tf[G.nt] - F.tc[G.nt - 1]));
  } else {
    v = (F.x[cidx(G, il, jf, k)] - F.x[cidx(G, il, jf - 1, k)]) / (rci * F.dth[jf - 1]);
  }
  F.Bt[(long long)il * ntf * G.PK + (long long)jf * G.PK + k] = v;
}

__global__ void k_field_p(FieldArgs F) {
  const Grid &G = F.G;
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)G.nr_loc * G.nt * G.np) return;
  int k = (int)(c % G.np);
  long long t = c / G.np;
  int j = (int)(t % G.nt);
  int il = (int)(t / G.nt);
  int kp = (k == G.np - 1) ? 0 : k + 1;
  double v = (F.x[cidx(G, il, j, kp)] - F.x[cidx(G, il, j, k)]) /
             (F.rc[G.i0 + il] * F.st[j] * F.dph[k]);
  F.Bp[cidx(G, il, j, k) - G.plane] = v;
}

}  // namespace pot3d
