// kernels.cu -- the sm_100a kernels around the two fused passes;
// the passes themselves are in passes.cu, the PC2 sweeps in pc2.cu.
//
//   k_metrics         a1  1-D metric factors from the faces (A1-A7)
//   k_br_mean, k_rhs  a2  closed-wall mean removal (A8); b on the photosphere shell
//                         (Eq.2)
//   k_init_dots       a10 rho_0 = b.M^-1 b and ||b|| (deterministic grid reduction)
//   k_edge_p          a5  p_k on the two edge shells (NCCL path, PC2, or
//                         POT3D_EDGE_IN_A=0), stored locally and -- peer memory --
//                         into the neighbours' ghost shells; can finalise the
//                         previous pass B's beta from the mailbox (fold)
//   k_finalize_*      a6  multi-rank scalar updates: rank-order sums of the NCCL
//                         all-gather (k_finalize_alpha/beta/rr/rho, k_init_finalize)
//                         or of the peer mailbox (k_finalize_mail)
//   k_apply           unfused 7-point apply (diagnostics, true residual)
//   k_gauge_*         closed-wall zero volume-weighted-mean gauge
//   k_pole_avg, k_field_r/t/p   a11 Eq.3 pole rings, B = grad Phi on staggered faces (A16)
//   k_transpose       user layout (r fastest) <-> device layout (phi fastest)
#include "device_common.cuh"

namespace pot3d {

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
  if (t == 0) {
    // padding entries read for ghost shells (results discarded): finite values
    for (int i : {-1, nr}) {
      arp[i] = 1.0;
      arm[i] = 1.0;
      dr[i] = 1.0;
      ss[i] = 0.0;
    }
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
                         double *p_new, int mode, const PeerTab *peers, int parity_new,
                         double *hist, int fold) {
  pdl_trigger();
  pdl_wait();
  if (mode >= 0 && S->stop) return;
  const unsigned long long t_start = (S->trace && blockIdx.x == 0 && threadIdx.x == 0) ? global_ns() : 0ull;
  // fold (peer memory, PC1): finalise the previous pass B here -- every block sums
  // the ranks' (r.z, r.r) from the mailbox in rank order and takes the same
  // decisions; only the last block (after every block has read S) writes S
  __shared__ double s_beta, s_rz, s_rr;
  __shared__ int s_stop, s_status;
  const bool pend = fold && S->pend_b;
  const long long iter0 = S->iter;
  if (threadIdx.x == 0) {
    s_stop = 0;
    s_status = 0;
    s_beta = (mode >= 0) ? S->beta : 0.0;
    if (pend) {
      double rz, rr;
      if (!mail_collect(peers, MAIL_B, mail_seq(S->epoch, iter0 + 1), S, rz, rr)) {
        s_stop = 1;
        s_status = -5;
      } else {
        s_rz = rz;
        s_rr = rr;
        const double rn = sqrt(rr);
        if (rn <= S->rtol * S->bnorm) {
          s_stop = 1;
          s_status = 0;
        } else if (iter0 + 1 >= S->maxit) {
          s_stop = 1;
          s_status = 1;
        }
        s_beta = rz / S->rho;
      }
    }
  }
  __syncthreads();
  const double beta = s_beta;
  const long long iter = pend ? iter0 + 1 : iter0;  // the iteration p_k belongs to
  if (t_start) {
    S->trace[(iter & 63) * 16 + TR_EDGE0] = t_start;
    S->trace[(iter & 63) * 16 + TR_EDGEM] = global_ns();  // mailbox collected
  }
  const long long per = (long long)G.nt * G.np;
  const long long n = (mode < 0) ? per * G.nr_loc : (s_stop ? 0 : 2 * per);
  // peer memory: shell 0 also lands in rank-1's top ghost shell, shell nr_loc-1
  // in rank+1's bottom ghost shell (same [il+1][j][c] layout, shifted by whole planes)
  double *lo = nullptr, *hi = nullptr;
  if (peers) {
    lo = peers->p_lo[parity_new];
    hi = peers->p_hi[parity_new];
    if (lo) lo += (long long)peers->nr_lo * G.plane;
    if (hi) hi -= (long long)G.nr_loc * G.plane;
  }
  bool last_edge = false;  // every block counts in, also when the loop stops here
  if (mode >= 0)
    last_edge = edge_shells(G, M, S, src, p_old, p_new, peers, parity_new, beta, blockIdx.x,
                            gridDim.x, !s_stop);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < (mode < 0 ? n : 0);
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
      zv = jacobi(src[o], diag_at(__ldg(M.dp + k), d, __ldg(M.app + k), __ldg(M.apm + k)));
    }
    // same arithmetic as pass A, so the ghost copy equals the owner's value bitwise
    const double v = (mode < 0) ? zv : fma(beta, p_old[o], zv);
    p_new[o] = v;
    if (k == 0) p_new[o + G.np] = v;           // periodic ghost columns
    if (k == G.np - 1) p_new[o - G.np] = v;
    double *rem = (mode < 0) ? nullptr : (sidx == 0 ? lo : hi);
    if (rem) {
      rem[o] = v;
      if (k == 0) rem[o + G.np] = v;
      if (k == G.np - 1) rem[o - G.np] = v;
    }
  }
  if (peers && mode >= 0) {
    if (last_edge && threadIdx.x == 0) {
      S->counter[4] = 0u;
      if (S->trace) S->trace[(iter & 63) * 16 + TR_EDGE1] = global_ns();  // iteration of p_k
      if (pend) {  // finalize_beta of the previous iteration
        S->pend_b = 0;
        if (s_status == -5) {
          S->status = -5;
          S->stop = 1;
        } else {
          S->iter = iter;
          S->rr = s_rr;
          if (hist && iter < S->hist_len) hist[iter] = sqrt(s_rr) / S->bnorm;
          S->alpha_prev = S->alpha;
          if (s_stop) {
            S->status = s_status;
            S->stop = 1;
          } else {
            S->beta = beta;
            S->rho = s_rz;
          }
        }
      }
      if (!s_stop) raise_halo_flags(peers, mail_seq(S->epoch, iter + 1));
    }
  }
}

// Peer-memory finalisation (one thread): the reductions of every rank, summed in
// rank order, then the same scalar updates as the single-rank path.
__global__ void k_finalize_mail(Scalars *S, const PeerTab *peers, int kind, int what, double *hist) {
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  if (what == 0) trace_mark(S, TR_F0);
  // kinds A/B belong to iteration iter+1 (iter not yet advanced); C follows finalize_rr
  const unsigned long long seq = mail_seq(S->epoch, what == 3 ? S->iter : S->iter + 1);
  double s0, s1;
  if (!mail_collect(peers, kind, seq, S, s0, s1)) {
    S->status = -5;
    S->stop = 1;
    return;
  }
  if (what == 0) {
    finalize_alpha(S, s0);
    trace_mark(S, TR_F1);
  } else if (what == 1)
    finalize_beta(S, s0, s1, hist);
  else if (what == 2)
    finalize_rr(S, s1, hist);
  else
    finalize_rho(S, s0);
}

// ---------------------------------------------------------------------------
// Init: rho_0 = b . D^-1 b (PC1) and ||b||^2 over this rank's cells.
// r already holds b.  Grid-stride over cells.  Warm start (keep_b, one rank): r holds
// r_0 = b - A x0 and S->bnorm = ||b|| already; rr = ||r_0||^2, the loop stops at once
// if ||r_0|| <= rtol ||b|| (A9), hist0[0] = ||r_0|| / ||b||.
// ---------------------------------------------------------------------------
__global__ void k_init_dots(Grid G, Metrics M, Scalars *S, const double *r, double *partials,
                            int finalize, double *local_sum, int use_z, const double *z, int keep_b,
                            double *hist0) {
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
      zv = jacobi(rv, diag_at(__ldg(M.dp + k), d, __ldg(M.app + k), __ldg(M.apm + k)));
    }
    a0 += rv * zv;
    a1 += rv * rv;
  }
  double v[2] = {a0, a1}, tot[2];
  if (grid_sum<2>(v, partials, &S->counter[2], sred, tot) && threadIdx.x == 0) {
    if (finalize) {
      S->rho = tot[0];
      if (!keep_b) S->bnorm = sqrt(tot[1]);
      S->rr = tot[1];
      S->iter = 0;
      S->beta = 0.0;
      S->alpha = 0.0;
      S->alpha_prev = 0.0;
      S->status = 0;
      if (keep_b) {
        const double bn = S->bnorm, rn = sqrt(tot[1]);
        S->stop = (bn == 0.0 || rn <= S->rtol * bn) ? 1 : 0;
        if (hist0) hist0[0] = bn > 0.0 ? rn / bn : 0.0;
      } else {
        S->stop = (tot[1] == 0.0) ? 1 : 0;
      }
    } else {
      local_sum[0] = tot[0];
      local_sum[1] = tot[1];
    }
  }
}

// keep_b (a warm start across ranks): the sums are r_0's, ||b|| is already in S (as
// k_init_dots' keep_b: the stopping test against ||b||, hist0[0] = ||r_0|| / ||b||)
__global__ void k_init_finalize(Scalars *S, const double *gathered, int nranks, int keep_b, double *hist0) {
  double rz = 0.0, bb = 0.0;
  for (int r = 0; r < nranks; r++) {
    rz += gathered[r * 2 + 0];
    bb += gathered[r * 2 + 1];
  }
  S->rho = rz;
  if (!keep_b) S->bnorm = sqrt(bb);
  S->rr = bb;
  S->iter = 0;
  S->beta = 0.0;
  S->alpha = 0.0;
  S->alpha_prev = 0.0;
  S->status = 0;
  if (keep_b) {
    const double bn = S->bnorm, rn = sqrt(bb);
    S->stop = (bn == 0.0 || rn <= S->rtol * bn) ? 1 : 0;
    if (hist0) hist0[0] = bn > 0.0 ? rn / bn : 0.0;
  } else {
    S->stop = (bb == 0.0) ? 1 : 0;
  }
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
      double bv = (il == b_il) ? bshell[pidx(G, j, k)] : 0.0;
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
    a0 += wgt * br[pidx(G, j, k)];
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
  long long o = pidx(G, j, k);
  bshell[o] = -r0 * r0 * __ldg(M.g + j) * __ldg(M.dp + k) * (br[o] - mean);
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
// user index i + ld*(j + nt*k) (ld >= ni: a slab of a larger r-fastest array)
__global__ void k_transpose(int ni, int nt, int np, long long stride_i, int PK, int coff,
                            const double *src, double *dst, int to_dev, int ld) {
  __shared__ double tile[32][33];
  const int j = blockIdx.z;
  const int i_b = blockIdx.y * 32, k_b = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (to_dev) {
    // read user: contiguous in i
    for (int kk = ty; kk < 32; kk += 8) {
      int k = k_b + kk, i = i_b + tx;
      if (k < np && i < ni) tile[kk][tx] = src[i + (long long)ld * (j + (long long)nt * k)];
    }
    __syncthreads();
    for (int ii = ty; ii < 32; ii += 8) {
      int i = i_b + ii, k = k_b + tx;
      if (k < np && i < ni) dst[i * stride_i + (long long)j * PK + k + coff] = tile[tx][ii];
    }
  } else {
    for (int ii = ty; ii < 32; ii += 8) {
      int i = i_b + ii, k = k_b + tx;
      if (k < np && i < ni) tile[tx][ii] = src[i * stride_i + (long long)j * PK + k + coff];
    }
    __syncthreads();
    for (int kk = ty; kk < 32; kk += 8) {
      int k = k_b + kk, i = i_b + tx;
      if (k < np && i < ni) dst[i + (long long)ld * (j + (long long)nt * k)] = tile[kk][tx];
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
    double ghost = x0 - (F.br[pidx(G, j, k)] - mean) * F.dr[0];
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
  F.Bp[(long long)il * G.plane + (long long)j * G.PK + k] = v;
}

}  // namespace pot3d
