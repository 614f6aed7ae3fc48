// cg1.cu -- the single-reduction PCG variant (opt-in:
// pot3d_runtime.variant = 1), PC1 only.
//
// Chronopoulos & Gear (1989), in the form of Ghysels & Vanroose (2014) Alg. 2
// (oracle/pot3d_oracle.c orc_pcg variant ORC_PCG_CG1 states it step by step):
//   p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s;
//   u = M^-1 r;  w = A u;  gamma = r.u, delta = w.u, ||r||^2  (ONE reduction)
// The paper names the inner products' "collective/synchronous nature" as the
// scaling limiter; this variant has one global reduction per
// iteration instead of two.  As in the standard PC1 path the stored residual
// is u = D^-1 r (reading A22), so r = D u is never stored.
//
//   k_cg1_update (K1): w = A u from the staged, haloed u box (U[par]); then per cell
//       p' = u + beta p, s' = w + beta s, u' = u - alpha D^-1 s' (into U[par^1]),
//       and on odd iterations x += alpha_{k-1} p_{k-1} + alpha_k p_k with
//       p_{k-1} = (p' - u) / beta (reading A23).  No reduction.  [48 / 64 B/cell]
//   k_cg1_dots   (K2): w' = A u' from the staged u' box; gamma = sum D u'^2,
//       delta = sum w' u', ||r||^2 = sum (D u')^2 -> finalize (alpha, beta,
//       convergence) in the last block.                                  [8 B/cell]
// Per iteration 56 B/cell on average + 8 B/cell, one reduction (PCG: 56 B, two).
//
// Across ranks with peer memory (Cg1Args::peers): K1's blocks that own shell 0 or
// nr_loc-1 also store those shells of u' into the neighbours' ghost shells (CUDA IPC /
// loopback pointers, the p_lo / p_hi maps: U[b] is P[b]); the last of them raises the
// neighbours' halo flags for this iteration.  K2's blocks whose chunk touches a ghost
// shell wait for their flag before the TMA unit reads it, and the last block posts
// (gamma, delta) and ||r||^2 into every rank's mailbox; k_finalize_cg1_mail sums them in
// rank order.  Every wait is on a kernel of the previous phase on another GPU (no
// co-residency assumption), and no rank can overwrite a ghost shell still being read:
// its next K1 needs this iteration's alpha, which needs every rank's K2.  With one
// reduction per iteration a fast rank can post iteration k+1 before a slow one has
// read iteration k, so the mailbox slots alternate by iteration parity (MAIL_A/B on
// even, MAIL_C/D on odd iterations): reaching k+2 needs every rank's k+1 posts, which
// follow their reads of k.
#include "pass_common.cuh"

namespace pot3d {

struct SmemC1 {
  double u[NS_C][TR][SROW];
  double p[NS_C][TJ][TKB];
  double s[NS_C][TJ][TKB];
  double x[NS_C][TJ][TKB];
  uint64_t bar[NS_C];
};
struct SmemC2 {
  double u[NS_D][TR][SROW];
  uint64_t bar[NS_D];
};
static_assert(sizeof(SmemC1) <= SMEM_C1 && sizeof(SmemC2) <= SMEM_C2, "CG1 shared memory");

// the CG1 scalar updates (one thread), rank-order sums already formed
__device__ __forceinline__ void finalize_cg1(Scalars *S, double gamma, double delta, double rr, double *hist,
                                             bool init) {
  if (init) {  // gamma_0 = r0.u0, delta_0 = (A u0).u0, alpha_0 = gamma_0 / delta_0, beta_0 = 0
    S->rho = gamma;
    S->sigma = delta;
    S->beta = 0.0;
    if (!(delta > 0.0)) {
      S->status = -4;
      S->stop = 1;
      return;
    }
    S->alpha = gamma / delta;
    return;
  }
  const long long it = S->iter + 1;
  S->iter = it;
  S->rr = rr;
  const double rn = sqrt(rr);
  if (hist && it < S->hist_len) hist[it] = rn / S->bnorm;
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
  const double beta = gamma / S->rho;
  const double den = delta - beta * gamma / S->alpha;  // = p.Ap in exact arithmetic
  S->sigma = den;
  if (!(den > 0.0)) {
    S->status = -4;
    S->stop = 1;
    return;
  }
  S->beta = beta;
  S->alpha = gamma / den;
  S->rho = gamma;
}

// sequence number of an iteration's CG1 exchange (the start's reduction: 0)
__device__ __forceinline__ unsigned long long cg1_seq(const Scalars *S, int init) {
  return mail_seq(S->epoch, init ? 0 : S->iter + 1);
}

__global__ void k_finalize_cg1_mail(Scalars *S, const PeerTab *peers, double *hist) {
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  const unsigned long long seq = cg1_seq(S, 0);
  const int k0 = (S->iter & 1) ? MAIL_C : MAIL_A;  // the slots of this iteration's parity
  double g, d, rr, unused;
  if (!mail_collect(peers, k0, seq, S, g, d) || !mail_collect(peers, k0 + 1, seq, S, rr, unused)) {
    S->status = -5;
    S->stop = 1;
    return;
  }
  finalize_cg1(S, g, d, rr, hist, false);
}

__global__ void k_finalize_cg1(Scalars *S, const double *gathered, int nranks, double *hist, int init) {
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  double g = 0.0, d = 0.0, rr = 0.0;
  for (int r = 0; r < nranks; r++) {
    g += gathered[4 * r + 0];
    d += gathered[4 * r + 1];
    rr += gathered[4 * r + 2];
  }
  finalize_cg1(S, g, d, rr, hist, init != 0);
}

// ---------------------------------------------------------------------------
// K1: the vector update of one iteration (parity: u is read from U[parity])
// ---------------------------------------------------------------------------
template <int XM, bool FAST>
__device__ __forceinline__ void cg1_update_body(const Cg1Maps &T, const Cg1Args &A, int parity, PassShared &sh) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemC1 &sm = *reinterpret_cast<SmemC1 *>(smem_raw);
  TileConst &tcs = sh.tcs;
  PlaneSm &pls = sh.pls;
  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.k0);
  load_planes(pls, M, G.i0 + t.c0 - 1, L + 2);
  const int cs = 2 + 2 * t.lane;
  const long long PL = G.plane;
  const void *map_u = &T.u_h[parity];
  constexpr unsigned UB = TR * SROW * 8u, IB = TJ * TKB * 8u;
  RowC rw[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) rw[e] = row_c(M, min(max(t.j0 - 1 + t.row[e], 0), G.nt - 1));
  int qi = 0, si = 0;
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      const bool rown = (qi >= 1) && (qi <= L);
      mbar_arrive_expect_tx(&sm.bar[si], rown ? UB + (XM == XM_PAIR ? 3 : 2) * IB : UB);
      tma_load_3d(&sm.u[si][0][0], map_u, &sm.bar[si], t.k0 - 3 + COFF, t.j0 - 1, il + 1);
      if (rown) {
        tma_load_3d(&sm.p[si][0][0], &T.p_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, il + 1);
        tma_load_3d(&sm.s[si][0][0], &T.s_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, il + 1);
        if (XM == XM_PAIR) tma_load_3d(&sm.x[si][0][0], &T.x_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, il + 1);
      }
    }
    ++qi;
    si = wrap_inc(si, NS_C);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS_C; s++) mbar_init(&sm.bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) trace_mark(S, TR_B0);
  const double alpha = S->alpha, beta = S->beta;
  const double cpair = (XM == XM_PAIR) ? S->alpha_prev / beta : 0.0;  // alpha_{k-1} / beta_k
  const double cp = cpair + alpha;
  if (threadIdx.x == 0)
    for (int s = 0; s < NS_C - 2; s++) issue();

  const double2 Z2 = make_double2(0.0, 0.0);
  double2 um[RPW], uc[RPW], un[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) um[e] = uc[e] = un[e] = Z2;
  double *g_u = A.u[parity ^ 1] + (long long)(t.c0 + 1) * PL;  // + rowoff[e]: plane c0
  // peer memory: u' of shell 0 / nr_loc-1 also lands in rank-1's top / rank+1's bottom
  // ghost shell (the same [il+1][j][c] layout shifted by whole planes)
  const PeerTab *pt = A.peers;
  double *lo = pt ? pt->p_lo[parity ^ 1] : nullptr, *hi = pt ? pt->p_hi[parity ^ 1] : nullptr;
  if (lo) lo += (long long)pt->nr_lo * PL;
  if (hi) hi -= (long long)G.nr_loc * PL;
  const bool edge_blk = pt && (t.c0 == 0 || t.c1 == G.nr_loc);
  double *g_p = A.p + (long long)(t.c0 + 1) * PL;
  double *g_s = A.s + (long long)(t.c0 + 1) * PL;
  double *g_x = A.x + (long long)(t.c0 + 1) * PL;
  int st = 0, so = NS_C - 1;
  unsigned ph = 0;
  auto st2 = [&](double *a, double2 v) {  // interior store (p, s, x: no ghost columns)
    if (FAST || (t.st0 && t.st1)) {
      __stcs(reinterpret_cast<double2 *>(a), v);
    } else {
      if (t.st0) a[0] = v.x;
      if (t.st1) a[1] = v.y;
    }
  };
#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    __syncthreads();  // stage (q-2)%NS_C is free
    if (threadIdx.x == 0) issue();
    const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
    const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
    const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
    const PlaneC P = plane_at(pls, q >= 1 ? q - 1 : 0);
    mbar_wait(&sm.bar[st], ph);
#pragma unroll
    for (int e = 0; e < RPW; e++) un[e] = *reinterpret_cast<const double2 *>(&sm.u[st][t.row[e]][cs]);
    if (q >= 2) {
      const double *sb = &sm.u[so][0][0];
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        if (!t.stencil[e]) continue;
        const int r = t.row[e];
        const double *sr = sb + r * SROW + cs;
        const double2 up = (RPW == 2 && e == 1) ? uc[0] : *reinterpret_cast<const double2 *>(sr - SROW);
        const double2 dn = (RPW == 2 && e == 0) ? uc[RPW - 1] : *reinterpret_cast<const double2 *>(sr + SROW);
        const double lf = sr[-1], rt = sr[2];
        const double w0 = stencil7(uc[e].x, un[e].x, um[e].x, dn.x, up.x, uc[e].y, lf, dp.x, ap.x, am.x, P, rw[e]);
        const double w1 = stencil7(uc[e].y, un[e].y, um[e].y, dn.y, up.y, rt, uc[e].x, dp.y, ap.y, am.y, P, rw[e]);
        const double2 pv = *reinterpret_cast<const double2 *>(&sm.p[so][r - 1][2 * t.lane]);
        const double2 sv = *reinterpret_cast<const double2 *>(&sm.s[so][r - 1][2 * t.lane]);
        double2 pn, sn, unw;
        pn.x = fma(beta, pv.x, uc[e].x);
        pn.y = fma(beta, pv.y, uc[e].y);
        sn.x = fma(beta, sv.x, w0);
        sn.y = fma(beta, sv.y, w1);
        const DiagRow d = diag_row(P, rw[e]);
        const double d0 = diag_at(dp.x, d, ap.x, am.x), d1 = diag_at(dp.y, d, ap.y, am.y);
        unw.x = fma(-alpha, jacobi(sn.x, d0), uc[e].x);
        unw.y = fma(-alpha, jacobi(sn.y, d1), uc[e].y);
        const long long o = t.rowoff[e];
        POT3D_CHK(S, in_range(g_u + o, A.u[parity ^ 1], (G.nr_loc + 2) * PL) &&
                         in_range(g_p + o, A.p, (G.nr_loc + 2) * PL), CHK_CG1_STORE);
        store_pair<FAST>(g_u + o, t, G.np, unw, true);
        if (edge_blk) {
          const int il = t.c0 + q - 2;  // the shell of this store
          double *rem = il == 0 ? lo : (il == G.nr_loc - 1 ? hi : nullptr);
          // (lanes past the grid's last column store nothing: their row offset may leave the plane)
          POT3D_CHK(S, !rem || !(FAST || t.st0 || t.st1) || (il == 0 ? in_range(rem + (g_u - A.u[parity ^ 1]) + o,
                                                   pt->p_lo[parity ^ 1] + (long long)(pt->nr_lo + 1) * PL, PL)
                                        : in_range(rem + (g_u - A.u[parity ^ 1]) + o, pt->p_hi[parity ^ 1], PL)),
                    CHK_PEER_STORE);
          if (rem) store_pair<FAST>(rem + (g_u - A.u[parity ^ 1]) + o, t, G.np, unw, false);
        }
        st2(g_p + o, pn);
        st2(g_s + o, sn);
        if (XM == XM_PAIR) {
          const double2 xv = *reinterpret_cast<const double2 *>(&sm.x[so][r - 1][2 * t.lane]);
          double2 xn;
          xn.x = fma(cp, pn.x, fma(-cpair, uc[e].x, xv.x));
          xn.y = fma(cp, pn.y, fma(-cpair, uc[e].y, xv.y));
          st2(g_x + o, xn);
        }
      }
      g_u += PL;
      g_p += PL;
      g_s += PL;
      g_x += PL;
    }
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      um[e] = uc[e];
      uc[e] = un[e];
    }
    so = st;
    st = wrap_inc(st, NS_C);
    ph ^= (st == 0);
  }
  // end of the last block (the dots kernel's griddepcontrol.wait covers this grid's stores)
  if (threadIdx.x == 0) trace_max(S, TR_B1);
  if (edge_blk) {  // every edge block's peer stores released, then the last raises the flags
    const unsigned nedge = (unsigned)(gridDim.x * (G.nchunks > 1 ? 2 : 1));
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(&S->counter[4], 1u) == nedge - 1) {
        S->counter[4] = 0u;
        raise_halo_flags(pt, cg1_seq(S, 0));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2: w' = A u' and the three inner products of the single reduction
// ---------------------------------------------------------------------------
template <bool FAST>
__device__ __forceinline__ void cg1_dots_body(const Cg1Maps &T, const Cg1Args &A, int parity, PassShared &sh) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemC2 &sm = *reinterpret_cast<SmemC2 *>(smem_raw);
  double *sred = sh.sred;
  TileConst &tcs = sh.tcs;
  PlaneSm &pls = sh.pls;
  const TileThread t = tile_thread(G);
  const bool m0 = FAST || t.st0, m1 = FAST || t.st1;
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.k0);
  load_planes(pls, M, G.i0 + t.c0 - 1, L + 2);
  const int cs = 2 + 2 * t.lane;
  const void *map_u = &T.u_h[parity];
  constexpr unsigned UB = TR * SROW * 8u;
  RowC rw[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) rw[e] = row_c(M, min(max(t.j0 - 1 + t.row[e], 0), G.nt - 1));
  int qi = 0, si = 0;
  const PeerTab *pt = A.init ? nullptr : A.peers;  // the start's halo comes by copies
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      if (pt && (il < 0 || il >= G.nr_loc)) {  // a ghost shell: the neighbour's u' of this iteration
        const int side = il < 0 ? 0 : 1;
        if (side == 0 ? pt->rank > 0 : pt->rank < pt->nranks - 1) {
          xfer_wait(&pt->mail[pt->rank]->halo[side], cg1_seq(S, 0), S);
          fence_proxy_async_global();
        }
      }
      mbar_arrive_expect_tx(&sm.bar[si], UB);
      tma_load_3d(&sm.u[si][0][0], map_u, &sm.bar[si], t.k0 - 3 + COFF, t.j0 - 1, t.c0 + qi);
    }
    ++qi;
    si = wrap_inc(si, NS_D);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS_D; s++) mbar_init(&sm.bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) trace_mark(S, TR_A0);
  if (threadIdx.x == 0)
    for (int s = 0; s < NS_D - 2; s++) issue();
  const double2 Z2 = make_double2(0.0, 0.0);
  double2 um[RPW], uc[RPW], un[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) um[e] = uc[e] = un[e] = Z2;
  double ag = 0.0, ad = 0.0, ar = 0.0;
  int st = 0, so = NS_D - 1;
  unsigned ph = 0;
#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    __syncthreads();  // stage (q-2)%NS_D is free
    if (threadIdx.x == 0) issue();
    const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
    const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
    const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
    const PlaneC P = plane_at(pls, q >= 1 ? q - 1 : 0);
    mbar_wait(&sm.bar[st], ph);
#pragma unroll
    for (int e = 0; e < RPW; e++) un[e] = *reinterpret_cast<const double2 *>(&sm.u[st][t.row[e]][cs]);
    if (q >= 2) {
      const double *sb = &sm.u[so][0][0];
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        if (!t.stencil[e]) continue;
        const int r = t.row[e];
        const double *sr = sb + r * SROW + cs;
        const double2 up = (RPW == 2 && e == 1) ? uc[0] : *reinterpret_cast<const double2 *>(sr - SROW);
        const double2 dn = (RPW == 2 && e == 0) ? uc[RPW - 1] : *reinterpret_cast<const double2 *>(sr + SROW);
        const double lf = sr[-1], rt = sr[2];
        const double w0 = stencil7(uc[e].x, un[e].x, um[e].x, dn.x, up.x, uc[e].y, lf, dp.x, ap.x, am.x, P, rw[e]);
        const double w1 = stencil7(uc[e].y, un[e].y, um[e].y, dn.y, up.y, rt, uc[e].x, dp.y, ap.y, am.y, P, rw[e]);
        const DiagRow d = diag_row(P, rw[e]);
        const double r0 = diag_at(dp.x, d, ap.x, am.x) * uc[e].x, r1 = diag_at(dp.y, d, ap.y, am.y) * uc[e].y;
        ag += (m0 ? r0 * uc[e].x : 0.0) + (m1 ? r1 * uc[e].y : 0.0);
        ad += (m0 ? w0 * uc[e].x : 0.0) + (m1 ? w1 * uc[e].y : 0.0);
        ar += (m0 ? r0 * r0 : 0.0) + (m1 ? r1 * r1 : 0.0);
      }
    }
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      um[e] = uc[e];
      uc[e] = un[e];
    }
    so = st;
    st = wrap_inc(st, NS_D);
    ph ^= (st == 0);
  }
  double v[3] = {ag, ad, ar}, tot[3];
  if (grid_sum<3>(v, A.partials, &S->counter[5], sred, tot, pass_bid(G), pass_nb(G)) && threadIdx.x == 0) {
    trace_mark(S, TR_A1);
    if (A.finalize) {
      finalize_cg1(S, tot[0], tot[1], tot[2], A.hist, A.init != 0);
    } else if (pt) {
      const unsigned long long seq = cg1_seq(S, 0);
      const int k0 = (S->iter & 1) ? MAIL_C : MAIL_A;  // slots alternate by iteration parity
      mail_post(pt, k0, tot[0], tot[1], seq, S);
      mail_post(pt, k0 + 1, tot[2], 0.0, seq, S);
    } else {
      A.local_sum[0] = tot[0];
      A.local_sum[1] = tot[1];
      A.local_sum[2] = tot[2];
    }
  }
}

#define POT3D_CG1(BODY, ...)                                    \
  __shared__ PassShared sh;                                     \
  if (tile_fast(A.G))                                           \
    BODY<__VA_ARGS__ true>(T, A, parity, sh);                   \
  else                                                          \
    BODY<__VA_ARGS__ false>(T, A, parity, sh)

__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_cg1_update_even(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity) {
  POT3D_CG1(cg1_update_body, XM_SKIP, );
}
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_cg1_update_odd(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity) {
  POT3D_CG1(cg1_update_body, XM_PAIR, );
}
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_cg1_dots(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity) {
  POT3D_CG1(cg1_dots_body, );
}

}  // namespace pot3d
