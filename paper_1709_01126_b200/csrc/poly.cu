// poly.cu -- PC3: Chebyshev-accelerated Jacobi, the "vector-friendly"
// preconditioner of SURVEY.md §8(f)-2 (the paper calls for vectorisable
// preconditioners; not in the paper itself).  z = M^-1 r is m steps of
// Saad's Chebyshev acceleration (Iterative Methods, 2nd ed., Alg. 12.1) of
// Jacobi on A z = r from z_0 = 0 (oracle/pot3d_oracle.c orc_cheb_apply states it
// step by step):
//   res_0 = D^-1 r, d_0 = res_0 / theta, z_1 = d_0
//   k = 1..m-1: res_k = res_{k-1} - D^-1 A d_{k-1};  d_k = c1_k d_{k-1} + c2_k res_k;
//               z_{k+1} = z_k + d_k
// i.e. a fixed SPD polynomial in D^-1 A times D^-1 (interval [2/ratio, 2] of
// D^-1 A's spectrum, bounded by Gershgorin).  It replaces the PC2 sweeps in the
// same PCG: pass A reads the stored z, pass B updates r.  Across ranks a halo of d
// precedes every step (abi.cu poly_steps) and the last step posts r.z to the mailboxes.
//
//   k_poly_init (K0): res, d_0 = z_1 from r, cell by cell          [8 + 24 B/cell]
//   k_poly_step (K_k): the stencil of d_{k-1} from the staged, haloed box, then
//       res, d (the other d buffer, ghost columns kept), z updated    [48 B/cell]
//       the last step writes z_m into z (ghost columns: pass A stages it) and
//       the partial r.z (r staged as well)                           [40 B/cell]
#include "pass_common.cuh"

namespace pot3d {

struct SmemP {
  double d[NS_C][TR][SROW];   // staged d_{k-1} (haloed)
  double res[NS_C][TJ][TKB];  // staged res_{k-1}
  double x[NS_C][TJ][TKB];    // staged z_k
  double r[NS_C][TJ][TKB];    // LAST: staged r for the r.z partial
  uint64_t bar[NS_C];
};
static_assert(sizeof(SmemP) <= SMEM_P, "SMEM_P");

__global__ void k_poly_init(PolyArgs A) {
  pdl_trigger();
  pdl_wait();
  const Grid &G = A.G;
  const Metrics &M = A.M;
  const long long vo = (long long)blockIdx.y * (G.nr_loc + 2) * G.plane;  // a batch: problem blockIdx.y
  if (A.predicated && A.S[blockIdx.y].stop) return;
  const long long per = (long long)G.nt * G.np, n = per * G.nr_loc;
  // peer memory: d_0's edge shells also into the neighbours' ghost shells of their d[0]
  const PeerTab *hp = A.hpeers;
  double *rlo = hp ? hp->d_lo[0] : nullptr, *rhi = hp ? hp->d_hi[0] : nullptr;
  if (rlo) rlo += (long long)hp->nr_lo * G.plane;
  if (rhi) rhi -= (long long)G.nr_loc * G.plane;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int il = (int)(c / per);
    const long long t = c - il * per;
    const int j = (int)(t / G.np), k = (int)(t - (long long)j * G.np);
    const long long o = cidx(G, il, j, k) + vo;
    const DiagRow d = diag_row(plane_c(M, G.i0 + il), row_c(M, j));
    const double rv = jacobi(A.r[o], diag_at(__ldg(M.dp + k), d, __ldg(M.app + k), __ldg(M.apm + k)));
    const double dv = rv / A.theta;
    A.res[o] = rv;
    A.x[o] = dv;  // z_1 = d_0
    double *d0 = A.d[0];
    d0[o] = dv;
    if (k == 0) d0[o + G.np] = dv;  // periodic ghost columns: d is a stencil operand
    if (k == G.np - 1) d0[o - G.np] = dv;
    double *rem = il == 0 ? rlo : (il == G.nr_loc - 1 ? rhi : nullptr);
    if (rem) {
      rem[o] = dv;
      if (k == 0) rem[o + G.np] = dv;
      if (k == G.np - 1) rem[o - G.np] = dv;
    }
  }
  if (hp) {  // every block's peer stores released, then the last raises the flags
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(&A.S->counter[4], 1u) == gridDim.x * gridDim.y - 1) {
        A.S->counter[4] = 0u;
        raise_dhalo_flags(hp, dhalo_seq(A.S, 0));
      }
    }
  }
}

template <bool LAST, bool FAST>
__device__ __forceinline__ void poly_step_body(const PolyMaps &T, const PolyArgs &A, int step, PassShared &sh) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S + blockIdx.z;  // a batch: the problem of this block (pass_common.cuh)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemP &sm = *reinterpret_cast<SmemP *>(smem_raw);
  double *sred = sh.sred;
  TileConst &tcs = sh.tcs;
  PlaneSm &pls = sh.pls;
  const TileThread t = tile_thread(G);
  const bool m0 = FAST || t.st0, m1 = FAST || t.st1;
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.k0);
  load_planes(pls, M, G.i0 + t.c0 - 1, L + 2);
  const int cs = 2 + 2 * t.lane;
  const long long PL = G.plane;
  const int zp = rhs_planes(G);
  const long long vo = zp * PL;
  const int src = (step - 1) & 1;  // d_{k-1} lives in d[(k-1) & 1]
  const void *map_d = &T.d_h[src];
  const PeerTab *hp = A.hpeers;  // peer memory: the d halo (flags) instead of host-side copies
  constexpr unsigned DB = TR * SROW * 8u, IB = TJ * TKB * 8u;
  RowC rw[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) rw[e] = row_c(M, min(max(t.j0 - 1 + t.row[e], 0), G.nt - 1));
  int qi = 0, si = 0;
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      const bool rown = (qi >= 1) && (qi <= L);
      if (hp && (il < 0 || il >= G.nr_loc)) {  // a ghost shell: the neighbour's d_{k-1}
        const int side = il < 0 ? 0 : 1;
        if (side == 0 ? hp->rank > 0 : hp->rank < hp->nranks - 1) {
          xfer_wait_ge(&hp->mail[hp->rank]->dhalo[side], dhalo_seq(S, step - 1), S);
          fence_proxy_async_global();
        }
      }
      mbar_arrive_expect_tx(&sm.bar[si], rown ? DB + (LAST ? 3 : 2) * IB : DB);
      tma_load_3d(&sm.d[si][0][0], map_d, &sm.bar[si], t.k0 - 3 + COFF, t.j0 - 1, zp + il + 1);
      if (rown) {
        tma_load_3d(&sm.res[si][0][0], &T.res_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, zp + il + 1);
        tma_load_3d(&sm.x[si][0][0], &T.x_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, zp + il + 1);
        if (LAST) tma_load_3d(&sm.r[si][0][0], &T.r_i, &sm.bar[si], t.k0 - 1 + COFF, t.j0, zp + il + 1);
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
  if (A.predicated && S->stop) return;
  const double c1 = A.c1[step], c2 = A.c2[step];
  if (threadIdx.x == 0)
    for (int s = 0; s < NS_C - 2; s++) issue();
  const double2 Z2 = make_double2(0.0, 0.0);
  double2 dm[RPW], dc[RPW], dn[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) dm[e] = dc[e] = dn[e] = Z2;
  double acc = 0.0;
  double *g_d = A.d[src ^ 1] + vo + (long long)(t.c0 + 1) * PL;  // + rowoff[e]: plane c0
  double *dlo = (hp && !LAST) ? hp->d_lo[src ^ 1] : nullptr, *dhi = (hp && !LAST) ? hp->d_hi[src ^ 1] : nullptr;
  if (dlo) dlo += (long long)hp->nr_lo * PL;
  if (dhi) dhi -= (long long)G.nr_loc * PL;
  const bool edge_blk = hp && !LAST && (t.c0 == 0 || t.c1 == G.nr_loc);
  double *g_res = A.res + vo + (long long)(t.c0 + 1) * PL;
  double *g_x = (LAST ? A.z : A.x) + vo + (long long)(t.c0 + 1) * PL;
  int st = 0, so = NS_C - 1;
  unsigned ph = 0;
  auto st2 = [&](double *a, double2 v) {  // interior store (res, z_k: no ghost columns)
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
    for (int e = 0; e < RPW; e++) dn[e] = *reinterpret_cast<const double2 *>(&sm.d[st][t.row[e]][cs]);
    if (q >= 2) {
      const double *sb = &sm.d[so][0][0];
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        if (!t.stencil[e]) continue;
        const int r = t.row[e];
        const double *sr = sb + r * SROW + cs;
        const double2 up = (RPW == 2 && e == 1) ? dc[0] : *reinterpret_cast<const double2 *>(sr - SROW);
        const double2 dw = (RPW == 2 && e == 0) ? dc[RPW - 1] : *reinterpret_cast<const double2 *>(sr + SROW);
        const double lf = sr[-1], rt = sr[2];
        const double q0 = stencil7(dc[e].x, dn[e].x, dm[e].x, dw.x, up.x, dc[e].y, lf, dp.x, ap.x, am.x, P, rw[e]);
        const double q1 = stencil7(dc[e].y, dn[e].y, dm[e].y, dw.y, up.y, rt, dc[e].x, dp.y, ap.y, am.y, P, rw[e]);
        const DiagRow d = diag_row(P, rw[e]);
        const double d0 = diag_at(dp.x, d, ap.x, am.x), d1 = diag_at(dp.y, d, ap.y, am.y);
        const double2 rv = *reinterpret_cast<const double2 *>(&sm.res[so][r - 1][2 * t.lane]);
        const double2 xv = *reinterpret_cast<const double2 *>(&sm.x[so][r - 1][2 * t.lane]);
        double2 resn, dnw, xn;
        resn.x = rv.x - jacobi(q0, d0);
        resn.y = rv.y - jacobi(q1, d1);
        dnw.x = fma(c1, dc[e].x, c2 * resn.x);
        dnw.y = fma(c1, dc[e].y, c2 * resn.y);
        xn.x = xv.x + dnw.x;
        xn.y = xv.y + dnw.y;
        const long long o = t.rowoff[e];
        if (LAST) {
          const double2 rr = *reinterpret_cast<const double2 *>(&sm.r[so][r - 1][2 * t.lane]);
          acc += (m0 ? rr.x * xn.x : 0.0) + (m1 ? rr.y * xn.y : 0.0);
          POT3D_CHK(S, in_range(g_x + o, A.z + vo, (G.nr_loc + 2) * PL), CHK_PASS_STORE);
          store_pair<FAST>(g_x + o, t, G.np, xn, true);  // z: pass A stages it (ghost columns)
        } else {
          POT3D_CHK(S, in_range(g_d + o, A.d[src ^ 1] + vo, (G.nr_loc + 2) * PL), CHK_PASS_STORE);
          store_pair<FAST>(g_d + o, t, G.np, dnw, true);
          if (edge_blk) {
            const int il = t.c0 + q - 2;  // the shell of this store
            double *rem = il == 0 ? dlo : (il == G.nr_loc - 1 ? dhi : nullptr);
            if (rem) store_pair<FAST>(rem + (g_d - (A.d[src ^ 1] + vo)) + o, t, G.np, dnw, false);
          }
          st2(g_res + o, resn);
          st2(g_x + o, xn);
        }
      }
      g_d += PL;
      g_res += PL;
      g_x += PL;
    }
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      dm[e] = dc[e];
      dc[e] = dn[e];
    }
    so = st;
    st = wrap_inc(st, NS_C);
    ph ^= (st == 0);
  }
  if (edge_blk) {  // every edge block's peer stores released, then the last raises the flags
    const unsigned nedge = (unsigned)(gridDim.x * (G.nchunks > 1 ? 2 : 1));
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      if (atomicAdd(&S->counter[4], 1u) == nedge - 1) {
        S->counter[4] = 0u;
        raise_dhalo_flags(hp, dhalo_seq(S, step));
      }
    }
  }
  if (LAST) {
    double v[1] = {acc}, tot[1];
    if (grid_sum<1>(v, A.partials + blockIdx.z * A.pstride, &S->counter[2], sred, tot, pass_bid(G), pass_nb(G)) &&
        threadIdx.x == 0) {
      if (A.finalize)
        finalize_rho(S, tot[0]);
      else if (A.peers)  // the same slot and sequence as the PC2 sweeps' r.z
        mail_post(A.peers, MAIL_C, tot[0], 0.0, mail_seq(S->epoch, S->iter), S);
      else
        A.local_sum[0] = tot[0];
    }
  }
}

#define POT3D_POLY(LAST)                                        \
  __shared__ PassShared sh;                                     \
  if (tile_fast(A.G))                                           \
    poly_step_body<LAST, true>(T, A, step, sh);                 \
  else                                                          \
    poly_step_body<LAST, false>(T, A, step, sh)

__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_poly_step(const __grid_constant__ PolyMaps T, PolyArgs A, int step) {
  POT3D_POLY(false);
}
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_poly_last(const __grid_constant__ PolyMaps T, PolyArgs A, int step) {
  POT3D_POLY(true);
}

}  // namespace pot3d
