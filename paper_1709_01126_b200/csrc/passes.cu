// passes.cu -- the two fused sm_100a passes of one PCG iteration (SURVEY.md
// §8(a) rows a3, a7, a8).
//
//   pass A (k_pass_a_*):  p_k = z + beta p_{k-1}  (PC1: z = D^-1 r on the fly)
//                          q   = A p_k            (7-point flux form, A1-A7)
//                          sigma_partial = p_k . q                     [24 B/cell]
//   pass B (k_pass_b_*):  q = A p_k (recomputed: cheaper than storing q)
//                          x += alpha p_k;  r -= alpha q
//                          PC1: z = D^-1 r, partials r.z, r.r  [40 B/cell]
//
// Both march along r through a TJ x TK theta-phi tile (2.5-D blocking).  For
// every plane one elected thread loads the haloed box (TR rows x SROW columns,
// i.e. one halo row above/below and the halo columns left/right -- the
// periodic wrap neighbours come with the physical ghost columns) with a TMA
// tensor copy (cp.async.bulk.tensor) into an NS-stage shared ring completed on
// an mbarrier; rows outside the grid are zero-filled by the TMA unit.  Each
// lane owns RPW rows x 2 phi-adjacent cells.  Pass A turns each staged plane
// into p_k in a 2-slot shared ring; the r neighbours of a cell stay in its
// thread's registers.  One __syncthreads per plane (it also frees the stage
// the producer refills).  Per-block partials are reduced deterministically.
#include "device_common.cuh"

namespace pot3d {

struct SmemA {
  double r[NS_A][TR][SROW];   // staged r (PC1) / z (PC2) / final p on ghost shells
  double p[NS_A][TR][SROW];   // staged p_{k-1}
  double pn[2][TR][SROW];     // p_k of the current / next plane
  uint64_t bar[NS_A];
};
struct SmemB {
  double pn[NS_B][TR][SROW];  // staged p_k
  double r[NS_B][TJ][TK];     // staged r (interior rows)
  double x[NS_B][TJ][TK];     // staged x (interior rows)
  uint64_t bar[NS_B];
};
static_assert(sizeof(SmemA) <= SMEM_A, "SMEM_A");
static_assert(sizeof(SmemB) <= SMEM_B, "SMEM_B");
static_assert((TR * SROW * 8) % 128 == 0 && (TJ * TK * 8) % 128 == 0, "TMA boxes 128-B aligned");
static_assert(TR % RPW == 0, "rows per warp");

__device__ __forceinline__ void chunk_bounds(const Grid &G, int c, int &c0, int &c1) {
  int base = G.nr_loc / G.nchunks, rem = G.nr_loc % G.nchunks;
  c0 = c * base + (c < rem ? c : rem);
  c1 = c0 + base + (c < rem ? 1 : 0);
}

// Metric factors of the tile staged once per block: per smem column slot s
// (logical column k0-2+s, periodic) dp, app, apm, and per haloed row r
// (theta row j0-1+r) g, atp, atm, q.
struct TileConst {
  double dp[SROW], app[SROW], apm[SROW];
  double g[TR], atp[TR], atm[TR], q[TR];
};

__device__ __forceinline__ void load_tile_const(TileConst &tc, const Grid &G, const Metrics &M,
                                                int j0, int k0) {
  for (int s = threadIdx.x; s < SROW; s += blockDim.x) {
    int k = k0 - 2 + s;
    k = (k < 0) ? k + G.np : k;
    k = (k >= G.np) ? (k - G.np) % G.np : k;
    tc.dp[s] = __ldg(M.dp + k);
    tc.app[s] = __ldg(M.app + k);
    tc.apm[s] = __ldg(M.apm + k);
  }
  for (int r = threadIdx.x; r < TR; r += blockDim.x) {
    int j = min(max(j0 - 1 + r, 0), G.nt - 1);
    tc.g[r] = __ldg(M.g + j);
    tc.atp[r] = __ldg(M.atp + j);
    tc.atm[r] = __ldg(M.atm + j);
    tc.q[r] = __ldg(M.q + j);
  }
}

__device__ __forceinline__ RowC row_tc(const TileConst &tc, int r) {
  RowC c;
  c.g = tc.g[r];
  c.atp = tc.atp[r];
  c.atm = tc.atm[r];
  c.q = tc.q[r];
  return c;
}

// Per-plane r metric factors through pointers advanced one shell per plane
// (the metric arrays carry one padding entry on each side for ghost shells).
struct PlanePtr {
  const double *arp, *arm, *dr, *ss;
  __device__ __forceinline__ PlaneC get() const {
    PlaneC c;
    c.arp = __ldg(arp);
    c.arm = __ldg(arm);
    c.dr = __ldg(dr);
    c.ss = __ldg(ss);
    return c;
  }
  __device__ __forceinline__ void next() { ++arp; ++arm; ++dr; ++ss; }
};
__device__ __forceinline__ PlanePtr plane_ptr(const Metrics &M, int ig) {
  PlanePtr p;
  p.arp = M.arp + ig;
  p.arm = M.arm + ig;
  p.dr = M.dr + ig;
  p.ss = M.ss + ig;
  return p;
}

__device__ __forceinline__ int wrap_inc(int s, int n) { return (s + 1 == n) ? 0 : s + 1; }

// (A p)_m = dp_k [g_j (arp (c - p_{i+1}) + arm (c - p_{i-1}) + ss c) + dr (atp (c - p_{j+1})
//           + atm (c - p_{j-1}))] + dr q_j (app (c - p_{k+1}) + apm (c - p_{k-1}))
__device__ __forceinline__ double stencil7(double c, double ip, double im, double jp, double jm,
                                           double kp, double km, double dpk, double appk,
                                           double apmk, const PlaneC &P, const RowC &R) {
  return dpk * (R.g * (P.arp * (c - ip) + P.arm * (c - im) + P.ss * c) +
                P.dr * (R.atp * (c - jp) + R.atm * (c - jm))) +
         P.dr * R.q * (appk * (c - kp) + apmk * (c - km));
}

// Per-thread geometry of a tile.
struct TileThread {
  int lane, w;
  int j0, k0, c0, c1;
  int k;
  bool kv0, kv1;
  int row[RPW];          // haloed rows w*RPW + e
  bool stencil[RPW];     // interior row inside the grid
  long long rowoff[RPW]; // j*PK + k + COFF (clamped)
  bool gl0, gr0, gr1;    // element holds logical k = np-1 (left ghost dup) / k = 0 (right ghost dup)
};

__device__ __forceinline__ TileThread tile_thread(const Grid &G) {
  TileThread t;
  t.lane = threadIdx.x & 31;
  t.w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  t.j0 = (tile % G.ntj) * TJ;
  t.k0 = (tile / G.ntj) * TK;
  chunk_bounds(G, blockIdx.y, t.c0, t.c1);
  t.k = t.k0 + 2 * t.lane;
  t.kv0 = t.k < G.np;
  t.kv1 = (t.k + 1) < G.np;
#pragma unroll
  for (int e = 0; e < RPW; e++) {
    const int r = RPW * t.w + e;
    const int j = t.j0 - 1 + r;
    const bool jv = (j >= 0) && (j < G.nt);
    t.row[e] = r;
    t.stencil[e] = (r >= 1) && (r <= TJ) && jv;
    t.rowoff[e] = (long long)(jv ? j : 0) * G.PK + (t.kv0 ? t.k : 0) + COFF;
  }
  t.gr0 = (t.k == 0);            // element 0 is k = 0: also store at physical np+2
  t.gl0 = (t.k == G.np - 1);     // element 0 is k = np-1: also store at physical 1
  t.gr1 = (t.k + 1 == G.np - 1); // element 1 is k = np-1
  return t;
}

// stores of a p / r pair with the periodic ghost-column duplicates
__device__ __forceinline__ void store_pair(double *row_k, const TileThread &t, int np, double2 v,
                                           bool streaming) {
  // row_k points at physical column of logical k (element 0)
  if (t.kv1) {
    if (streaming)
      __stcs(reinterpret_cast<double2 *>(row_k), v);
    else
      *reinterpret_cast<double2 *>(row_k) = v;
  } else if (t.kv0) {
    row_k[0] = v.x;
  }
  if (t.gr0) row_k[np] = v.x;                 // logical k=0 -> physical np+2
  if (t.gl0) row_k[-np] = v.x;                // logical np-1 -> physical 1
  if (t.gr1) row_k[1 - np] = v.y;             // logical np-1 (element 1) -> physical 1
}

// ---------------------------------------------------------------------------
// pass A
// ---------------------------------------------------------------------------
template <bool USE_Z>
__device__ __forceinline__ void pass_a_body(const TMaps &T, const PassArgs &A, int parity) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  if (S->stop) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemA &sm = *reinterpret_cast<SmemA *>(smem_raw);
  __shared__ double sred[NTHREADS / 32];
  __shared__ TileConst tcs;

  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.j0, t.k0);
  const int cs = 2 + 2 * t.lane;  // smem column slot of element 0
  const double beta = S->beta;
  const long long PL = G.plane;
  const void *map_src = &T.src_h;
  const void *map_old = &T.p_h[parity];
  const void *map_new = &T.p_h[parity ^ 1];
  constexpr unsigned STAGE_BYTES = 2u * TR * SROW * 8u;

  // producer (thread 0): plane q (il = c0-1+q) -> stage q % NS_A
  int qi = 0, si = 0;
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      const bool ghost = (il < 0) || (il >= G.nr_loc);  // ghost shells hold the final p_k
      mbar_arrive_expect_tx(&sm.bar[si], STAGE_BYTES);
      tma_load_3d(&sm.r[si][0][0], ghost ? map_new : map_src, &sm.bar[si], t.k0, t.j0 - 1, il + 1);
      // p_{k-1} on a ghost shell is not used: an out-of-range shell zero-fills the stage
      tma_load_3d(&sm.p[si][0][0], map_old, &sm.bar[si], t.k0, t.j0 - 1, ghost ? G.nr_loc + 2 : il + 1);
    }
    ++qi;
    si = wrap_inc(si, NS_A);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS_A; s++) mbar_init(&sm.bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NS_A - 1; s++) issue();

  const double2 Z2 = make_double2(0.0, 0.0);
  double2 pm[RPW], pc[RPW], pn[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) pm[e] = pc[e] = pn[e] = Z2;
  double *g_pn = A.p_new + (long long)(t.c0 + 1) * PL;  // + rowoff[e]: p_k at plane c0
  const double m0 = t.kv0 ? 1.0 : 0.0, m1 = t.kv1 ? 1.0 : 0.0;
  PlanePtr pp = plane_ptr(M, G.i0 + t.c0 - 1);  // metrics of the transformed plane
  PlanePtr ps = plane_ptr(M, G.i0 + t.c0);      // metrics of the stencil plane
  const bool hl = (t.lane == 0), hr = (t.lane == 31);  // halo-column duty (s = 1 / TK+2)
  const int hs = hl ? 1 : TK + 2;
  double acc = 0.0;
  int st = 0;
  unsigned ph = 0;  // mbarrier parity of stage st

#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    __syncthreads();  // stage (q-1)%NS_A and slot (q&1) are free
    if (threadIdx.x == 0) issue();
    const int il = t.c0 - 1 + q;
    const bool ghost = (il < 0) || (il >= G.nr_loc);
    const bool own = (q >= 1) && (q <= L);
    const int sl = q & 1;
    const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
    const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
    const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
    const double dph = tcs.dp[hs], sph = tcs.app[hs] + tcs.apm[hs];
    PlaneC P = pp.get();
    mbar_wait(&sm.bar[st], ph);
    // ---- transform plane il -> p_k ----
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      const int r = t.row[e];
      const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[st][r][cs]);
      const double2 pv = *reinterpret_cast<const double2 *>(&sm.p[st][r][cs]);
      const RowC R = row_tc(tcs, r);
      if (USE_Z) {
        pn[e].x = fma(beta, pv.x, rv.x);  // ghost shells: pv = 0 -> pn = rv (final p_k)
        pn[e].y = fma(beta, pv.y, rv.y);
      } else {
        const DiagRow d = diag_row(P, R);
        const double2 t2 = make_double2(fdiv(rv.x, dp.x * d.a + d.b * (ap.x + am.x)) + beta * pv.x,
                                        fdiv(rv.y, dp.y * d.a + d.b * (ap.y + am.y)) + beta * pv.y);
        pn[e] = ghost ? rv : t2;
      }
      if (hl || hr) {
        const double hv = sm.r[st][r][hs], hp = sm.p[st][r][hs];
        double v;
        if (USE_Z) {
          v = fma(beta, hp, hv);
        } else {
          const DiagRow d = diag_row(P, R);
          v = ghost ? hv : fdiv(hv, dph * d.a + d.b * sph) + beta * hp;
        }
        sm.pn[sl][r][hs] = v;
      }
      *reinterpret_cast<double2 *>(&sm.pn[sl][r][cs]) = pn[e];
      if (own && t.stencil[e]) store_pair(g_pn + t.rowoff[e], t, G.np, pn[e], false);
    }
    // ---- stencil of plane il-1 (its slot was completed before this barrier) ----
    if (q >= 2) {
      const PlaneC Ps = ps.get();
      const double *sb = &sm.pn[sl ^ 1][0][0];
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        if (!t.stencil[e]) continue;
        const int r = t.row[e];
        const RowC rw = row_tc(tcs, r);
        const double *so = sb + r * SROW + cs;
        const double2 up = (RPW == 2 && e == 1) ? pc[0] : *reinterpret_cast<const double2 *>(so - SROW);
        const double2 dn = (RPW == 2 && e == 0) ? pc[RPW - 1] : *reinterpret_cast<const double2 *>(so + SROW);
        const double lf = so[-1], rt = so[2];
        const double q0 = stencil7(pc[e].x, pn[e].x, pm[e].x, dn.x, up.x, pc[e].y, lf, dp.x, ap.x, am.x, Ps, rw);
        const double q1 = stencil7(pc[e].y, pn[e].y, pm[e].y, dn.y, up.y, rt, pc[e].x, dp.y, ap.y, am.y, Ps, rw);
        acc = fma(m0 * pc[e].x, q0, acc);
        acc = fma(m1 * pc[e].y, q1, acc);
      }
      ps.next();
    }
    pp.next();
    if (own) g_pn += PL;
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      pm[e] = pc[e];
      pc[e] = pn[e];
    }
    st = wrap_inc(st, NS_A);
    ph ^= (st == 0);
  }

  double v[1] = {acc}, tot[1];
  if (grid_sum<1>(v, A.partials, &S->counter[0], sred, tot) && threadIdx.x == 0) {
    if (A.finalize)
      finalize_alpha(S, tot[0]);
    else
      A.local_sum[0] = tot[0];
  }
}

// ---------------------------------------------------------------------------
// pass B
// ---------------------------------------------------------------------------
template <bool USE_Z>
__device__ __forceinline__ void pass_b_body(const TMaps &T, const PassArgs &A, int parity) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  if (S->stop) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemB &sm = *reinterpret_cast<SmemB *>(smem_raw);
  __shared__ double sred[2 * NTHREADS / 32];
  __shared__ TileConst tcs;

  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.j0, t.k0);
  const int cs = 2 + 2 * t.lane;
  const double alpha = S->alpha;
  const long long PL = G.plane;
  const void *map_p = &T.p_h[parity ^ 1];
  const void *map_r = &T.r_i;
  const void *map_x = &T.x_i;
  constexpr unsigned PB = TR * SROW * 8u, RB = TJ * TK * 8u;

  int qi = 0, si = 0;
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      const bool rown = (qi >= 1) && (qi <= L);
      mbar_arrive_expect_tx(&sm.bar[si], rown ? PB + 2 * RB : PB);
      tma_load_3d(&sm.pn[si][0][0], map_p, &sm.bar[si], t.k0, t.j0 - 1, il + 1);
      if (rown) {
        tma_load_3d(&sm.r[si][0][0], map_r, &sm.bar[si], t.k0 + COFF, t.j0, il + 1);
        tma_load_3d(&sm.x[si][0][0], map_x, &sm.bar[si], t.k0 + COFF, t.j0, il + 1);
      }
    }
    ++qi;
    si = wrap_inc(si, NS_B);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS_B; s++) mbar_init(&sm.bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NS_B - 2; s++) issue();

  const double2 Z2 = make_double2(0.0, 0.0);
  double2 pm[RPW], pc[RPW], pn[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) pm[e] = pc[e] = pn[e] = Z2;
  double acc_rz = 0.0, acc_rr = 0.0;
  const double m0 = t.kv0 ? 1.0 : 0.0, m1 = t.kv1 ? 1.0 : 0.0;
  double *g_w = A.r_out + (long long)(t.c0 + 1) * PL;  // + rowoff[e]: r of plane c0
  double *g_x = A.x + (long long)(t.c0 + 1) * PL;      // + rowoff[e]: x of plane c0
  PlanePtr ps = plane_ptr(M, G.i0 + t.c0);             // metrics of the stencil plane
  int st = 0, so = NS_B - 1;                           // stages of planes q and q-1
  unsigned ph = 0;

#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    __syncthreads();  // stage (q-2)%NS_B is free
    if (threadIdx.x == 0) issue();
    const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
    const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
    const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
    PlaneC P;
    if (q >= 2) P = ps.get();
    mbar_wait(&sm.bar[st], ph);
#pragma unroll
    for (int e = 0; e < RPW; e++) pn[e] = *reinterpret_cast<const double2 *>(&sm.pn[st][t.row[e]][cs]);
    if (q >= 2) {
      const double *sb = &sm.pn[so][0][0];
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        if (!t.stencil[e]) continue;
        const int r = t.row[e];
        const RowC rw = row_tc(tcs, r);
        const double *sr = sb + r * SROW + cs;
        const double2 up = (RPW == 2 && e == 1) ? pc[0] : *reinterpret_cast<const double2 *>(sr - SROW);
        const double2 dn = (RPW == 2 && e == 0) ? pc[RPW - 1] : *reinterpret_cast<const double2 *>(sr + SROW);
        const double lf = sr[-1], rt = sr[2];
        const double q0 = stencil7(pc[e].x, pn[e].x, pm[e].x, dn.x, up.x, pc[e].y, lf, dp.x, ap.x, am.x, P, rw);
        const double q1 = stencil7(pc[e].y, pn[e].y, pm[e].y, dn.y, up.y, rt, pc[e].x, dp.y, ap.y, am.y, P, rw);
        const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[so][r - 1][2 * t.lane]);
        double2 rn;
        rn.x = fma(-alpha, q0, rv.x);
        rn.y = fma(-alpha, q1, rv.y);
        if (USE_Z) {
          acc_rr = fma(m0 * rn.x, rn.x, acc_rr);
          acc_rr = fma(m1 * rn.y, rn.y, acc_rr);
        } else {
          const DiagRow d = diag_row(P, rw);
          const double z0 = fdiv(rn.x, dp.x * d.a + d.b * (ap.x + am.x));
          const double z1 = fdiv(rn.y, dp.y * d.a + d.b * (ap.y + am.y));
          acc_rz = fma(m0 * rn.x, z0, acc_rz);
          acc_rz = fma(m1 * rn.y, z1, acc_rz);
          acc_rr = fma(m0 * rn.x, rn.x, acc_rr);
          acc_rr = fma(m1 * rn.y, rn.y, acc_rr);
        }
        store_pair(g_w + t.rowoff[e], t, G.np, rn, true);
        const double2 xv = *reinterpret_cast<const double2 *>(&sm.x[so][r - 1][2 * t.lane]);
        const double2 xn = make_double2(fma(alpha, pc[e].x, xv.x), fma(alpha, pc[e].y, xv.y));
        if (t.kv1)
          __stcs(reinterpret_cast<double2 *>(g_x + t.rowoff[e]), xn);
        else if (t.kv0)
          g_x[t.rowoff[e]] = xn.x;
      }
      ps.next();
      g_w += PL;
      g_x += PL;
    }
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      pm[e] = pc[e];
      pc[e] = pn[e];
    }
    so = st;
    st = wrap_inc(st, NS_B);
    ph ^= (st == 0);
  }

  double v[2] = {acc_rz, acc_rr}, tot[2];
  if (grid_sum<2>(v, A.partials, &S->counter[1], sred, tot) && threadIdx.x == 0) {
    if (A.finalize) {
      if (USE_Z)
        finalize_rr(S, tot[1], A.hist);  // PC2: rho' comes from the sweeps
      else
        finalize_beta(S, tot[0], tot[1], A.hist);
    } else {
      A.local_sum[0] = tot[0];
      A.local_sum[1] = tot[1];
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_a_pc1(const __grid_constant__ TMaps T, PassArgs A, int parity) { pass_a_body<false>(T, A, parity); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_a_pc2(const __grid_constant__ TMaps T, PassArgs A, int parity) { pass_a_body<true>(T, A, parity); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_b_pc1(const __grid_constant__ TMaps T, PassArgs A, int parity) { pass_b_body<false>(T, A, parity); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_b_pc2(const __grid_constant__ TMaps T, PassArgs A, int parity) { pass_b_body<true>(T, A, parity); }

// ghost columns of shells [il0, il0 + n): physical 1 <- k = np-1, physical np+2 <- k = 0
__global__ void k_fix_ghost_cols(Grid G, double *a, int il0, int n) {
  const long long rows = (long long)n * G.nt;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < rows;
       c += (long long)gridDim.x * blockDim.x) {
    const int il = il0 + (int)(c / G.nt), j = (int)(c % G.nt);
    double *row = a + cidx(G, il, j, 0);
    const double v0 = row[0], vl = row[G.np - 1];
    row[-1] = vl;
    row[G.np] = v0;
  }
}

}  // namespace pot3d
