// passes.cu -- the two fused sm_100a passes of one PCG iteration (SURVEY.md
// §8(a) rows a3, a7, a8).
//
//   pass A (k_pass_a_*):  p_k = z + beta p_{k-1}  (PC1: z = D^-1 r on the fly)
//                          q   = A p_k            (7-point flux form, A1-A7)
//                          sigma_partial = p_k . q
//                          x  += alpha_{k-1} p_{k-1}   (lazy x update)
//   pass B (k_pass_b_*):  q = A p_k (recomputed: cheaper than storing q)
//                          r -= alpha q;  PC1: z = D^-1 r, partials r.z, r.r
//
// Both march along r through a TJ x TK theta-phi tile (2.5-D blocking).  The
// input planes of the tile (with one halo row above/below and one halo column
// left/right, the periodic phi wrap resolved by index) stream through a
// multi-stage cp.async (LDGSTS) ring in shared memory with zero-fill for
// everything outside the grid, so the loads in flight cost no registers.
// Pass A turns each staged plane into p_k in a 2-slot shared ring; the r
// neighbours of a cell stay in its thread's registers.  One __syncthreads per
// plane.  The per-block partials are reduced deterministically (a6).
#include "device_common.cuh"

namespace pot3d {

struct SmemA {
  double r[NS_A][TR][SROW];   // staged r (PC1) / z (PC2) / final p on ghost shells
  double p[NS_A][TR][SROW];   // staged p_{k-1}
  double pn[2][TR][SROW];     // p_k of the current / next plane
};
struct SmemB {
  double pn[NS_B][TR][SROW];  // staged p_k
  double r[NS_B][TJ][TK];     // staged r (interior rows)
};
static_assert(sizeof(SmemA) == SMEM_A, "SMEM_A");
static_assert(sizeof(SmemB) == SMEM_B, "SMEM_B");

__device__ __forceinline__ void chunk_bounds(const Grid &G, int c, int &c0, int &c1) {
  int base = G.nr_loc / G.nchunks, rem = G.nr_loc % G.nchunks;
  c0 = c * base + (c < rem ? c : rem);
  c1 = c0 + base + (c < rem ? 1 : 0);
}

// Per-thread geometry of a tile (shared by both passes).
struct TileThread {
  int lane, w;       // w = haloed row 0..TR-1
  int j0, k0, c0, c1;
  int j, k, kend;
  bool jv, kv0, kv1, stencil;   // stencil: interior row inside the grid
  int nbytes;                   // own item bytes (0 / 8 / 16)
  long long rowoff;             // j*PK + k (clamped)
  bool hduty, hjv;              // halo-column duty (warps 0 / TR-1, lanes < TJ)
  int hrow, hpos, hcol, hj;
  long long hoff;
};

__device__ __forceinline__ TileThread tile_thread(const Grid &G) {
  TileThread t;
  t.lane = threadIdx.x & 31;
  t.w = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  t.j0 = (tile % G.ntj) * TJ;
  t.k0 = (tile / G.ntj) * TK;
  chunk_bounds(G, blockIdx.y, t.c0, t.c1);
  t.j = t.j0 - 1 + t.w;
  t.jv = (t.j >= 0) && (t.j < G.nt);
  t.k = t.k0 + 2 * t.lane;
  t.kv0 = t.k < G.np;
  t.kv1 = (t.k + 1) < G.np;
  t.kend = min(t.k0 + TK, G.np);
  t.stencil = (t.w >= 1) && (t.w <= TJ) && t.jv;
  t.nbytes = (t.jv && t.kv0) ? (t.kv1 ? 16 : 8) : 0;
  t.rowoff = (long long)(t.jv ? t.j : 0) * G.PK + (t.kv0 ? t.k : 0);
  t.hduty = (t.w == 0 || t.w == TR - 1) && (t.lane < TJ);
  t.hrow = t.lane + 1;
  t.hj = t.j0 + t.lane;
  t.hjv = t.hduty && (t.hj < G.nt);
  t.hcol = (t.w == 0) ? (t.k0 == 0 ? G.np - 1 : t.k0 - 1) : (t.kend == G.np ? 0 : t.kend);
  t.hpos = (t.w == 0) ? 1 : TK + 2;
  t.hoff = (long long)(t.hjv ? t.hj : 0) * G.PK + t.hcol;
  return t;
}

// Metric factors of the tile staged once per block: per smem column slot
// s (column k0-2+s) dp, app, apm, and per haloed row w (theta row j0-1+w)
// g, atp, atm, q.  Keeps them out of the register file.
struct TileConst {
  double dp[SROW], app[SROW], apm[SROW];
  double g[TR], atp[TR], atm[TR], q[TR];
};

__device__ __forceinline__ void load_tile_const(TileConst &tc, const Grid &G, const Metrics &M,
                                                int j0, int k0) {
  for (int s = threadIdx.x; s < SROW; s += blockDim.x) {
    int k = k0 - 2 + s;
    k = (k < 0) ? k + G.np : k;                 // left halo of the first tile wraps
    k = (k >= G.np) ? (k - G.np) % G.np : k;    // pads / right wrap (values unused for pads)
    tc.dp[s] = __ldg(M.dp + k);
    tc.app[s] = __ldg(M.app + k);
    tc.apm[s] = __ldg(M.apm + k);
  }
  for (int w = threadIdx.x; w < TR; w += blockDim.x) {
    int j = min(max(j0 - 1 + w, 0), G.nt - 1);
    tc.g[w] = __ldg(M.g + j);
    tc.atp[w] = __ldg(M.atp + j);
    tc.atm[w] = __ldg(M.atm + j);
    tc.q[w] = __ldg(M.q + j);
  }
}

__device__ __forceinline__ RowC row_tc(const TileConst &tc, int w) {
  RowC r;
  r.g = tc.g[w];
  r.atp = tc.atp[w];
  r.atm = tc.atm[w];
  r.q = tc.q[w];
  return r;
}

// (A p)_m = dp_k [g_j (arp (c - p_{i+1}) + arm (c - p_{i-1}) + ss c) + dr (atp (c - p_{j+1})
//           + atm (c - p_{j-1}))] + dr q_j (app (c - p_{k+1}) + apm (c - p_{k-1}))
__device__ __forceinline__ double stencil7(double c, double ip, double im, double jp, double jm,
                                           double kp, double km, double dpk, double appk,
                                           double apmk, const PlaneC &P, const RowC &R) {
  return dpk * (R.g * (P.arp * (c - ip) + P.arm * (c - im) + P.ss * c) +
                P.dr * (R.atp * (c - jp) + R.atm * (c - jm))) +
         P.dr * R.q * (appk * (c - kp) + apmk * (c - km));
}

// ---------------------------------------------------------------------------
// pass A
// ---------------------------------------------------------------------------
template <bool USE_Z>
__device__ __forceinline__ void pass_a_body(const PassArgs &A) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  if (S->stop) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemA &sm = *reinterpret_cast<SmemA *>(smem_raw);
  __shared__ double sred[NTHREADS / 32];

  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;
  const double *src = USE_Z ? A.z : A.r;

  auto issue = [&](int q) {
    const int il = t.c0 - 1 + q;
    if (il <= t.c1) {
      const bool ghost = (il < 0) || (il >= G.nr_loc);
      const long long pb = (long long)(il + 1) * G.plane;
      const int st = q % NS_A;
      const double *s1 = ghost ? A.p_new : src;  // ghost shells hold the final p_k (halo)
      cp_async16(&sm.r[st][t.w][2 + 2 * t.lane], s1 + pb + t.rowoff, t.nbytes);
      cp_async16(&sm.p[st][t.w][2 + 2 * t.lane], A.p_old + pb + t.rowoff, ghost ? 0 : t.nbytes);
      if (t.hduty) {
        cp_async8(&sm.r[st][t.hrow][t.hpos], s1 + pb + t.hoff, t.hjv ? 8 : 0);
        cp_async8(&sm.p[st][t.hrow][t.hpos], A.p_old + pb + t.hoff, (t.hjv && !ghost) ? 8 : 0);
      }
    }
    cp_async_commit();
  };

  __shared__ TileConst tcs;
  load_tile_const(tcs, G, M, t.j0, t.k0);
  const int cs = 2 + 2 * t.lane;  // smem column slot of element 0
  const double beta = S->beta;
  const double alpha_prev = S->alpha_prev;

#pragma unroll 1
  for (int q = 0; q < NS_A - 1; q++) issue(q);

  double2 pm = make_double2(0.0, 0.0), pc = pm, pn = pm;
  double2 xnext = pm;
  const bool xown = t.stencil && t.kv0;
  if (xown && L > 0) xnext = *reinterpret_cast<const double2 *>(A.x + (long long)(t.c0 + 1) * G.plane + t.rowoff);
  double acc = 0.0;

#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    cp_async_wait<NS_A - 2>();
    __syncthreads();
    issue(q + NS_A - 1);
    const int il = t.c0 - 1 + q;
    const bool ghost = (il < 0) || (il >= G.nr_loc);
    const bool own = (il >= t.c0) && (il < t.c1);
    const int st = q % NS_A, sl = q & 1;
    // ---- transform plane il -> p_k ----
    const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[st][t.w][2 + 2 * t.lane]);
    double2 xv = xnext;
    if (own && xown && il + 1 < t.c1)
      xnext = *reinterpret_cast<const double2 *>(A.x + (long long)(il + 2) * G.plane + t.rowoff);
    if (ghost) {
      pn = rv;
    } else {
      const double2 pv = *reinterpret_cast<const double2 *>(&sm.p[st][t.w][2 + 2 * t.lane]);
      if (USE_Z) {
        pn.x = rv.x + beta * pv.x;
        pn.y = rv.y + beta * pv.y;
      } else {
        const PlaneC P = plane_c(M, G.i0 + il);
        const DiagRow d = diag_row(P, row_tc(tcs, t.w));
        const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
        const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
        const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
        pn.x = fdiv(rv.x, dp.x * d.a + d.b * (ap.x + am.x)) + beta * pv.x;
        pn.y = fdiv(rv.y, dp.y * d.a + d.b * (ap.y + am.y)) + beta * pv.y;
      }
      if (own && xown) {
        const long long o = (long long)(il + 1) * G.plane + t.rowoff;
        xv.x += alpha_prev * pv.x;
        xv.y += alpha_prev * pv.y;
        if (t.kv1) {
          *reinterpret_cast<double2 *>(A.p_new + o) = pn;
          __stcs(reinterpret_cast<double2 *>(A.x + o), xv);
        } else {
          A.p_new[o] = pn.x;
          A.x[o] = xv.x;
        }
      }
    }
    *reinterpret_cast<double2 *>(&sm.pn[sl][t.w][2 + 2 * t.lane]) = pn;
    if (t.hduty) {
      const double hr = sm.r[st][t.hrow][t.hpos];
      double v;
      if (ghost) {
        v = hr;
      } else {
        const double hp = sm.p[st][t.hrow][t.hpos];
        if (USE_Z) {
          v = hr + beta * hp;
        } else {
          const PlaneC P = plane_c(M, G.i0 + il);
          const DiagRow d = diag_row(P, row_tc(tcs, t.hrow));
          v = fdiv(hr, tcs.dp[t.hpos] * d.a + d.b * (tcs.app[t.hpos] + tcs.apm[t.hpos])) + beta * hp;
        }
      }
      sm.pn[sl][t.hrow][t.hpos] = v;
    }
    // ---- stencil of plane il-1 (slot written before this iteration's barrier) ----
    if (q >= 2 && t.stencil) {
      const int is = il - 1;
      const int so = sl ^ 1;
      const PlaneC P = plane_c(M, G.i0 + is);
      const double2 up = *reinterpret_cast<const double2 *>(&sm.pn[so][t.w - 1][2 + 2 * t.lane]);
      const double2 dn = *reinterpret_cast<const double2 *>(&sm.pn[so][t.w + 1][2 + 2 * t.lane]);
      const double lf = sm.pn[so][t.w][1 + 2 * t.lane];
      const double hrt = sm.pn[so][t.w][TK + 2];
      const double rt0 = t.kv1 ? pc.y : hrt;
      const double rt1 = (t.k + 2 < t.kend) ? sm.pn[so][t.w][4 + 2 * t.lane] : hrt;
      const RowC rw = row_tc(tcs, t.w);
      const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
      const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
      const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
      const double q0 = stencil7(pc.x, pn.x, pm.x, dn.x, up.x, rt0, lf, dp.x, ap.x, am.x, P, rw);
      const double q1 = stencil7(pc.y, pn.y, pm.y, dn.y, up.y, rt1, pc.x, dp.y, ap.y, am.y, P, rw);
      if (t.kv0) acc += pc.x * q0;
      if (t.kv1) acc += pc.y * q1;
    }
    pm = pc;
    pc = pn;
  }
  cp_async_wait<0>();

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
__device__ __forceinline__ void pass_b_body(const PassArgs &A) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S;
  if (S->stop) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemB &sm = *reinterpret_cast<SmemB *>(smem_raw);
  __shared__ double sred[2 * NTHREADS / 32];

  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;

  auto issue = [&](int q) {
    const int il = t.c0 - 1 + q;
    if (il <= t.c1) {
      const long long pb = (long long)(il + 1) * G.plane;
      const int st = q % NS_B;
      cp_async16(&sm.pn[st][t.w][2 + 2 * t.lane], A.p_new + pb + t.rowoff, t.nbytes);
      if (t.stencil && il >= t.c0 && il < t.c1)
        cp_async16(&sm.r[st][t.w - 1][2 * t.lane], A.r + pb + t.rowoff, t.nbytes);
      if (t.hduty) cp_async8(&sm.pn[st][t.hrow][t.hpos], A.p_new + pb + t.hoff, t.hjv ? 8 : 0);
    }
    cp_async_commit();
  };

  __shared__ TileConst tcs;
  load_tile_const(tcs, G, M, t.j0, t.k0);
  const int cs = 2 + 2 * t.lane;
  const double alpha = S->alpha;

#pragma unroll 1
  for (int q = 0; q < NS_B - 2; q++) issue(q);

  double2 pm = make_double2(0.0, 0.0), pc = pm, pn = pm;
  double acc_rz = 0.0, acc_rr = 0.0;

#pragma unroll 1
  for (int q = 0; q <= L + 1; q++) {
    cp_async_wait<NS_B - 3>();
    __syncthreads();
    issue(q + NS_B - 2);
    const int st = q % NS_B;
    pn = *reinterpret_cast<const double2 *>(&sm.pn[st][t.w][2 + 2 * t.lane]);
    if (q >= 2 && t.stencil) {
      const int is = t.c0 - 2 + q;
      const int so = (q + NS_B - 1) % NS_B;
      const PlaneC P = plane_c(M, G.i0 + is);
      const double2 up = *reinterpret_cast<const double2 *>(&sm.pn[so][t.w - 1][2 + 2 * t.lane]);
      const double2 dn = *reinterpret_cast<const double2 *>(&sm.pn[so][t.w + 1][2 + 2 * t.lane]);
      const double lf = sm.pn[so][t.w][1 + 2 * t.lane];
      const double hrt = sm.pn[so][t.w][TK + 2];
      const double rt0 = t.kv1 ? pc.y : hrt;
      const double rt1 = (t.k + 2 < t.kend) ? sm.pn[so][t.w][4 + 2 * t.lane] : hrt;
      const RowC rw = row_tc(tcs, t.w);
      const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
      const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
      const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
      const double q0 = stencil7(pc.x, pn.x, pm.x, dn.x, up.x, rt0, lf, dp.x, ap.x, am.x, P, rw);
      const double q1 = stencil7(pc.y, pn.y, pm.y, dn.y, up.y, rt1, pc.x, dp.y, ap.y, am.y, P, rw);
      const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[so][t.w - 1][2 * t.lane]);
      double2 rn;
      rn.x = rv.x - alpha * q0;
      rn.y = rv.y - alpha * q1;
      if (USE_Z) {
        if (t.kv0) acc_rr += rn.x * rn.x;
        if (t.kv1) acc_rr += rn.y * rn.y;
      } else {
        const DiagRow d = diag_row(P, rw);
        const double z0 = fdiv(rn.x, dp.x * d.a + d.b * (ap.x + am.x));
        const double z1 = fdiv(rn.y, dp.y * d.a + d.b * (ap.y + am.y));
        if (t.kv0) {
          acc_rz += rn.x * z0;
          acc_rr += rn.x * rn.x;
        }
        if (t.kv1) {
          acc_rz += rn.y * z1;
          acc_rr += rn.y * rn.y;
        }
      }
      if (t.kv0) {
        const long long o = (long long)(is + 1) * G.plane + t.rowoff;
        if (t.kv1)
          __stcs(reinterpret_cast<double2 *>(A.r_out + o), rn);
        else
          A.r_out[o] = rn.x;
      }
    }
    pm = pc;
    pc = pn;
  }
  cp_async_wait<0>();

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

__global__ void __launch_bounds__(NTHREADS, 2) k_pass_a_pc1(PassArgs A) { pass_a_body<false>(A); }
__global__ void __launch_bounds__(NTHREADS, 2) k_pass_a_pc2(PassArgs A) { pass_a_body<true>(A); }
__global__ void __launch_bounds__(NTHREADS, 2) k_pass_b_pc1(PassArgs A) { pass_b_body<false>(A); }
__global__ void __launch_bounds__(NTHREADS, 2) k_pass_b_pc2(PassArgs A) { pass_b_body<true>(A); }

}  // namespace pot3d
