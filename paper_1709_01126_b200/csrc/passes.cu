// passes.cu -- the two fused sm_100a passes of one PCG iteration (SURVEY.md
// §8(a) rows a3, a7, a8).
//
//   pass A (k_pass_a):    p_k = z + beta p_{k-1}  (z: the stored preconditioned
//                          residual -- PC1 keeps z = D^-1 r itself, PC2 the sweeps' z)
//                          q   = A p_k            (7-point flux form, A1-A7)
//                          sigma_partial = p_k . q                     [24 B/cell]
//   pass B (k_pass_b_*):  q = A p_k (recomputed: cheaper than storing q)
//                          x += alpha p_k
//                          PC1: z -= alpha D^-1 q (= D^-1 (r - alpha q)),
//                               partials r.z = (D z).z, r.r = (D z).(D z)
//                          PC2: r -= alpha q, partial r.r               [40 B/cell]
//
// PC1 stores z = D^-1 r instead of r (reading A22): the recurrence
// r_{k+1} = r_k - alpha q_k premultiplied by D^-1.  Pass A then needs no
// division (p = z + beta p over the haloed box is one fma per cell) and pass B
// divides once per interior cell, where it divided before as well.
//
// Both march along r through a TJ x TK theta-phi tile (2.5-D blocking).  For
// every plane one elected thread loads the haloed box (TR rows x SROW columns:
// one halo row above/below, the halo columns left/right -- the periodic wrap
// neighbours come with the physical ghost columns) with a TMA tensor copy
// (cp.async.bulk.tensor) into a shared ring completed on an mbarrier; rows
// outside the grid are zero-filled by the TMA unit.  Lane l of a warp owns the
// logical columns k0-1+2l and k0+2l of RPW rows, so the halo columns are
// ordinary lane work (lanes 0 and 31) and every shared/global access is
// 128-bit.  Pass A turns each staged plane into p_k in a 3-slot shared ring
// and is unrolled by 3 so stage, slot and register roles are compile-time;
// the r neighbours of a cell stay in its thread's registers.  One
// __syncthreads per plane.  Per-block partials are reduced deterministically.
#include "pass_common.cuh"

// pass A code-generation switches (tuning variants)

#ifndef POT3D_A_FLUX   // pass A shares the r flux between consecutive stencil planes
#define POT3D_A_FLUX 1
#endif

namespace pot3d {

static_assert(NS_A == 3, "pass A is unrolled by its stage count");

struct SmemA {
  double r[NS_A][TR][SROW];   // staged z (PC1: D^-1 r, PC2: the sweeps' z) / final p on ghost shells
  double p[NS_A][TR][SROW];   // staged p_{k-1}
  double pn[3][TR][SROW];     // p_k ring
  uint64_t bar[NS_A];
};
struct SmemB {
  double pn[NS_B][TR][SROW];  // staged p_k
  double r[NS_B][TJ][TKB];    // staged z (PC1) / r (PC2) (interior rows)
  double x[NS_B][TJ][TKB];    // staged x (interior rows)
  uint64_t bar[NS_B];
};
static_assert(sizeof(SmemA) <= SMEM_A, "SMEM_A");
static_assert(sizeof(SmemB) <= SMEM_B, "SMEM_B");
static_assert((TR * SROW * 8) % 128 == 0 && (TJ * TKB * 8) % 128 == 0, "TMA boxes 128-B aligned");
static_assert(TR % RPW == 0 && TKB == 2 * 32 && TK == TKB, "tile geometry");


// ---------------------------------------------------------------------------
// pass A
// ---------------------------------------------------------------------------
template <bool PROBE, bool FAST>
__device__ __forceinline__ void pass_a_body(const TMaps &T, const PassArgs &A, int parity, PassShared &sh) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S + blockIdx.z;  // batch: the right-hand side of this block (pass_common.cuh)
  if (G.role_rows && blockIdx.y == 0) {
    // edge role (peer memory): p_k on the two edge shells, locally and into the
    // neighbours' ghost shells, then the halo flags -- scheduled first, beside the
    // interior chunks; these blocks add nothing to sigma
    double *sred_e = sh.sred;
    pdl_trigger();
    pdl_wait();
    if (S->stop) return;
    const bool last = edge_shells(G, M, S, A.z, A.p_old, A.p_new, A.peers, parity ^ 1, S->beta,
                                  blockIdx.x, gridDim.x);
    if (last && threadIdx.x == 0) {
      S->counter[4] = 0u;
      raise_halo_flags(A.peers, mail_seq(S->epoch, S->iter + 1));
    }
    double v[1] = {0.0}, tot[1];
    if (grid_sum<1>(v, A.partials, &S->counter[0], sred_e, tot, pass_bid(G), pass_nb(G)) && threadIdx.x == 0) {
      trace_mark(S, TR_A1);
      mail_post(A.peers, MAIL_A, tot[0], 0.0, mail_seq(S->epoch, S->iter + 1), S);
    }
    return;
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemA &sm = *reinterpret_cast<SmemA *>(smem_raw);
  double *sred = sh.sred;
  TileConst &tcs = sh.tcs;
  PlaneSm &pls = sh.pls;
  const TileThread t = tile_thread(G);
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.k0);
  const int ig0 = G.i0 + t.c0 - 1;           // global shell of plane q = 0
  load_planes(pls, M, ig0, L + 2);
  const int cs = 2 + 2 * t.lane;  // smem index of element 0
  const long long PL = G.plane;
  const int zp = rhs_planes(G);   // batch: TMA plane offset / element offset of this RHS
  const long long vo = zp * PL;
  const void *map_src = &T.src_h;
  const void *map_old = &T.p_h[parity];
  const void *map_new = &T.p_h[parity ^ 1];
  constexpr unsigned STAGE_BYTES = 2u * TR * SROW * 8u;
  RowC rw[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) rw[e] = row_c(M, min(max(t.j0 - 1 + t.row[e], 0), G.nt - 1));

  // producer (thread 0): plane q (il = c0-1+q) -> stage st
  auto issue = [&](int q, int st) {
    if (q <= L + 1) {
      const int il = t.c0 - 1 + q;
      if ((il < 0) || (il >= G.nr_loc)) {
        // ghost shell: it holds the final p_k (halo / zeros); p_{k-1} is not loaded
        // (a fully out-of-range box is not a reliable zero fill).  With peer
        // memory the neighbour stores it there: wait for its flag of this iteration.
        if (A.peers) {
          const int side = (il < 0) ? 0 : 1;
          if (side == 0 ? A.peers->rank > 0 : A.peers->rank < A.peers->nranks - 1) {
            xfer_wait(&A.peers->mail[A.peers->rank]->halo[side], mail_seq(S->epoch, S->iter + 1), S);
            fence_proxy_async_global();
            trace_max(S, TR_AHALO);
          }
        }
        mbar_arrive_expect_tx(&sm.bar[st], STAGE_BYTES / 2);
        tma_load_3d(&sm.r[st][0][0], map_new, &sm.bar[st], t.k0 - 3 + COFF, t.j0 - 1, zp + il + 1);
      } else {
        mbar_arrive_expect_tx(&sm.bar[st], STAGE_BYTES);
        tma_load_3d(&sm.r[st][0][0], map_src, &sm.bar[st], t.k0 - 3 + COFF, t.j0 - 1, zp + il + 1);
        tma_load_3d(&sm.p[st][0][0], map_old, &sm.bar[st], t.k0 - 3 + COFF, t.j0 - 1, zp + il + 1);
      }
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS_A; s++) mbar_init(&sm.bar[s], 1);
    fence_mbar_init();
  }
  // slot columns 0 and 67 are never produced by the transform (1 and 66, the halo
  // columns, come from lanes 0 and 31); keep every slot column finite
  for (int i = threadIdx.x; i < 3 * TR; i += blockDim.x) {
    double *row = &sm.pn[i / TR][i % TR][0];
    row[0] = row[1] = row[SROW - 2] = row[SROW - 1] = 0.0;
  }
  __syncthreads();
  // everything above reads only launch constants and metrics: with PDL it overlaps
  // the previous kernel's tail; S, r|z and p are read only after the wait
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) trace_mark(A.S, TR_A0);
  const double beta = S->beta;
  double acc = 0.0;
  if (t.valid) {  // a cluster padding block only joins the reduction
    if (threadIdx.x == 0) {
      issue(0, 0);
      issue(1, 1);
    }

    const double2 Z2 = make_double2(0.0, 0.0);
    double2 R[3][RPW];  // p_k of planes q (R[q%3]), q-1, q-2 of this lane's cells
#pragma unroll
    for (int u = 0; u < 3; u++)
#pragma unroll
      for (int e = 0; e < RPW; e++) R[u][e] = Z2;
    double *g_pn = A.p_new + vo + (long long)t.c0 * PL;  // + rowoff[e]: p_k at plane q (il = c0-1+q)
    unsigned ph = 0;  // mbarrier parity of the current group of 3 planes

    // per-thread constants of the stencil: smem offsets of the theta neighbours
    // (clamped on the tile's outer rows, which skip the stencil) and the column masks
    // (FAST tiles: every column is an interior cell)
    int up_off[RPW], dn_off[RPW];
#pragma unroll
    for (int e = 0; e < RPW; e++) {
      const int r = t.row[e];
      up_off[e] = (r == 0) ? 0 : -SROW;
      dn_off[e] = (r == TR - 1) ? 0 : SROW;
    }
    const bool m0 = FAST || t.st0, m1 = FAST || t.st1;
    const bool halo_lane = (t.lane == 0) || (t.lane == 31);
    const int hcol = (t.lane == 0) ? 1 : SROW - 2;  // smem column of this lane's halo column

    // One plane step.  STENCIL = false only for q = 0, 1 (peeled), so the steady
    // state is one basic block: the transform's fp64 chains (plane q) and the
    // stencil of plane q-1 are independent and can be interleaved by the scheduler.
#if POT3D_A_FLUX
    double2 fl[RPW];  // upper r flux arp (c - ip) of the last stencil plane, per row and cell
#endif
    auto step = [&](auto U, auto STENCIL, int q, auto FIRST) {
      constexpr int u = decltype(U)::value;       // stage, slot and register set of plane q
      constexpr bool do_st = decltype(STENCIL)::value;
      constexpr bool first = decltype(FIRST)::value;  // first stencil plane of the chunk
      (void)first;
      constexpr int um = (u + 2) % 3, umm = (u + 1) % 3;
      __syncthreads();  // stage um and slot u are free
      if (threadIdx.x == 0) issue(q + 2, um);
      const int il = t.c0 - 1 + q;
      const bool ghost = (il < 0) || (il >= G.nr_loc);
      const bool store = (q >= 1) && (q <= L);
      const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
      const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
      const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
      const PlaneC Ps = plane_at(pls, do_st ? q - 1 : q);
      mbar_wait(&sm.bar[u], ph);
      // ---- transform plane il -> p_k = z + beta p_{k-1} (ghost shells: the final p_k) ----
#pragma unroll
      for (int e = 0; e < RPW; e++) {
        const int r = t.row[e];
        const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[u][r][cs]);
        const double2 pv = *reinterpret_cast<const double2 *>(&sm.p[u][r][cs]);  // unused on ghosts
        double2 pn;
        pn.x = selp(rv.x, fma(beta, pv.x, rv.x), ghost);
        pn.y = selp(rv.y, fma(beta, pv.y, rv.y), ghost);
        R[u][e] = pn;
        *reinterpret_cast<double2 *>(&sm.pn[u][r][cs]) = pn;
        if (halo_lane) {  // the halo columns k0-2 (lane 0) and k0+63 (lane 31)
          const double hr = sm.r[u][r][hcol], hp = sm.p[u][r][hcol];
          sm.pn[u][r][hcol] = selp(hr, fma(beta, hp, hr), ghost);
        }
        if (store && t.stencil[e]) {
          POT3D_CHK(S, in_range(g_pn + t.rowoff[e], A.p_new + vo, (G.nr_loc + 2) * PL), CHK_PASS_STORE);
          store_pair<FAST>(g_pn + t.rowoff[e], t, G.np, pn, false);
        }
      }
      g_pn += PL;
      // ---- stencil of plane il-1 (its slot was completed before this barrier) ----
      if (do_st) {
        const double *sb = &sm.pn[um][0][0];
        // FAST tiles: the faces between the thread's two rows and two columns, once
        const FaceTerms ft = face_terms(R[um][0], R[um][RPW - 1], rw[0], ap.x);
#pragma unroll
        for (int e = 0; e < RPW; e++) {
          if (!t.stencil[e]) continue;  // halo rows (warp-uniform)
          const int r = t.row[e];
          const double *so = sb + r * SROW + cs;
          const double2 c = R[um][e];
          const double2 up = (RPW == 2 && e == 1) ? R[um][0] : *reinterpret_cast<const double2 *>(so + up_off[e]);
          const double2 dn = (RPW == 2 && e == 0) ? R[um][RPW - 1] : *reinterpret_cast<const double2 *>(so + dn_off[e]);
          const double lf = so[-1], rt = so[2];
#if POT3D_A_FLUX
          // lower r flux: computed on the chunk's first stencil plane, then the negated
          // upper flux of the previous plane
          const double fdx = first ? Ps.arm * (c.x - R[umm][e].x) : -fl[e].x;
          const double fdy = first ? Ps.arm * (c.y - R[umm][e].y) : -fl[e].y;
          double q0, q1;
          if (FAST && RPW == 2) {  // the shared theta / phi faces (face_terms)
            const double pk = e == 0 ? ft.p0 : ft.p1;
            const double2 jo = e == 0 ? up : dn;  // the theta neighbour outside the thread
            const double ajo = e == 0 ? rw[0].atm : rw[RPW - 1].atp;
            q0 = stencil7fs(c.x, R[u][e].x, fdx, e == 0 ? ft.tx : -ft.tx, ajo, jo.x, pk, am.x, lf, dp.x, Ps, rw[e],
                            fl[e].x);
            q1 = stencil7fs(c.y, R[u][e].y, fdy, e == 0 ? ft.ty : -ft.ty, ajo, jo.y, -pk, ap.y, rt, dp.y, Ps, rw[e],
                            fl[e].y);
          } else {
            q0 = stencil7f(c.x, R[u][e].x, fdx, dn.x, up.x, c.y, lf, dp.x, ap.x, am.x, Ps, rw[e], fl[e].x);
            q1 = stencil7f(c.y, R[u][e].y, fdy, dn.y, up.y, rt, c.x, dp.y, ap.y, am.y, Ps, rw[e], fl[e].y);
          }
#else
          const double q0 = stencil7(c.x, R[u][e].x, R[umm][e].x, dn.x, up.x, c.y, lf, dp.x, ap.x, am.x, Ps, rw[e]);
          const double q1 = stencil7(c.y, R[u][e].y, R[umm][e].y, dn.y, up.y, rt, c.x, dp.y, ap.y, am.y, Ps, rw[e]);
#endif
          acc += (m0 ? c.x * q0 : 0.0) + (m1 ? c.y * q1 : 0.0);
          // diagnostic instantiation only (pot3d_apply_fused which = 2): q of plane il-1
          if (PROBE) store_pair<FAST>(A.q_probe + (long long)il * PL + t.rowoff[e], t, G.np, make_double2(q0, q1), false);
        }
      }
    };

    const int last = L + 1;  // >= 2
    step(IC<0>{}, std::false_type{}, 0, std::false_type{});
    step(IC<1>{}, std::false_type{}, 1, std::false_type{});
    step(IC<2>{}, std::true_type{}, 2, std::true_type{});
    ph ^= 1u;
#pragma unroll 1
    for (int q = 3; q <= last; q += 3) {
      step(IC<0>{}, std::true_type{}, q, std::false_type{});
      if (q + 1 > last) break;
      step(IC<1>{}, std::true_type{}, q + 1, std::false_type{});
      if (q + 2 > last) break;
      step(IC<2>{}, std::true_type{}, q + 2, std::false_type{});
      ph ^= 1u;
    }

  }
  double v[1] = {acc}, tot[1];
  if (grid_sum<1>(v, A.partials + blockIdx.z * A.pstride, &S->counter[0], sred, tot, pass_bid(G), pass_nb(G)) &&
      threadIdx.x == 0) {
    trace_max(A.S, TR_A1);  // batch: the end of the last right-hand side
    if (A.finalize)
      finalize_alpha(S, tot[0]);
    else if (A.peers)
      mail_post(A.peers, MAIL_A, tot[0], 0.0, mail_seq(S->epoch, S->iter + 1), S);
    else
      A.local_sum[0] = tot[0];
  }
}

// ---------------------------------------------------------------------------
// pass B
// ---------------------------------------------------------------------------
// USE_Z = false: PC1, the stored vector is z = D^-1 r; true: PC2, the stored vector is r.
// XM (pass_common.cuh): XM_EVERY x += alpha_k p_k (PC2); PC1 XM_SKIP on even iterations
// (x untouched, 24 B/cell) and XM_PAIR on odd ones (40 B/cell): 32 B/cell on average.
template <bool USE_Z, int XM, bool FAST>
__device__ __forceinline__ void pass_b_body(const TMaps &T, const PassArgs &A, int parity, PassShared &sh) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  Scalars *S = A.S + blockIdx.z;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SmemB &sm = *reinterpret_cast<SmemB *>(smem_raw);
  double *sred = sh.sred;
  TileConst &tcs = sh.tcs;
  PlaneSm &pls = sh.pls;
  const TileThread t = tile_thread(G);
  const bool m0 = FAST || t.st0, m1 = FAST || t.st1;  // FAST tiles: every column is a cell
  const int L = t.c1 - t.c0;
  load_tile_const(tcs, G, M, t.k0);
  const int ig0 = G.i0 + t.c0 - 1;
  load_planes(pls, M, ig0, L + 2);
  const int cs = 2 + 2 * t.lane;
  const long long PL = G.plane;
  const int zp = rhs_planes(G);
  const long long vo = zp * PL;
  const void *map_p = &T.p_h[parity ^ 1];
  const void *map_r = &T.r_i;
  const void *map_x = &T.x_i;
  constexpr unsigned PB = TR * SROW * 8u, RB = TJ * TKB * 8u;
  RowC rw[RPW];
#pragma unroll
  for (int e = 0; e < RPW; e++) rw[e] = row_c(M, min(max(t.j0 - 1 + t.row[e], 0), G.nt - 1));

  int qi = 0, si = 0;
  auto issue = [&]() {
    if (qi <= L + 1) {
      const int il = t.c0 - 1 + qi;
      const bool rown = (qi >= 1) && (qi <= L);
      mbar_arrive_expect_tx(&sm.bar[si], rown ? PB + (XM == XM_SKIP ? 1 : 2) * RB : PB);
      tma_load_3d(&sm.pn[si][0][0], map_p, &sm.bar[si], t.k0 - 3 + COFF, t.j0 - 1, zp + il + 1);
      if (rown) {
        tma_load_3d(&sm.r[si][0][0], map_r, &sm.bar[si], t.k0 - 1 + COFF, t.j0, zp + il + 1);
        if (XM != XM_SKIP) tma_load_3d(&sm.x[si][0][0], map_x, &sm.bar[si], t.k0 - 1 + COFF, t.j0, zp + il + 1);
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
  pdl_trigger();
  pdl_wait();
  if (S->stop) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) trace_mark(A.S, TR_B0);
  const double alpha = S->alpha;
  // XM_PAIR: c = alpha_{k-1} / beta_{k-1}; cp = c + alpha_k multiplies p_k, -c multiplies z_k
  const double cpair = (XM == XM_PAIR) ? S->alpha_prev / S->beta : 0.0;
  const double cp = (XM == XM_PAIR) ? cpair + alpha : alpha;
  double acc_rz = 0.0, acc_rr = 0.0;
  if (t.valid) {  // a cluster padding block only joins the reduction
    if (threadIdx.x == 0)
      for (int s = 0; s < NS_B - 2; s++) issue();

    const double2 Z2 = make_double2(0.0, 0.0);
    double2 pm[RPW], pc[RPW], pn[RPW];
#pragma unroll
    for (int e = 0; e < RPW; e++) pm[e] = pc[e] = pn[e] = Z2;
    double *g_w = A.r_out + vo + (long long)(t.c0 + 1) * PL;  // + rowoff[e]: r of plane c0
    double *g_x = A.x + vo + (long long)(t.c0 + 1) * PL;      // + rowoff[e]: x of plane c0
    int st = 0, so = NS_B - 1;                           // stages of planes q and q-1
    unsigned ph = 0;

#pragma unroll 1
    for (int q = 0; q <= L + 1; q++) {
      __syncthreads();  // stage (q-2)%NS_B is free
      if (threadIdx.x == 0) issue();
      const double2 dp = *reinterpret_cast<const double2 *>(&tcs.dp[cs]);
      const double2 ap = *reinterpret_cast<const double2 *>(&tcs.app[cs]);
      const double2 am = *reinterpret_cast<const double2 *>(&tcs.apm[cs]);
      const PlaneC P = plane_at(pls, q >= 1 ? q - 1 : 0);  // stencil plane il-1
      mbar_wait(&sm.bar[st], ph);
#pragma unroll
      for (int e = 0; e < RPW; e++) pn[e] = *reinterpret_cast<const double2 *>(&sm.pn[st][t.row[e]][cs]);
      if (q >= 2) {
        const double *sb = &sm.pn[so][0][0];
        const FaceTerms ft = face_terms(pc[0], pc[RPW - 1], rw[0], ap.x);  // FAST: shared faces
#pragma unroll
        for (int e = 0; e < RPW; e++) {
          if (!t.stencil[e]) continue;
          const int r = t.row[e];
          const double *sr = sb + r * SROW + cs;
          const double2 up = (RPW == 2 && e == 1) ? pc[0] : *reinterpret_cast<const double2 *>(sr - SROW);
          const double2 dn = (RPW == 2 && e == 0) ? pc[RPW - 1] : *reinterpret_cast<const double2 *>(sr + SROW);
          const double lf = sr[-1], rt = sr[2];
          double q0, q1;
          if (FAST && RPW == 2) {
            const double pk = e == 0 ? ft.p0 : ft.p1;
            const double2 jo = e == 0 ? up : dn;
            const double ajo = e == 0 ? rw[0].atm : rw[RPW - 1].atp;
            q0 = stencil7s(pc[e].x, pn[e].x, pm[e].x, e == 0 ? ft.tx : -ft.tx, ajo, jo.x, pk, am.x, lf, dp.x, P,
                           rw[e]);
            q1 = stencil7s(pc[e].y, pn[e].y, pm[e].y, e == 0 ? ft.ty : -ft.ty, ajo, jo.y, -pk, ap.y, rt, dp.y, P,
                           rw[e]);
          } else {
            q0 = stencil7(pc[e].x, pn[e].x, pm[e].x, dn.x, up.x, pc[e].y, lf, dp.x, ap.x, am.x, P, rw[e]);
            q1 = stencil7(pc[e].y, pn[e].y, pm[e].y, dn.y, up.y, rt, pc[e].x, dp.y, ap.y, am.y, P, rw[e]);
          }
          const double2 rv = *reinterpret_cast<const double2 *>(&sm.r[so][r - 1][2 * t.lane]);
          double2 rn, xn;  // rn: the stored vector after the update (PC1: z, PC2: r)
          if (XM != XM_SKIP) {
            const double2 xv = *reinterpret_cast<const double2 *>(&sm.x[so][r - 1][2 * t.lane]);
            if (XM == XM_PAIR) {
              xn.x = fma(cp, pc[e].x, fma(-cpair, rv.x, xv.x));
              xn.y = fma(cp, pc[e].y, fma(-cpair, rv.y, xv.y));
            } else {
              xn.x = fma(alpha, pc[e].x, xv.x);
              xn.y = fma(alpha, pc[e].y, xv.y);
            }
          }
          if (USE_Z) {
            rn.x = fma(-alpha, q0, rv.x);
            rn.y = fma(-alpha, q1, rv.y);
            acc_rr += (m0 ? rn.x * rn.x : 0.0) + (m1 ? rn.y * rn.y : 0.0);
          } else {
            // z_{k+1} = z_k - alpha D^-1 q;  r_{k+1} = D z_{k+1}
            const DiagRow d = diag_row(P, rw[e]);
            const double d0 = diag_at(dp.x, d, ap.x, am.x), d1 = diag_at(dp.y, d, ap.y, am.y);
            rn.x = fma(-alpha, jacobi(q0, d0), rv.x);
            rn.y = fma(-alpha, jacobi(q1, d1), rv.y);
            const double s0 = d0 * rn.x, s1 = d1 * rn.y;
            acc_rz += (m0 ? s0 * rn.x : 0.0) + (m1 ? s1 * rn.y : 0.0);
            acc_rr += (m0 ? s0 * s0 : 0.0) + (m1 ? s1 * s1 : 0.0);
          }
          POT3D_CHK(S, in_range(g_w + t.rowoff[e], A.r_out + vo, (G.nr_loc + 2) * PL), CHK_PASS_STORE);
          POT3D_CHK(S, XM == XM_SKIP || in_range(g_x + t.rowoff[e], A.x + vo, (G.nr_loc + 2) * PL), CHK_PASS_STORE);
          store_pair<FAST>(g_w + t.rowoff[e], t, G.np, rn, true);
          if (XM != XM_SKIP) {
            if (FAST || (t.st0 && t.st1)) {
              __stcs(reinterpret_cast<double2 *>(g_x + t.rowoff[e]), xn);
            } else {
              if (t.st0) g_x[t.rowoff[e]] = xn.x;
              if (t.st1) g_x[t.rowoff[e] + 1] = xn.y;
            }
          }
        }
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

  }
  double v[2] = {acc_rz, acc_rr}, tot[2];
  if (grid_sum<2>(v, A.partials + blockIdx.z * A.pstride, &S->counter[1], sred, tot, pass_bid(G), pass_nb(G)) &&
      threadIdx.x == 0) {
    trace_max(A.S, TR_B1);
    double *hist = A.hist ? A.hist + blockIdx.z * A.hstride : nullptr;
    if (A.finalize) {
      if (USE_Z)
        finalize_rr(S, tot[1], hist);  // PC2: rho' comes from the sweeps
      else
        finalize_beta(S, tot[0], tot[1], hist);
    } else if (A.fold) {
      mail_post(A.peers, MAIL_B, tot[0], tot[1], mail_seq(S->epoch, S->iter + 1), S);
      S->pend_b = 1;  // finalised by the next edge-shell kernel
    } else if (A.peers) {
      mail_post(A.peers, MAIL_B, tot[0], tot[1], mail_seq(S->epoch, S->iter + 1), S);
    } else {
      A.local_sum[0] = tot[0];
      A.local_sum[1] = tot[1];
    }
  }
}

// Each pass runs the FAST instantiation on tiles away from the periodic seam and the
// phi end (tile_fast, block-uniform) and the masked one elsewhere.
#define POT3D_PASS(BODY, ...)                                   \
  __shared__ PassShared sh;                                     \
  if (tile_fast(A.G))                                           \
    BODY<__VA_ARGS__, true>(T, A, parity, sh);                  \
  else                                                          \
    BODY<__VA_ARGS__, false>(T, A, parity, sh)

__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_a(const __grid_constant__ TMaps T, PassArgs A, int parity) { POT3D_PASS(pass_a_body, false); }
// diagnostic instantiation: also stores q = A p_k into A.q_probe (pot3d_apply_fused which = 2)
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_a_probe(const __grid_constant__ TMaps T, PassArgs A, int parity) { POT3D_PASS(pass_a_body, true); }
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_b_pc1_even(const __grid_constant__ TMaps T, PassArgs A, int parity) {
  POT3D_PASS(pass_b_body, false, XM_SKIP);
}
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_b_pc1_odd(const __grid_constant__ TMaps T, PassArgs A, int parity) {
  POT3D_PASS(pass_b_body, false, XM_PAIR);
}
__global__ void __launch_bounds__(NTHREADS, PASS_MINB)
    k_pass_b_pc2(const __grid_constant__ TMaps T, PassArgs A, int parity) { POT3D_PASS(pass_b_body, true, XM_EVERY); }

// PC1 after the loop: x += alpha_K p_K when the last iteration K was even (its x
// update was deferred to the pair that never came, A23)
__global__ void k_x_finish(Grid G, const Scalars *S, double *x, const double *p) {
  const double alpha = S->alpha;
  const long long n = (long long)G.nr_loc * G.plane;
  double *xs = x + G.plane;
  const double *ps = p + G.plane;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(c % G.PK);
    if (col >= COFF && col < G.np + COFF) xs[c] = fma(alpha, ps[c], xs[c]);
  }
}

// ghost columns of shells [il0, il0 + n): physical 0 <- k = np-1, physical np+1 <- k = 0
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
