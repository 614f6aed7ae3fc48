// pc2.cu -- PC2: zero-fill ILU of each r-slab block ("non-overlapping
// domain decomposition with zero-fill incomplete LU"), as the D-ILU
// factorisation that ILU0 reduces to for the 7-point pattern (A11):
//
//   factor:   d_m = diag_m - sum_{n in N-(m)} A_mn^2 / d_n
//   forward:  w_m = (r_m + sum_{n in N-(m)} A_mn w_n) / d_m           (D + L) w = r
//   backward: z_m = w_m + (1/d_m) sum_{n in N+(m)} A_mn z_n            (I + D^-1 U) z = w
//
// with A_mn > 0 the face coupling (off-diagonal -A_mn), N-(m) = {i-1, j-1, k-1}
// and N+(m) = {i+1, j+1, k+1} inside the block: couplings that leave the
// block's shells and the periodic phi wrap are dropped; the full
// diagonal is kept.  The triangular solves are "not vectorizable" as a
// sequential sweep; here they run as a 3-D wavefront on hyperplanes
// i+j+k, tiled: a CTA owns a WJ x WK theta-phi tile over all shells of one
// block and walks its own hyperplanes (thread (jj,kk) handles shell
// t-jj-kk at step t, neighbours inside the tile through a shared double
// buffer, the r neighbour in a register); the values a tile needs from the
// tiles above / to the left arrive through sentinel-armed edge slots (no
// flags, no fences), CTAs take tiles in topological order from a ticket
// counter so that every tile a CTA waits on belongs to a CTA that is already
// running, and every wait is bounded.  Every cell is
// computed by exactly the sequential formula, only the order of the three
// neighbour terms is fixed (r, theta, phi), so the sweep equals the
// sequential ILU0 solve up to rounding.
#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <string>

#include "device_common.cuh"

namespace pot3d {

template <int V>
using IC2 = std::integral_constant<int, V>;

constexpr int WJ = 8;            // tile rows (theta)
constexpr int WK = 32;           // tile columns (phi): one warp per row
constexpr int WT = WJ * WK;      // threads per CTA


enum SweepMode { SW_FACTOR = 0, SW_FWD = 1, SW_BWD = 2 };

struct Pc2 {
  Grid G;
  int nblk;                 // ILU blocks on this rank
  int ntj, ntk, ntiles;     // tile grid
  int *d_l0;                // block bounds: nblk+1 local shell indices
  int2 *d_order;            // tiles in topological (start-time) order
  int *d_sync;              // [0] ticket, [1] flags: 1 breakdown, 2 handoff protocol error
  int nsync;
  double *edge;             // tile-edge handoff slots (sentinel-armed)
  long long edge_len;       // doubles
  int nbmax;                // largest block (shells)
  double *inv_d;            // 1/d_m, cell layout
  // run-vectorised sweeps (k_sweep4)
  int ntj4, ntk4, ntiles4, koff_f, koff_b;
  int2 *d_order4;
  int2 *d_orderS;           // k_sweepS: tiles by estimated start step tj*SWJ + tk
  bool scan;                // k_sweepS (default) or k_sweep4 (POT3D_PC2_SWEEP=4)
  double *edge4;
  long long edge4_len;      // all problems' slots (nrhs x the per-problem slots)
  int nrhs;                 // problems per sweep launch (a batch leader: pot3d_runtime.nrhs)
  std::vector<void *> allocs;
  size_t bytes;
};

struct SweepArgs {
  Grid G;
  Metrics M;
  Scalars *S;
  const int *l0;
  const int2 *order;
  int *sync;
  int nblk, ntj, ntk, ntiles;
  const double *r;   // FWD: rhs r; BWD: r for the r.z partial
  double *z;         // FWD: writes w; BWD: w -> z in place
  double *inv_d;     // FACTOR writes, FWD/BWD read
  double *partials;
  double *edge;
  long long edge_len;  // doubles of `edge` (POT3D_CHECK bounds)
  int nbmax;
  int predicated;    // skip when the PCG loop has stopped
  int finalize;      // BWD: 1 single rank (rho/beta), 0 local_sum
  double *local_sum;
  const PeerTab *peers;  // BWD, nranks > 1 with peer memory: post r.z to every mailbox
  int nrhs;              // k_sweepS of a batch: problems per launch (tickets interleave them)
  long long vstride, pstride;  // a batch: doubles between the problems' vectors / partials
};

// Tile-edge handoff without flags or fences: the bottom row / right column of
// every tile is also written into an edge buffer whose slots hold a sentinel
// (a signalling-NaN bit pattern arithmetic never produces) until the producer
// stores the value; the single consumer prefetches the slot PD steps ahead with
// ld.global.cv, polls only while it still reads the sentinel, and re-arms it.
constexpr unsigned long long SENT = 0x7FF57FF57FF57FF5ull;
#ifndef POT3D_SWEEP_D
#define POT3D_SWEEP_D 8
#endif
constexpr int PD = POT3D_SWEEP_D;  // prefetch distance (steps)

// polling load: volatile asm so the compiler cannot hoist it out of a spin loop
__device__ __forceinline__ double ld_poll(const double *p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ bool is_sent(double v) {
  return (unsigned long long)__double_as_longlong(v) == SENT;
}

// Wait until the edge slot p holds a value (v: its prefetched content).  Bounded:
// after POLL_TIMEOUT_NS, or at once when another thread has already given up
// (flags bit 2), the protocol error is recorded and the sweep runs on with
// garbage, which the solve then reports.
constexpr unsigned long long POLL_TIMEOUT_NS = 2000000000ull;  // 2 s
__device__ __forceinline__ double poll_slot(const double *p, double v, int *flags, bool &proto) {
  if (!is_sent(v)) return v;
  const unsigned long long t0 = global_ns();
  for (int n = 0;; n++) {
    v = ld_poll(p);
    if (!is_sent(v)) return v;
    if ((n & 63) == 63) {
      if (*reinterpret_cast<volatile int *>(flags) & 2) break;
      if (global_ns() - t0 > POLL_TIMEOUT_NS) {
        atomicOr(flags, 2);
        break;
      }
    }
  }
  proto = true;
  return v;
}

#ifndef POT3D_SWEEP_MINB
#define POT3D_SWEEP_MINB 1
#endif
// D-ILU factorisation (setup only): d_m = diag_m - sum_{N-} A_mn^2 / d_n as a
// one-cell-per-thread wavefront over 8 x 32 tiles; writes 1/d.
__global__ void __launch_bounds__(WT, POT3D_SWEEP_MINB) k_factor(SweepArgs A) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  if (A.predicated && A.S->stop) return;
  __shared__ double sw[2][WJ][WK];
  __shared__ int s_ticket;
  const int tid = threadIdx.x;
  const int jj = tid / WK, kk = tid % WK;
  if (tid == 0) s_ticket = atomicAdd(&A.sync[0], 1);
  __syncthreads();
  const int ticket = s_ticket;
  const int b = ticket % A.nblk;
  const int pos = ticket / A.nblk;
  const int2 tl = A.order[pos];  // virtual tile (tj, tk)
  const int l0 = A.l0[b], l1 = A.l0[b + 1];
  const int nb = l1 - l0;
  // dependencies on i-1, j-1, k-1 (the factor runs in natural order)
  const int jv = tl.x * WJ + jj, kv = tl.y * WK + kk;
  const bool valid = (jv < G.nt) && (kv < G.np);
  const int j = jv;
  const int k = kv;
  const int jc = valid ? j : 0, kc = valid ? k : 0;
  const int nsteps = nb + WJ + WK - 2;
  // edge buffers of this tile (producer) and of its up / left neighbours (consumer)
  const int my = tl.x * A.ntk + tl.y;
  const long long tstride = (long long)A.nbmax * (WK + WJ);
  double *eb_base = A.edge + (long long)b * A.ntiles * tstride;
  // slots are plane-contiguous per column/row: [kk][iv] and [jj][iv]
  double *my_bot = eb_base + my * tstride + (long long)kk * A.nbmax;
  double *my_rgt = eb_base + my * tstride + (long long)A.nbmax * (WK + jj);
  const bool put_bot = valid && (jj == WJ - 1) && (jv + 1 < G.nt);
  const bool put_rgt = valid && (kk == WK - 1) && (kv + 1 < G.np);
  const bool need_j = valid && (jj == 0) && (jv > 0);
  const bool need_k = valid && (kk == 0) && (kv > 0);
  double *up_bot = need_j ? eb_base + (long long)(my - A.ntk) * tstride + (long long)kk * A.nbmax : nullptr;
  double *lf_rgt = need_k ? eb_base + (long long)(my - 1) * tstride + (long long)A.nbmax * (WK + jj) : nullptr;

  // row / column factors
  const double g = __ldg(M.g + jc), q = __ldg(M.q + jc);
  const double atp = __ldg(M.atp + jc), atm = __ldg(M.atm + jc);
  const double dpk = __ldg(M.dp + kc), app = __ldg(M.app + kc), apm = __ldg(M.apm + kc);
  // couplings to the predecessors (zero across the pole / the dropped wrap)
  const double ct = atm;                         // x dr_i dp_k
  const double cp = (k > 0) ? apm : 0.0;         // x dr_i q_j
  const long long o_base = cidx(G, l0, jc, kc);
  const long long o_step = G.plane;
  const int ig_base = G.i0 + l0;

  // prefetch ring of the neighbour-tile values this thread needs PD steps ahead
  double rnj[PD], rnk[PD];
  auto fetch = [&](int ts, double &xj, double &xk) {
    const int iv = ts - jj - kk;
    xj = xk = 0.0;
    if (valid && iv >= 0 && iv < nb) {
      // re-polled at use while still the sentinel
      if (need_j) xj = ld_poll(up_bot + iv);
      if (need_k) xk = ld_poll(lf_rgt + iv);
    }
  };
  bool proto = false;
#pragma unroll
  for (int u = 0; u < PD; u++) fetch(u, rnj[u], rnk[u]);

  double wprev = 0.0;
  bool bad = false;
  for (int t0 = 0; t0 < nsteps; t0 += PD) {
#pragma unroll
    for (int u = 0; u < PD; u++) {
      const int t = t0 + u;
      if (t >= nsteps) break;
      __syncthreads();  // step t-1 complete in this CTA (shared double buffer)
      double nj = rnj[u], nk = rnk[u];
      fetch(t + PD, rnj[u], rnk[u]);
      const int ivt = t - jj - kk;  // virtual local shell of this thread at step t
      if (valid && ivt >= 0 && ivt < nb) {
        if (need_j) {  // value of the tile above (virtual), produced at its step t+WJ-1
          nj = poll_slot(up_bot + ivt, nj, A.sync + 1, proto);
          __stcg(reinterpret_cast<unsigned long long *>(up_bot + ivt), SENT);  // re-arm
        }
        if (need_k) {
          nk = poll_slot(lf_rgt + ivt, nk, A.sync + 1, proto);
          __stcg(reinterpret_cast<unsigned long long *>(lf_rgt + ivt), SENT);
        }
        const long long o = o_base + (long long)ivt * o_step;
        const int ig = ig_base + ivt;
        const double dr = __ldg(M.dr + ig);
        const double vi = (ivt > 0) ? wprev : 0.0;
        const double vj = (jj > 0) ? sw[(t - 1) & 1][jj - 1][kk] : (need_j ? nj : 0.0);
        const double vk = (kk > 0) ? sw[(t - 1) & 1][jj][kk - 1] : (need_k ? nk : 0.0);
        const double cr = (ivt > 0) ? __ldg(M.arm + ig) : 0.0;
        const double Ar = cr * g * dpk, At = dr * ct * dpk, Ap = dr * q * cp;
        const double diag = dpk * (g * (__ldg(M.arp + ig) + __ldg(M.arm + ig) + __ldg(M.ss + ig)) +
                                   dr * (atp + atm)) + dr * q * (app + apm);
        // the wrap coupling and the inter-block couplings are dropped from L/U,
        // the full diagonal is kept (A11); vi, vj, vk hold 1/d of the predecessors
        const double d = diag - Ar * Ar * vi - At * At * vj - Ap * Ap * vk;
        bad |= !(d > 1e-300);
        const double val = 1.0 / d;
        A.inv_d[o] = val;
        if (put_bot) __stcg(my_bot + ivt, val);
        if (put_rgt) __stcg(my_rgt + ivt, val);
        wprev = val;
        sw[t & 1][jj][kk] = val;
      }
    }
  }
  if (__syncthreads_or(proto) && tid == 0) atomicOr(&A.sync[1], 2);  // protocol error
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&A.sync[1], 1);      // pivot breakdown
}

// ---------------------------------------------------------------------------
// Run-vectorised forward / backward sweeps.  Same wavefront and handoff
// protocol as k_factor, but a thread owns SV = 4 phi-consecutive cells of one
// row (a "run", one 32-B sector per array) instead of one cell: step t of
// thread (jj, m) handles shell t - jj - m of run m, so the lanes of a warp read
// and write whole sectors (the one-cell mapping used a quarter of every sector
// it moved).  Inside a run the phi dependency is sequential in the thread;
// the run's first cell takes the last cell of run m-1 (previous step, shared
// memory, or the left tile's edge slot).  Runs are aligned to 32 B in memory
// (virtual offset koff), operands are prefetched SPD steps ahead by cp.async
// into a shared ring, edge slots included (re-polled at use while they still
// hold the sentinel).  FACTOR keeps the one-cell kernel (setup only).
// ---------------------------------------------------------------------------
constexpr int SV = 4;            // cells per thread along phi
constexpr int SNR = 32;          // runs per tile row (one warp)
constexpr int SWK = SV * SNR;    // 128 phi columns per tile
#ifndef POT3D_SWJ
#define POT3D_SWJ 16
#endif
constexpr int SWJ = POT3D_SWJ;   // tile rows
constexpr int SWT = SWJ * SNR;   // 256 threads
#ifndef POT3D_SPD
#define POT3D_SPD 1
#endif
constexpr int SPD = POT3D_SPD;   // register prefetch depth (steps)

template <int MODE> struct Sw4 {
  static constexpr int XW = 2 * SWJ * SNR * SV;        // doubles of the step exchange
  static constexpr size_t SMEM = (size_t)XW * sizeof(double);
};

// virtual phi offset of the first run so that every run starts on a 32-B
// boundary of the physical columns (c = k + COFF): FWD k = kv, BWD k = np-1-kv
__host__ __device__ inline int sweep4_koff(int np, bool rev) {
  if (!rev) return -1;                  // kv0 = 4m - 1  ->  c0 = 4m
  int o = (np - 3) % 4;                 // kv0 = np - 3 (mod 4) -> lowest column 4m
  return o > 0 ? o - 4 : o;
}

// 256-bit global accesses (one L1TEX wavefront per lane and run)
__device__ __forceinline__ void ldg4(const double *p, double (&v)[4]) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void ldg4_cg(const double *p, double (&v)[4]) {  // L2 only (edge slots)
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void stg4(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ void stg4_cg(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ double ldg_cg(const double *p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(SWT, 1) k_sweep4(SweepArgs A, int koff, int ntk4) {
  constexpr bool rev = (MODE == SW_BWD);
  constexpr int PD = SPD;
  const Grid &G = A.G;
  const Metrics &M = A.M;
  if (A.predicated && A.S->stop) return;
  extern __shared__ __align__(16) double sm4[];
  double *xw = sm4;                         // [2][SWJ][SNR][SV] step exchange
  double *crs = xw + Sw4<MODE>::XW;         // [nbmax] r coupling factor of virtual shell iv
  double *drs = crs + A.nbmax;              // [nbmax] dr of virtual shell iv
  __shared__ int s_ticket;
  __shared__ double sred[SWT / 32];
  const int tid = threadIdx.x;
  const int jj = tid / SNR, m = tid % SNR;
  if (tid == 0) s_ticket = atomicAdd(&A.sync[0], 1);
  __syncthreads();
  const int ticket = s_ticket;
  const int b = ticket % A.nblk;
  const int pos = ticket / A.nblk;
  const int2 tl = A.order[pos];
  const int l0 = A.l0[b], l1 = A.l0[b + 1];
  const int nb = l1 - l0;
  // per-shell factors of this block in virtual order (r predecessor: arm for FWD, arp for BWD)
  for (int iv = tid; iv < nb; iv += SWT) {
    const int ig = G.i0 + (rev ? l1 - 1 - iv : l0 + iv);
    crs[iv] = (iv > 0) ? (rev ? __ldg(M.arp + ig) : __ldg(M.arm + ig)) : 0.0;
    drs[iv] = __ldg(M.dr + ig);
  }
  const int jv = tl.x * SWJ + jj;
  const bool vrow = jv < G.nt;
  const int jc = vrow ? (rev ? G.nt - 1 - jv : jv) : 0;
  const int kv0 = koff + tl.y * SWK + SV * m;        // virtual k of element 0
  const double g = __ldg(M.g + jc), q = __ldg(M.q + jc);
  const double ct = rev ? __ldg(M.atp + jc) : __ldg(M.atm + jc);
  bool ve[SV];
  double gd[SV], td[SV], qc[SV];  // g dp_k, ct dp_k, q cp_k: A^r = cr gd, A^t = dr td, A^p = dr qc
  bool any = false, full = true;
#pragma unroll
  for (int e = 0; e < SV; e++) {
    const int kv = kv0 + e;
    ve[e] = vrow && kv >= 0 && kv < G.np;
    any |= ve[e];
    full &= ve[e];
    const int k = rev ? G.np - 1 - kv : kv;
    const int kc = ve[e] ? k : 0;
    const double dpk = ve[e] ? __ldg(M.dp + kc) : 0.0;
    const double cpk = !ve[e] ? 0.0 : rev ? ((k < G.np - 1) ? __ldg(M.app + kc) : 0.0)
                                          : ((k > 0) ? __ldg(M.apm + kc) : 0.0);
    gd[e] = g * dpk;
    td[e] = ct * dpk;
    qc[e] = q * cpk;
  }
  // lowest physical column of the run (32-B aligned); element e <-> col_lo + (rev ? 3-e : e)
  const int col_lo = rev ? G.np - kv0 - 3 : kv0 + COFF;
  // cell offset of the run at step ts: o0 + ts * ostep (virtual shell iv = ts - jj - m)
  const long long ostep = rev ? -G.plane : G.plane;
  const long long o0 = (long long)((rev ? l1 - 1 : l0) + 1) * G.plane + (long long)jc * G.PK + col_lo -
                       (long long)(jj + m) * ostep;

  // edge slots: per tile, bottom [SNR][nbmax][SV] then right [SWJ][nbmax][2]
  const int my = tl.x * ntk4 + tl.y;
  const long long tstride = (long long)A.nbmax * (SNR * SV + SWJ * 2);
  double *eb = A.edge + (long long)b * A.ntiles * tstride;
  double *my_bot = eb + my * tstride + (long long)m * A.nbmax * SV;
  double *my_rgt = eb + my * tstride + (long long)SNR * A.nbmax * SV + (long long)jj * A.nbmax * 2;
  const bool put_bot = (jj == SWJ - 1) && (jv + 1 < G.nt) && any;
  const bool put_rgt = (m == SNR - 1) && vrow && (kv0 + SV < G.np);
  const bool need_j = (jj == 0) && vrow && (jv > 0) && any;
  const bool need_k = (m == 0) && vrow && (kv0 > 0);
  double *up_bot = eb + (long long)(my - ntk4) * tstride + (long long)m * A.nbmax * SV;
  double *lf_rgt = eb + (long long)(my - 1) * tstride + (long long)SNR * A.nbmax * SV + (long long)jj * A.nbmax * 2;

  const double *src0 = (MODE == SW_FWD) ? A.r : A.z;  // FWD: r; BWD: w (forward output)
  const double *src1 = A.inv_d;
  const double *src2 = A.r;                          // BWD: r for the r.z partial
  const int ts_lo = jj + m;                          // first step with a cell of this thread
  double *xo_me = xw + (jj * SNR + m) * SV;
  const double *xj_me = xw + ((jj > 0 ? jj - 1 : 0) * SNR + m) * SV;
  const double *xk_me = xw + (jj * SNR + (m > 0 ? m - 1 : 0)) * SV + SV - 1;
  constexpr int XB = SWJ * SNR * SV;

  // register prefetch ring (PD steps ahead), slot = step mod PD (compile-time by unrolling)
  double ra[PD][SV], rb[PD][SV], rc[PD][SV], rj[PD][SV], rk[PD];
  int pf_t = 0;
  long long pf_o = o0;
  auto prefetch = [&](auto U) {
    constexpr int u = decltype(U)::value;
    const int iv = pf_t - ts_lo;
    if (any && (unsigned)iv < (unsigned)nb) {
      ldg4(src0 + pf_o, ra[u]);
      ldg4(src1 + pf_o, rb[u]);
      if (MODE == SW_BWD) ldg4(src2 + pf_o, rc[u]);
      if (need_j) ldg4_cg(up_bot + iv * SV, rj[u]);
      if (need_k) rk[u] = ldg_cg(lf_rgt + iv * 2);
    }
    ++pf_t;
    pf_o += ostep;
  };

  double wprev[SV];
#pragma unroll
  for (int e = 0; e < SV; e++) wprev[e] = 0.0;
  double acc = 0.0;
  bool proto = false;
  double *zr = A.z + o0;  // the run at step t (advanced every step)

  auto step = [&](auto U, int t) {
    constexpr int u = decltype(U)::value;
    __syncthreads();  // step t-1 of the neighbouring threads is in xw; crs/drs staged
    const int ivt = t - ts_lo;
    if (any && (unsigned)ivt < (unsigned)nb) {
      double a0[SV], b0[SV], c0[SV];
#pragma unroll
      for (int e = 0; e < SV; e++) {  // registers hold physical column order
        const int pe = rev ? SV - 1 - e : e;
        a0[e] = ra[u][pe];
        b0[e] = rb[u][pe];
        c0[e] = (MODE == SW_BWD) ? rc[u][pe] : 0.0;
      }
      const double *xp = (t & 1) ? xw : xw + XB;  // buffer of step t-1
      double vj[SV], vk;
      if (jj > 0) {
        const double2 u0 = *reinterpret_cast<const double2 *>(xp + (xj_me - xw));
        const double2 u1 = *reinterpret_cast<const double2 *>(xp + (xj_me - xw) + 2);
        vj[0] = u0.x; vj[1] = u0.y; vj[2] = u1.x; vj[3] = u1.y;
      } else if (need_j) {
        double *slot = up_bot + (long long)ivt * SV;
#pragma unroll
        for (int e = 0; e < SV; e++) {
          double v = rj[u][e];
          if (ve[e] && is_sent(v)) v = poll_slot(slot + e, v, A.sync + 1, proto);
          vj[e] = ve[e] ? v : 0.0;
        }
        // re-arm all four slots: the producer stores whole runs, FWD / BWD share them
        stg4_cg(slot, __longlong_as_double((long long)SENT), __longlong_as_double((long long)SENT),
                __longlong_as_double((long long)SENT), __longlong_as_double((long long)SENT));
      } else {
        vj[0] = vj[1] = vj[2] = vj[3] = 0.0;
      }
      if (m > 0) {
        vk = xp[xk_me - xw];
      } else if (need_k) {
        vk = rk[u];
        if (is_sent(vk)) vk = poll_slot(lf_rgt + (long long)ivt * 2, vk, A.sync + 1, proto);
        __stcg(reinterpret_cast<unsigned long long *>(lf_rgt + (long long)ivt * 2), SENT);
      } else {
        vk = 0.0;
      }
      const double cr = crs[ivt], dr = drs[ivt];
      double val[SV];
#pragma unroll
      for (int e = 0; e < SV; e++) {
        const double Ar = cr * gd[e], At = dr * td[e], Ap = dr * qc[e];
        double v;
        if (MODE == SW_FWD)
          v = (a0[e] + Ar * wprev[e] + At * vj[e] + Ap * vk) * b0[e];
        else
          v = a0[e] + b0[e] * (Ar * wprev[e] + At * vj[e] + Ap * vk);
        v = ve[e] ? v : 0.0;
        if (MODE == SW_BWD) acc += c0[e] * v;
        val[e] = v;
        vk = v;
      }
      // results: z (w for FWD), physical order col_lo .. col_lo+3
      POT3D_CHK(A.S, in_range(zr, A.z, (G.nr_loc + 2) * G.plane) && in_range(zr + SV - 1, A.z, (G.nr_loc + 2) * G.plane),
                CHK_SWEEP_STORE);
#if POT3D_CHECK
      if (put_bot) {  // the consumer re-armed this slot (a value not yet read must not be overwritten)
        double sv[4];
        ldg4_cg(my_bot + (long long)ivt * SV, sv);
        POT3D_CHK(A.S, in_range(my_bot + (long long)ivt * SV + SV - 1, A.edge, A.edge_len), CHK_SWEEP_STORE);
        POT3D_CHK(A.S, is_sent(sv[0]) && is_sent(sv[1]) && is_sent(sv[2]) && is_sent(sv[3]), CHK_SLOT_REUSE);
      }
      if (put_rgt) {
        POT3D_CHK(A.S, in_range(my_rgt + (long long)ivt * 2, A.edge, A.edge_len), CHK_SWEEP_STORE);
        POT3D_CHK(A.S, is_sent(ldg_cg(my_rgt + (long long)ivt * 2)), CHK_SLOT_REUSE);
      }
#endif
      if (full) {
        if (rev)
          stg4(zr, val[3], val[2], val[1], val[0]);
        else
          stg4(zr, val[0], val[1], val[2], val[3]);
      } else {
        if (rev ? ve[3] : ve[0]) zr[0] = rev ? val[3] : val[0];
        if (rev ? ve[2] : ve[1]) zr[1] = rev ? val[2] : val[1];
        if (rev ? ve[1] : ve[2]) zr[2] = rev ? val[1] : val[2];
        if (rev ? ve[0] : ve[3]) zr[3] = rev ? val[0] : val[3];
      }
      if (put_bot) stg4_cg(my_bot + (long long)ivt * SV, val[0], val[1], val[2], val[3]);
      if (put_rgt) __stcg(my_rgt + (long long)ivt * 2, val[SV - 1]);
      double *xo = ((t & 1) ? xw + XB : xw) + (xo_me - xw);
      *reinterpret_cast<double2 *>(xo) = make_double2(val[0], val[1]);
      *reinterpret_cast<double2 *>(xo + 2) = make_double2(val[2], val[3]);
#pragma unroll
      for (int e = 0; e < SV; e++) wprev[e] = val[e];
    }
    zr += ostep;
    prefetch(U);  // step t + PD into this slot
  };

  const int nsteps = nb + SWJ + SNR - 2;
  prefetch(IC2<0>{});
  if (PD > 1) prefetch(IC2<(PD > 1 ? 1 : 0)>{});
  if (PD > 2) prefetch(IC2<(PD > 2 ? 2 : 0)>{});
  if (PD > 3) prefetch(IC2<(PD > 3 ? 3 : 0)>{});
#pragma unroll 1
  for (int t = 0; t < nsteps; t += PD) {
    step(IC2<0>{}, t);
    if (PD > 1) { if (t + 1 >= nsteps) break; step(IC2<(PD > 1 ? 1 : 0)>{}, t + 1); }
    if (PD > 2) { if (t + 2 >= nsteps) break; step(IC2<(PD > 2 ? 2 : 0)>{}, t + 2); }
    if (PD > 3) { if (t + 3 >= nsteps) break; step(IC2<(PD > 3 ? 3 : 0)>{}, t + 3); }
  }
  if (__syncthreads_or(proto) && tid == 0) atomicOr(&A.sync[1], 2);  // protocol error
  if (MODE == SW_BWD) {
    double v[1] = {acc}, tot[1];
    if (grid_sum<1>(v, A.partials, &A.S->counter[2], sred, tot, ticket, A.nblk * A.ntiles) && tid == 0) {
      if (A.finalize)
        finalize_rho(A.S, tot[0]);
      else if (A.peers)
        mail_post(A.peers, MAIL_C, tot[0], 0.0, mail_seq(A.S->epoch, A.S->iter), A.S);
      else
        A.local_sum[0] = tot[0];
    }
  }
}

// ---------------------------------------------------------------------------
// Row-scan sweeps (k_sweepS, the default): the D-ILU recurrences, tile grid and
// edge-slot handoff of k_sweep4, but the 32 lanes of a warp work on ONE shell of
// one theta row: lane m owns the run of SV = 4 phi-consecutive cells 4m .. 4m+3
// of the tile, so each warp-wide load or store is one contiguous 1-KB segment
// (k_sweep4's lanes sit on 32 different shells: one L1TEX wavefront per lane and
// access bounds its 0.72 us step).  Along the row the recurrence
// w_k = c_k + m_k w_{k-1} is an affine map per cell; the lane composes its run's
// four maps, an inclusive scan of the lanes' maps (5 shuffle rounds) gives every
// lane the value entering its run, and the carry into lane 0 is the last cell of
// the tile to the left (edge slot).  Step t: warp jj handles shell t - jj; the
// theta neighbour comes from warp jj-1's previous step (shared memory) or the
// tile above (edge slot); the r neighbour stays in registers.  The scan
// re-associates the phi recurrence (same operator, rounding of the composed maps).
// ---------------------------------------------------------------------------
// FULL: every cell of the tile lies inside the grid (no masks; all tiles but the
// last theta row and the two phi ends)
template <int MODE, bool FULL>
__device__ __forceinline__ void sweepS_body(const SweepArgs &A, int koff, int ntk4, int ticket, double *sred) {
  constexpr bool rev = (MODE == SW_BWD);
  constexpr int PD = SPD;
  const Grid &G = A.G;
  const Metrics &M = A.M;
  extern __shared__ __align__(16) double sm4[];
  double *xw = sm4;                         // [2][SWJ][SNR][SV] rows of the previous step
  double *crs = xw + Sw4<MODE>::XW;         // [nbmax] r coupling factor of virtual shell iv
  double *drs = crs + A.nbmax;              // [nbmax] dr of virtual shell iv
  const int tid = threadIdx.x;
  const int jj = tid / SNR, m = tid % SNR;
  const int b = ticket % A.nblk;
  const int pos = ticket / A.nblk;
  const int2 tl = A.order[pos];
  const int l0 = A.l0[b], l1 = A.l0[b + 1];
  const int nb = l1 - l0;
  for (int iv = tid; iv < nb; iv += SWT) {
    const int ig = G.i0 + (rev ? l1 - 1 - iv : l0 + iv);
    crs[iv] = (iv > 0) ? (rev ? __ldg(M.arp + ig) : __ldg(M.arm + ig)) : 0.0;
    drs[iv] = __ldg(M.dr + ig);
  }
  const int jv = tl.x * SWJ + jj;
  const bool vrow = FULL || jv < G.nt;  // warp-uniform
  const int jc = vrow ? (rev ? G.nt - 1 - jv : jv) : 0;
  const int kv0 = koff + tl.y * SWK + SV * m;        // virtual k of element 0
  const double g = __ldg(M.g + jc), q = __ldg(M.q + jc);
  const double ct = rev ? __ldg(M.atp + jc) : __ldg(M.atm + jc);
  bool ve[SV];
  double gd[SV], td[SV], qc[SV];
  bool any = false, full = true;
#pragma unroll
  for (int e = 0; e < SV; e++) {
    const int kv = kv0 + e;
    ve[e] = FULL || (vrow && kv >= 0 && kv < G.np);
    any |= ve[e];
    full &= ve[e];
    const int k = rev ? G.np - 1 - kv : kv;
    const int kc = ve[e] ? k : 0;
    const double dpk = ve[e] ? __ldg(M.dp + kc) : 0.0;
    const double cpk = !ve[e] ? 0.0 : rev ? ((k < G.np - 1) ? __ldg(M.app + kc) : 0.0)
                                          : ((k > 0) ? __ldg(M.apm + kc) : 0.0);
    gd[e] = g * dpk;
    td[e] = ct * dpk;
    qc[e] = q * cpk;
  }
  const int col_lo = rev ? G.np - kv0 - 3 : kv0 + COFF;
  const long long ostep = rev ? -G.plane : G.plane;
  const long long o0 = (long long)((rev ? l1 - 1 : l0) + 1) * G.plane + (long long)jc * G.PK + col_lo -
                       (long long)jj * ostep;

  const int my = tl.x * ntk4 + tl.y;
  const long long tstride = (long long)A.nbmax * (SNR * SV + SWJ * 2);
  double *eb = A.edge + (long long)b * A.ntiles * tstride;
  double *my_bot = eb + my * tstride + (long long)m * A.nbmax * SV;
  double *my_rgt = eb + my * tstride + (long long)SNR * A.nbmax * SV + (long long)jj * A.nbmax * 2;
  if (FULL) {
    any = true;
    full = true;
  }
  const bool put_bot = (jj == SWJ - 1) && (jv + 1 < G.nt) && any;
  const bool put_rgt = (m == SNR - 1) && vrow && (kv0 + SV < G.np);
  const bool need_j = (jj == 0) && vrow && (jv > 0) && any;
  const bool need_k = (m == 0) && vrow && (kv0 > 0);
  double *up_bot = eb + (long long)(my - ntk4) * tstride + (long long)m * A.nbmax * SV;
  double *lf_rgt = eb + (long long)(my - 1) * tstride + (long long)SNR * A.nbmax * SV + (long long)jj * A.nbmax * 2;

  const double *src0 = (MODE == SW_FWD) ? A.r : A.z;
  const double *src1 = A.inv_d;
  const double *src2 = A.r;
  const int ts_lo = jj;  // first step with a cell of this warp
  double *xo_me = xw + (jj * SNR + m) * SV;
  const double *xj_me = xw + ((jj > 0 ? jj - 1 : 0) * SNR + m) * SV;
  constexpr int XB = SWJ * SNR * SV;

  double ra[PD][SV], rb[PD][SV], rc[PD][SV], rj[PD][SV], rk[PD];
  int pf_t = 0;
  long long pf_o = o0;
  auto prefetch = [&](auto U) {
    constexpr int u = decltype(U)::value;
    const int iv = pf_t - ts_lo;
    if (any && (unsigned)iv < (unsigned)nb) {
      ldg4(src0 + pf_o, ra[u]);
      ldg4(src1 + pf_o, rb[u]);
      if (MODE == SW_BWD) ldg4(src2 + pf_o, rc[u]);
      if (need_j) ldg4_cg(up_bot + iv * SV, rj[u]);
      if (need_k) rk[u] = ldg_cg(lf_rgt + iv * 2);
    }
    ++pf_t;
    pf_o += ostep;
  };

  double wprev[SV];
#pragma unroll
  for (int e = 0; e < SV; e++) wprev[e] = 0.0;
  double acc = 0.0;
  bool proto = false;
  double *zr = A.z + o0;

  auto step = [&](auto U, int t) {
    constexpr int u = decltype(U)::value;
    __syncthreads();  // row jj-1 of step t-1 is in xw; crs/drs staged
    const int ivt = t - ts_lo;
    if (vrow && (unsigned)ivt < (unsigned)nb) {  // warp-uniform: every lane takes part in the scan
      double a0[SV], b0[SV], c0[SV];
#pragma unroll
      for (int e = 0; e < SV; e++) {
        const int pe = rev ? SV - 1 - e : e;
        a0[e] = ra[u][pe];
        b0[e] = rb[u][pe];
        c0[e] = (MODE == SW_BWD) ? rc[u][pe] : 0.0;
      }
      const double *xp = (t & 1) ? xw : xw + XB;  // buffer of step t-1
      double vj[SV];
      if (jj > 0) {
        const double2 u0 = *reinterpret_cast<const double2 *>(xp + (xj_me - xw));
        const double2 u1 = *reinterpret_cast<const double2 *>(xp + (xj_me - xw) + 2);
        vj[0] = u0.x; vj[1] = u0.y; vj[2] = u1.x; vj[3] = u1.y;
      } else if (need_j) {
        double *slot = up_bot + (long long)ivt * SV;
        bool waiting = false;  // one test for the usual case: all four values arrived
#pragma unroll
        for (int e = 0; e < SV; e++) waiting |= (FULL || ve[e]) && is_sent(rj[u][e]);
        if (waiting) {
#pragma unroll
          for (int e = 0; e < SV; e++)
            if ((FULL || ve[e]) && is_sent(rj[u][e])) rj[u][e] = poll_slot(slot + e, rj[u][e], A.sync + 1, proto);
        }
#pragma unroll
        for (int e = 0; e < SV; e++) vj[e] = (FULL || ve[e]) ? rj[u][e] : 0.0;
        stg4_cg(slot, __longlong_as_double((long long)SENT), __longlong_as_double((long long)SENT),
                __longlong_as_double((long long)SENT), __longlong_as_double((long long)SENT));
      } else {
        vj[0] = vj[1] = vj[2] = vj[3] = 0.0;
      }
      double vk0 = 0.0;  // the carry into lane 0: the left tile's last cell of this row and shell
      if (need_k) {
        vk0 = rk[u];
        if (is_sent(vk0)) vk0 = poll_slot(lf_rgt + (long long)ivt * 2, vk0, A.sync + 1, proto);
        __stcg(reinterpret_cast<unsigned long long *>(lf_rgt + (long long)ivt * 2), SENT);
      }
      const double cr = crs[ivt], dr = drs[ivt];
      // per cell: w_e = cc_e + mm_e w_{e-1}
      double cc[SV], mm[SV];
#pragma unroll
      for (int e = 0; e < SV; e++) {
        const double Ar = cr * gd[e], At = dr * td[e], Ap = dr * qc[e];
        double c, mul;
        if (MODE == SW_FWD) {
          c = (a0[e] + Ar * wprev[e] + At * vj[e]) * b0[e];
          mul = Ap * b0[e];
        } else {
          c = a0[e] + b0[e] * (Ar * wprev[e] + At * vj[e]);
          mul = b0[e] * Ap;
        }
        cc[e] = (FULL || ve[e]) ? c : 0.0;
        mm[e] = (FULL || ve[e]) ? mul : 0.0;
      }
      // the run's map w_out = C + Mr w_in, then the inclusive scan over the lanes
      double C = cc[0], Mr = mm[0];
#pragma unroll
      for (int e = 1; e < SV; e++) {
        C = fma(mm[e], C, cc[e]);
        Mr = mm[e] * Mr;
      }
#pragma unroll
      for (int o = 1; o < SNR; o <<= 1) {
        const double Cp = __shfl_up_sync(0xffffffffu, C, o);
        const double Mp = __shfl_up_sync(0xffffffffu, Mr, o);
        if (m >= o) {
          C = fma(Mr, Cp, C);
          Mr = Mr * Mp;
        }
      }
      double Ce = __shfl_up_sync(0xffffffffu, C, 1), Me = __shfl_up_sync(0xffffffffu, Mr, 1);
      if (m == 0) {
        Ce = 0.0;
        Me = 1.0;
      }
      vk0 = __shfl_sync(0xffffffffu, vk0, 0);
      double vk = fma(Me, vk0, Ce);  // the value entering this lane's run
      double val[SV];
#pragma unroll
      for (int e = 0; e < SV; e++) {
        double v = fma(mm[e], vk, cc[e]);
        v = (FULL || ve[e]) ? v : 0.0;
        // lanes past the grid take part in the scan with unloaded operands: select, never multiply
        if (MODE == SW_BWD) acc += (FULL || ve[e]) ? c0[e] * v : 0.0;
        val[e] = v;
        vk = v;
      }
      POT3D_CHK(A.S, !any || (in_range(zr, A.z, (G.nr_loc + 2) * G.plane) &&
                              in_range(zr + SV - 1, A.z, (G.nr_loc + 2) * G.plane)), CHK_SWEEP_STORE);
#if POT3D_CHECK
      if (put_bot) {
        double sv[4];
        ldg4_cg(my_bot + (long long)ivt * SV, sv);
        POT3D_CHK(A.S, in_range(my_bot + (long long)ivt * SV + SV - 1, A.edge, A.edge_len), CHK_SWEEP_STORE);
        POT3D_CHK(A.S, is_sent(sv[0]) && is_sent(sv[1]) && is_sent(sv[2]) && is_sent(sv[3]), CHK_SLOT_REUSE);
      }
      if (put_rgt) {
        POT3D_CHK(A.S, in_range(my_rgt + (long long)ivt * 2, A.edge, A.edge_len), CHK_SWEEP_STORE);
        POT3D_CHK(A.S, is_sent(ldg_cg(my_rgt + (long long)ivt * 2)), CHK_SLOT_REUSE);
      }
#endif
      if (full) {
        if (rev)
          stg4(zr, val[3], val[2], val[1], val[0]);
        else
          stg4(zr, val[0], val[1], val[2], val[3]);
      } else if (any) {
        if (rev ? ve[3] : ve[0]) zr[0] = rev ? val[3] : val[0];
        if (rev ? ve[2] : ve[1]) zr[1] = rev ? val[2] : val[1];
        if (rev ? ve[1] : ve[2]) zr[2] = rev ? val[1] : val[2];
        if (rev ? ve[0] : ve[3]) zr[3] = rev ? val[0] : val[3];
      }
      if (put_bot) stg4_cg(my_bot + (long long)ivt * SV, val[0], val[1], val[2], val[3]);
      if (put_rgt) __stcg(my_rgt + (long long)ivt * 2, val[SV - 1]);
      double *xo = ((t & 1) ? xw + XB : xw) + (xo_me - xw);
      *reinterpret_cast<double2 *>(xo) = make_double2(val[0], val[1]);
      *reinterpret_cast<double2 *>(xo + 2) = make_double2(val[2], val[3]);
#pragma unroll
      for (int e = 0; e < SV; e++) wprev[e] = val[e];
    }
    zr += ostep;
    prefetch(U);  // step t + PD into this slot
  };

  const int nsteps = nb + SWJ - 1;
  prefetch(IC2<0>{});
  if (PD > 1) prefetch(IC2<(PD > 1 ? 1 : 0)>{});
  if (PD > 2) prefetch(IC2<(PD > 2 ? 2 : 0)>{});
  if (PD > 3) prefetch(IC2<(PD > 3 ? 3 : 0)>{});
#pragma unroll 1
  for (int t = 0; t < nsteps; t += PD) {
    step(IC2<0>{}, t);
    if (PD > 1) { if (t + 1 >= nsteps) break; step(IC2<(PD > 1 ? 1 : 0)>{}, t + 1); }
    if (PD > 2) { if (t + 2 >= nsteps) break; step(IC2<(PD > 2 ? 2 : 0)>{}, t + 2); }
    if (PD > 3) { if (t + 3 >= nsteps) break; step(IC2<(PD > 3 ? 3 : 0)>{}, t + 3); }
  }
  if (__syncthreads_or(proto) && tid == 0) atomicOr(&A.sync[1], 2);
  if (MODE == SW_BWD) {
    double v[1] = {acc}, tot[1];
    if (grid_sum<1>(v, A.partials, &A.S->counter[2], sred, tot, ticket, A.nblk * A.ntiles) && tid == 0) {
      if (A.finalize)
        finalize_rho(A.S, tot[0]);
      else if (A.peers)
        mail_post(A.peers, MAIL_C, tot[0], 0.0, mail_seq(A.S->epoch, A.S->iter), A.S);
      else
        A.local_sum[0] = tot[0];
    }
  }
}

// A batch (A.nrhs > 1): ticket t is problem t % nrhs's ticket t / nrhs, so the
// problems' wavefronts advance side by side and every wait is still on a tile of the
// same problem taken earlier; a stopped problem's CTAs leave after their ticket.
// CTAs per SM the row-scan sweeps are compiled for.  Measured (tools/gpu/sws2.sh): 16-row
// tiles at one CTA per SM beat 8-row tiles at one or two (medium 1477 vs 1520 / 1619 us
// per sweep pair, large 3665 vs 4399 / 3731 us, a 4-problem batch 1.80 vs 2.15 / 1.82 ms)
#ifndef POT3D_SWS_MINB
#define POT3D_SWS_MINB 1
#endif
template <int MODE>
__global__ void __launch_bounds__(SWT, POT3D_SWS_MINB) k_sweepS(SweepArgs A, int koff, int ntk4) {
  if (A.nrhs <= 1 && A.predicated && A.S->stop) return;
  __shared__ int s_ticket;
  __shared__ double sred[SWT / 32];
  if (threadIdx.x == 0) s_ticket = atomicAdd(&A.sync[0], 1);
  __syncthreads();
  int ticket = s_ticket;
  if (A.nrhs > 1) {
    const int q = ticket % A.nrhs;
    ticket /= A.nrhs;
    A.S += q;
    if (A.predicated && A.S->stop) return;
    A.r += q * A.vstride;
    A.z += q * A.vstride;
    A.partials += q * A.pstride;
    A.edge_len /= A.nrhs;
    A.edge += q * A.edge_len;
  }
  const int2 tl = A.order[ticket / A.nblk];
  const int kv_lo = koff + tl.y * SWK;
  const bool full = (tl.x + 1) * SWJ <= A.G.nt && kv_lo >= 0 && kv_lo + SWK <= A.G.np;
  if (full)
    sweepS_body<MODE, true>(A, koff, ntk4, ticket, sred);
  else
    sweepS_body<MODE, false>(A, koff, ntk4, ticket, sred);
}

__global__ void k_fill_u64(unsigned long long *a, long long n, unsigned long long v) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x)
    a[c] = v;
}

// periodic ghost columns of z (read by the TMA boxes of pass A)
__global__ void k_pc2_ghost(Grid G, double *a, const Scalars *S, int predicated, long long vstride) {
  S += blockIdx.y;  // a batch: problem blockIdx.y
  a += blockIdx.y * vstride;
  if (predicated && S->stop) return;
  const long long rows = (long long)G.nr_loc * G.nt;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < rows;
       c += (long long)gridDim.x * blockDim.x) {
    const int il = (int)(c / G.nt), j = (int)(c % G.nt);
    double *row = a + cidx(G, il, j, 0);
    row[-1] = row[G.np - 1];
    row[G.np] = row[0];
  }
}

static void *p_alloc(Pc2 *P, size_t bytes, void *(*alloc)(size_t, void *), void *actx) {
  void *p = nullptr;
  if (alloc)
    p = alloc(bytes, actx);
  else if (cudaMalloc(&p, bytes) != cudaSuccess)
    p = nullptr;
  if (p) {
    P->allocs.push_back(p);
    P->bytes += bytes;
  }
  return p;
}

int pc2_create(Pc2 **out, const Grid &G, int nblocks_local, const int *block_l0,
               void *(*alloc)(size_t, void *), void *actx, cudaStream_t s, int nrhs) {
  Pc2 *P = new Pc2();
  P->G = G;
  P->nrhs = std::max(nrhs, 1);
  P->nblk = nblocks_local;
  P->ntj = (G.nt + WJ - 1) / WJ;
  P->ntk = (G.np + WK - 1) / WK;
  P->ntiles = P->ntj * P->ntk;
  P->nsync = 2;
  {
    std::vector<int> l(block_l0, block_l0 + nblocks_local + 1);
    P->nbmax = 0;
    for (int q = 0; q < nblocks_local; q++) P->nbmax = std::max(P->nbmax, l[q + 1] - l[q]);
  }
  P->edge_len = (long long)P->nblk * P->ntiles * P->nbmax * (WJ + WK);
  P->bytes = 0;
  P->d_l0 = (int *)p_alloc(P, sizeof(int) * (nblocks_local + 1), alloc, actx);
  P->d_order = (int2 *)p_alloc(P, sizeof(int2) * P->ntiles, alloc, actx);
  P->d_sync = (int *)p_alloc(P, sizeof(int) * P->nsync, alloc, actx);
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  P->inv_d = (double *)p_alloc(P, sizeof(double) * cells, alloc, actx);
  P->edge = (double *)p_alloc(P, sizeof(double) * P->edge_len, alloc, actx);
  // run-vectorised sweep geometry (FWD and BWD share the tile grid: the larger one)
  P->koff_f = sweep4_koff(G.np, false);
  P->koff_b = sweep4_koff(G.np, true);
  P->ntj4 = (G.nt + SWJ - 1) / SWJ;
  P->ntk4 = std::max((G.np - P->koff_f + SWK - 1) / SWK, (G.np - P->koff_b + SWK - 1) / SWK);
  P->ntiles4 = P->ntj4 * P->ntk4;
  P->edge4_len = (long long)P->nblk * P->ntiles4 * P->nbmax * (SNR * SV + SWJ * 2) * P->nrhs;
  P->d_order4 = (int2 *)p_alloc(P, sizeof(int2) * P->ntiles4, alloc, actx);
  P->d_orderS = (int2 *)p_alloc(P, sizeof(int2) * P->ntiles4, alloc, actx);
  P->edge4 = (double *)p_alloc(P, sizeof(double) * P->edge4_len, alloc, actx);
  {
    const char *e = getenv("POT3D_PC2_SWEEP");
    P->scan = !(e && atoi(e) == 4);
  }
  if (!P->d_l0 || !P->d_order || !P->d_sync || !P->inv_d || !P->edge || !P->d_order4 || !P->d_orderS ||
      !P->edge4) {
    *out = P;
    return -1;
  }
  // the attribute is per function, shared by every context of the process: only raise it
  // (a smaller context created later must not shrink a larger one's allowance)
  static int nbmax_set = 0;
  nbmax_set = std::max(nbmax_set, P->nbmax);
  if (cudaFuncSetAttribute(k_sweep4<SW_FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(Sw4<SW_FWD>::SMEM + 16 * nbmax_set)) != cudaSuccess ||
      cudaFuncSetAttribute(k_sweep4<SW_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(Sw4<SW_BWD>::SMEM + 16 * nbmax_set)) != cudaSuccess ||
      cudaFuncSetAttribute(k_sweepS<SW_FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(Sw4<SW_FWD>::SMEM + 16 * nbmax_set)) != cudaSuccess ||
      cudaFuncSetAttribute(k_sweepS<SW_BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(Sw4<SW_BWD>::SMEM + 16 * nbmax_set)) != cudaSuccess) {
    *out = P;
    return -1;
  }
  // topological order: by estimated start step tj*WJ + tk*WK (both predecessors
  // start strictly earlier), ties by tj
  std::vector<int2> order;
  order.reserve(P->ntiles);
  for (int a = 0; a < P->ntj; a++)
    for (int c = 0; c < P->ntk; c++) order.push_back(make_int2(a, c));
  std::stable_sort(order.begin(), order.end(), [](const int2 &x, const int2 &y) {
    const int sx = x.x * WJ + x.y * WK, sy = y.x * WJ + y.y * WK;
    return sx != sy ? sx < sy : x.x < y.x;
  });
  std::vector<int2> order4;
  order4.reserve(P->ntiles4);
  for (int a = 0; a < P->ntj4; a++)
    for (int c = 0; c < P->ntk4; c++) order4.push_back(make_int2(a, c));
  std::stable_sort(order4.begin(), order4.end(), [](const int2 &x, const int2 &y) {
    const int sx = x.x * SWJ + x.y * SNR, sy = y.x * SWJ + y.y * SNR;
    return sx != sy ? sx < sy : x.x < y.x;
  });
  // k_sweepS: a tile's row waits for the same row and shell of the tile to its left
  // (one step) and for the bottom row of the tile above (SWJ steps)
  std::vector<int2> orderS(order4);
  std::stable_sort(orderS.begin(), orderS.end(), [](const int2 &x, const int2 &y) {
    const int sx = x.x * SWJ + x.y, sy = y.x * SWJ + y.y;
    return sx != sy ? sx < sy : x.x < y.x;
  });
  // everything on the context stream (the factor kernel runs there too)
  cudaMemcpyAsync(P->d_order, order.data(), sizeof(int2) * P->ntiles, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->d_order4, order4.data(), sizeof(int2) * P->ntiles4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->d_orderS, orderS.data(), sizeof(int2) * P->ntiles4, cudaMemcpyHostToDevice, s);
  k_fill_u64<<<1024, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(P->edge4), P->edge4_len, SENT);
  cudaMemcpyAsync(P->d_l0, block_l0, sizeof(int) * (nblocks_local + 1), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(P->inv_d, 0, sizeof(double) * cells, s);
  k_fill_u64<<<1024, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(P->edge), P->edge_len, SENT);
  *out = P;
  return cudaStreamSynchronize(s) == cudaSuccess ? 0 : -1;
}

static SweepArgs sweep_args(Pc2 *P, const Metrics &M, Scalars *S, const double *r, double *z,
                            double *partials, int predicated, int finalize, double *local_sum) {
  SweepArgs a{};
  a.G = P->G;
  a.M = M;
  a.S = S;
  a.l0 = P->d_l0;
  a.order = P->d_order;
  a.sync = P->d_sync;
  a.nblk = P->nblk;
  a.ntj = P->ntj;
  a.ntk = P->ntk;
  a.ntiles = P->ntiles;
  a.r = r;
  a.z = z;
  a.inv_d = P->inv_d;
  a.partials = partials;
  a.edge = P->edge;
  a.edge_len = P->edge_len;
  a.nbmax = P->nbmax;
  a.predicated = predicated;
  a.finalize = finalize;
  a.local_sum = local_sum;
  return a;
}

int pc2_factor(Pc2 *P, const Metrics &M, cudaStream_t s, double *min_pivot_host) {
  cudaMemsetAsync(P->d_sync, 0, sizeof(int) * P->nsync, s);
  SweepArgs a = sweep_args(P, M, nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr);
  k_factor<<<P->nblk * P->ntiles, WT, 0, s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return -1;
  int flags[2];
  cudaMemcpyAsync(flags, P->d_sync, sizeof(int) * 2, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  if (getenv("POT3D_DEBUG")) fprintf(stderr, "POT3D_DEBUG pc2_factor flags %d\n", flags[1]);
  if (flags[1] & 2) return -1;             // handoff protocol error
  *min_pivot_host = (flags[1] & 1) ? 0.0 : 1.0;  // breakdown (pivot <= 1e-300) -> 0
  return 0;
}

// z = M^-1 r; returns the number of kernels launched (memsets excluded) or -1.
static thread_local std::string g_pc2_err;

int pc2_apply(Pc2 *P, const Metrics &M, Scalars *S, const double *r, double *z, double *partials,
              int finalize, double *local_sum, cudaStream_t s, bool iteration, const PeerTab *peers,
              int nrhs, long long vstride, long long pstride) {
  const int pred = iteration ? 1 : 0;
  const int nk = std::max(nrhs, 1);
  if (nk > P->nrhs || (nk > 1 && !P->scan)) {
    g_pc2_err = "PC2 batch: the sweeps were set up for fewer problems (or POT3D_PC2_SWEEP=4)";
    return -1;
  }
  SweepArgs a = sweep_args(P, M, S, r, z, partials, pred, finalize, local_sum);
  a.nrhs = nk;
  a.vstride = vstride;
  a.pstride = pstride;
  a.peers = iteration ? peers : nullptr;
  if (!iteration) a.finalize = 0, a.local_sum = local_sum;
  // run-vectorised / row-scan sweeps: their own tile order and edge slots
  a.order = P->scan ? P->d_orderS : P->d_order4;
  a.edge = P->edge4;
  a.edge_len = P->edge4_len / P->nrhs * nk;  // the slots of the nk problems
  a.ntiles = P->ntiles4;
  cudaMemsetAsync(P->d_sync, 0, sizeof(int), s);  // ticket only (flags accumulate)
  if (P->scan)
    k_sweepS<SW_FWD><<<P->nblk * P->ntiles4 * nk, SWT, Sw4<SW_FWD>::SMEM + 16 * P->nbmax, s>>>(a, P->koff_f,
                                                                                               P->ntk4);
  else
    k_sweep4<SW_FWD><<<P->nblk * P->ntiles4, SWT, Sw4<SW_FWD>::SMEM + 16 * P->nbmax, s>>>(a, P->koff_f, P->ntk4);
  cudaMemsetAsync(P->d_sync, 0, sizeof(int), s);
  if (P->scan)
    k_sweepS<SW_BWD><<<P->nblk * P->ntiles4 * nk, SWT, Sw4<SW_BWD>::SMEM + 16 * P->nbmax, s>>>(a, P->koff_b,
                                                                                               P->ntk4);
  else
    k_sweep4<SW_BWD><<<P->nblk * P->ntiles4, SWT, Sw4<SW_BWD>::SMEM + 16 * P->nbmax, s>>>(a, P->koff_b, P->ntk4);
  const Grid &G = P->G;
  k_pc2_ghost<<<dim3((unsigned)std::min<long long>(((long long)G.nr_loc * G.nt + 255) / 256, 4096), nk), 256,
                0, s>>>(G, z, S, pred, vstride);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_pc2_err = std::string("PC2 sweep launch: ") + cudaGetErrorString(e);
    return -1;
  }
  return 3;
}

const char *pc2_last_error() { return g_pc2_err.c_str(); }

// flags of the last sweeps (1: pivot breakdown, 2: handoff protocol error); a
// protocol error re-arms every edge slot so the next solve starts clean
int pc2_status(Pc2 *P, cudaStream_t s) {
  int f = 0;
  cudaMemcpyAsync(&f, P->d_sync + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (f & 2) {
    k_fill_u64<<<1024, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(P->edge), P->edge_len, SENT);
    k_fill_u64<<<1024, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(P->edge4), P->edge4_len, SENT);
    cudaMemsetAsync(P->d_sync + 1, 0, sizeof(int), s);
    cudaStreamSynchronize(s);
  }
  return f;
}

void pc2_destroy(Pc2 *P, void (*fr)(void *, void *), void *actx) {
  if (!P) return;
  for (void *p : P->allocs) {
    if (fr)
      fr(p, actx);
    else
      cudaFree(p);
  }
  delete P;
}

size_t pc2_bytes(const Pc2 *P) { return P ? P->bytes : 0; }
int pc2_kernels_per_apply(const Pc2 *P) { return P ? 3 : 0; }

}  // namespace pot3d
