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
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device_common.cuh"

namespace pot3d {

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
  int nbmax;
  int predicated;    // skip when the PCG loop has stopped
  int finalize;      // BWD: 1 single rank (rho/beta), 0 local_sum
  double *local_sum;
  const PeerTab *peers;  // BWD, nranks > 1 with peer memory: post r.z to every mailbox
};

// Tile-edge handoff without flags or fences: the bottom row / right column of
// every tile is also written into an edge buffer whose slots hold a sentinel
// (a signalling-NaN bit pattern arithmetic never produces) until the producer
// stores the value; the single consumer prefetches the slot PD steps ahead with
// ld.global.cv, polls only while it still reads the sentinel, and re-arms it.
constexpr unsigned SENT32 = 0x7FF57FF5u;
constexpr unsigned long long SENT = 0x7FF57FF57FF57FF5ull;
constexpr long long SPIN_LIMIT = 1ll << 26;  // bounded waits: a protocol error never hangs the GPU
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

#ifndef POT3D_SWEEP_MINB
#define POT3D_SWEEP_MINB 1
#endif
template <int MODE>
__global__ void __launch_bounds__(WT, POT3D_SWEEP_MINB) k_sweep(SweepArgs A) {
  const Grid &G = A.G;
  const Metrics &M = A.M;
  if (A.predicated && A.S->stop) return;
  __shared__ double sw[2][WJ][WK];
  __shared__ int s_ticket;
  __shared__ double sred[WT / 32];
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
  const bool rev = (MODE == SW_BWD);
  // virtual coordinates (dependencies on iv-1, jv-1, kv-1); real = mirrored for BWD
  const int jv = tl.x * WJ + jj, kv = tl.y * WK + kk;
  const bool valid = (jv < G.nt) && (kv < G.np);
  const int j = rev ? G.nt - 1 - jv : jv;
  const int k = rev ? G.np - 1 - kv : kv;
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
  // couplings to the virtual predecessors (zero across the pole / the dropped wrap)
  const double ct = rev ? atp : atm;                                              // x dr_i dp_k
  const double cp = rev ? ((k < G.np - 1) ? app : 0.0) : ((k > 0) ? apm : 0.0);  // x dr_i q_j
  const long long o_base = cidx(G, rev ? l1 - 1 : l0, jc, kc);
  const long long o_step = rev ? -G.plane : G.plane;  // one virtual shell
  const int ig_base = G.i0 + (rev ? l1 - 1 : l0), ig_step = rev ? -1 : 1;

  // prefetch ring: operands of the cell this thread handles at step t+PD
  double ra[PD], rb[PD], rc[PD], rnj[PD], rnk[PD];
  auto fetch = [&](int ts, double &xa, double &xb, double &xc, double &xj, double &xk) {
    const int iv = ts - jj - kk;
    xa = xb = xc = 0.0;
    xj = xk = 0.0;
    if (valid && iv >= 0 && iv < nb) {
      const long long o = o_base + (long long)iv * o_step;
      if (MODE == SW_FWD) {
        xa = __ldg(A.r + o);
        xb = __ldg(A.inv_d + o);
      } else if (MODE == SW_BWD) {
        xa = __ldcg(A.z + o);   // w of this cell (forward sweep output)
        xb = __ldg(A.inv_d + o);
        xc = __ldg(A.r + o);    // r of this cell for the r.z partial
      }
      // neighbour-tile values: prefetched, re-polled at use if still the sentinel
      if (need_j) xj = ld_poll(up_bot + iv);
      if (need_k) xk = ld_poll(lf_rgt + iv);
    }
  };
  bool proto = false;
#pragma unroll
  for (int u = 0; u < PD; u++) fetch(u, ra[u], rb[u], rc[u], rnj[u], rnk[u]);

  double wprev = 0.0, acc = 0.0;
  bool bad = false;
  for (int t0 = 0; t0 < nsteps; t0 += PD) {
#pragma unroll
    for (int u = 0; u < PD; u++) {
      const int t = t0 + u;
      if (t >= nsteps) break;
      __syncthreads();  // step t-1 complete in this CTA (shared double buffer)
      const double a0 = ra[u], b0 = rb[u], c0 = rc[u];
      double nj = rnj[u], nk = rnk[u];
      fetch(t + PD, ra[u], rb[u], rc[u], rnj[u], rnk[u]);
      const int ivt = t - jj - kk;  // virtual local shell of this thread at step t
      if (valid && ivt >= 0 && ivt < nb) {
        if (need_j) {  // value of the tile above (virtual), produced at its step t+WJ-1
          long long spins = 0;
          while (is_sent(nj) && spins++ < SPIN_LIMIT) nj = ld_poll(up_bot + ivt);
          proto |= is_sent(nj);
          __stcg(reinterpret_cast<unsigned long long *>(up_bot + ivt), SENT);  // re-arm
        }
        if (need_k) {
          long long spins = 0;
          while (is_sent(nk) && spins++ < SPIN_LIMIT) nk = ld_poll(lf_rgt + ivt);
          proto |= is_sent(nk);
          __stcg(reinterpret_cast<unsigned long long *>(lf_rgt + ivt), SENT);
        }
        const long long o = o_base + (long long)ivt * o_step;
        const int ig = ig_base + ivt * ig_step;
        const double dr = __ldg(M.dr + ig);
        const double vi = (ivt > 0) ? wprev : 0.0;
        const double vj = (jj > 0) ? sw[(t - 1) & 1][jj - 1][kk] : (need_j ? nj : 0.0);
        const double vk = (kk > 0) ? sw[(t - 1) & 1][jj][kk - 1] : (need_k ? nk : 0.0);
        const double cr = (ivt > 0) ? (rev ? __ldg(M.arp + ig) : __ldg(M.arm + ig)) : 0.0;
        const double Ar = cr * g * dpk, At = dr * ct * dpk, Ap = dr * q * cp;
        double val;
        if (MODE == SW_FACTOR) {
          const double diag = dpk * (g * (__ldg(M.arp + ig) + __ldg(M.arm + ig) + __ldg(M.ss + ig)) +
                                     dr * (atp + atm)) + dr * q * (app + apm);
          // the wrap coupling and the inter-block couplings are dropped from L/U,
          // the full diagonal is kept (A11)
          const double d = diag - Ar * Ar * vi - At * At * vj - Ap * Ap * vk;
          bad |= !(d > 1e-300);
          val = 1.0 / d;
          A.inv_d[o] = val;
        } else if (MODE == SW_FWD) {
          val = (a0 + Ar * vi + At * vj + Ap * vk) * b0;
          A.z[o] = val;
        } else {
          val = a0 + b0 * (Ar * vi + At * vj + Ap * vk);
          A.z[o] = val;
          acc += c0 * val;
        }
        if (put_bot) __stcg(my_bot + ivt, val);
        if (put_rgt) __stcg(my_rgt + ivt, val);
        wprev = val;
        sw[t & 1][jj][kk] = val;
      }
    }
  }
  if (__syncthreads_or(proto) && tid == 0) atomicOr(&A.sync[1], 2);  // protocol error
  if (MODE == SW_FACTOR) {
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&A.sync[1], 1);
  }
  if (MODE == SW_BWD) {
    double v[1] = {acc}, tot[1];
    // partials indexed by ticket (tile identity), not blockIdx: a fixed summation order
    if (grid_sum<1>(v, A.partials, &A.S->counter[2], sred, tot, ticket) && tid == 0) {
      if (A.finalize)
        finalize_rho(A.S, tot[0]);
      else if (A.peers)
        mail_post(A.peers, MAIL_C, tot[0], 0.0, mail_seq(A.S->epoch, A.S->iter));
      else
        A.local_sum[0] = tot[0];
    }
  }
}

__global__ void k_fill_u64(unsigned long long *a, long long n, unsigned long long v) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x)
    a[c] = v;
}

// periodic ghost columns of z (read by the TMA boxes of pass A)
__global__ void k_pc2_ghost(Grid G, double *a, const Scalars *S, int predicated) {
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
               void *(*alloc)(size_t, void *), void *actx, cudaStream_t s) {
  Pc2 *P = new Pc2();
  P->G = G;
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
  if (!P->d_l0 || !P->d_order || !P->d_sync || !P->inv_d || !P->edge) {
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
  // everything on the context stream (the factor kernel runs there too)
  cudaMemcpyAsync(P->d_order, order.data(), sizeof(int2) * P->ntiles, cudaMemcpyHostToDevice, s);
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
  a.nbmax = P->nbmax;
  a.predicated = predicated;
  a.finalize = finalize;
  a.local_sum = local_sum;
  return a;
}

int pc2_factor(Pc2 *P, const Metrics &M, cudaStream_t s, double *min_pivot_host) {
  cudaMemsetAsync(P->d_sync, 0, sizeof(int) * P->nsync, s);
  SweepArgs a = sweep_args(P, M, nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr);
  k_sweep<SW_FACTOR><<<P->nblk * P->ntiles, WT, 0, s>>>(a);
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
int pc2_apply(Pc2 *P, const Metrics &M, Scalars *S, const double *r, double *z, double *partials,
              int finalize, double *local_sum, cudaStream_t s, bool iteration, const PeerTab *peers) {
  const int pred = iteration ? 1 : 0;
  SweepArgs a = sweep_args(P, M, S, r, z, partials, pred, finalize, local_sum);
  a.peers = iteration ? peers : nullptr;
  cudaMemsetAsync(P->d_sync, 0, sizeof(int), s);  // ticket only (flags accumulate)
  k_sweep<SW_FWD><<<P->nblk * P->ntiles, WT, 0, s>>>(a);
  cudaMemsetAsync(P->d_sync, 0, sizeof(int), s);
  if (!iteration) a.finalize = 0, a.local_sum = local_sum;
  k_sweep<SW_BWD><<<P->nblk * P->ntiles, WT, 0, s>>>(a);
  const Grid &G = P->G;
  k_pc2_ghost<<<(unsigned)std::min<long long>(((long long)G.nr_loc * G.nt + 255) / 256, 4096), 256, 0,
                s>>>(G, z, S, pred);
  if (cudaGetLastError() != cudaSuccess) return -1;
  return 3;
}

// flags of the last sweeps (1: pivot breakdown, 2: handoff protocol error); a
// protocol error re-arms every edge slot so the next solve starts clean
int pc2_status(Pc2 *P, cudaStream_t s) {
  int f = 0;
  cudaMemcpyAsync(&f, P->d_sync + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  if (f & 2) {
    k_fill_u64<<<1024, 256, 0, s>>>(reinterpret_cast<unsigned long long *>(P->edge), P->edge_len, SENT);
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
