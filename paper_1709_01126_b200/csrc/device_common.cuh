// device_common.cuh -- device helpers shared by kernels.cu, passes.cu, pc2.cu:
// deterministic reductions (a6), device-side scalar updates (a10), metric
// helpers, a Newton-corrected fp64 quotient and cp.async wrappers.
#pragma once
#include "pot3d_internal.cuh"

namespace pot3d {

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
__device__ __forceinline__ bool grid_sum(double (&v)[N], double *partials, unsigned int *counter, double *sred,
                         double (&tot)[N], int bid = -1, int nb = -1) {
  __shared__ bool s_last;
  // bid: a deterministic identity of the block's work (default: blockIdx); nb:
  // the number of blocks of the reduction (several launches may share it)
  if (nb < 0) nb = gridDim.x * gridDim.y;
  if (bid < 0) bid = blockIdx.x + gridDim.x * blockIdx.y;
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
__device__ __forceinline__ void finalize_alpha(Scalars *S, double sigma) {
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
__device__ __forceinline__ void finalize_beta(Scalars *S, double rz, double rr, double *hist) {
  long long it = S->iter + 1;
  S->iter = it;
  S->rr = rr;
  double rn = sqrt(rr);
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
  S->beta = rz / S->rho;
  S->rho = rz;
}

// PC2 split of finalize_beta: ||r|| test after pass B, rho/beta after the sweeps.
__device__ __forceinline__ void finalize_rr(Scalars *S, double rr, double *hist) {
  long long it = S->iter + 1;
  S->iter = it;
  S->rr = rr;
  double rn = sqrt(rr);
  if (hist && it < S->hist_len) hist[it] = rn / S->bnorm;
  S->alpha_prev = S->alpha;
  if (rn <= S->rtol * S->bnorm) {
    S->stop = 1;
    S->status = 0;
  } else if (it >= S->maxit) {
    S->stop = 1;
    S->status = 1;
  }
}
__device__ __forceinline__ void finalize_rho(Scalars *S, double rz) {
  S->beta = rz / S->rho;
  S->rho = rz;
}
// ---------------------------------------------------------------------------
// Peer-memory exchange (nranks > 1, CUDA IPC over NVLink).  A producer stores its
// values into the destination's mailbox and then the sequence number with a
// system-scope release; a consumer spins on the sequence number with a
// system-scope acquire.  Every wait is bounded (XFER_TIMEOUT_NS of globaltimer)
// and gives up at once when another waiter has already expired.
// ---------------------------------------------------------------------------
constexpr unsigned long long XFER_TIMEOUT_NS = 20000000000ull;  // 20 s

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// generic-proxy data acquired from a peer, about to be read by TMA (async proxy)
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// this rank's (v0, v1) of `kind` into every rank's mailbox: all value stores, ONE
// system-scope fence, then the sequence numbers (fence + relaxed store = release);
// one NVLink round trip on the critical path instead of one per rank
__device__ __forceinline__ void mail_post(const PeerTab *T, int kind, double v0, double v1,
                                          unsigned long long seq, Scalars *S) {
  const int me = T->rank;
#if POT3D_CHECK
  for (int r = 0; r < T->nranks; r++) {  // slot reuse: the previous post of this slot is older
    const unsigned long long old = ld_acquire_sys(&T->mail[r]->e[kind][me].seq);
    if (!(old < seq)) atomicOr(&S->check, (unsigned)CHK_MAIL_ORDER);
  }
#endif
  for (int r = 0; r < T->nranks; r++) {
    MailEntry *e = &T->mail[r]->e[kind][me];
    *reinterpret_cast<volatile double *>(&e->v0) = v0;
    *reinterpret_cast<volatile double *>(&e->v1) = v1;
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int r = 0; r < T->nranks; r++) st_relaxed_sys(&T->mail[r]->e[kind][me].seq, seq);
}

// spin until *flag == seq; false (and S->xfer_error set) when the wait expired
__device__ __forceinline__ bool xfer_wait(const unsigned long long *flag, unsigned long long seq,
                                          Scalars *S) {
  if (ld_acquire_sys(flag) == seq) return true;
  const unsigned long long t0 = global_ns();
  volatile int *err = &S->xfer_error;
  while (ld_acquire_sys(flag) != seq) {
    if (*err || global_ns() - t0 > XFER_TIMEOUT_NS) {
      *err = 1;
      return false;
    }
  }
  return true;
}

// diagnostics (POT3D_TRACE): %globaltimer of an event of the current iteration
__device__ __forceinline__ void trace_mark(Scalars *S, int slot) {
  if (S->trace) S->trace[(S->iter & 63) * 16 + slot] = global_ns();
}
__device__ __forceinline__ void trace_max(Scalars *S, int slot) {
  if (S->trace) atomicMax(&S->trace[(S->iter & 63) * 16 + slot], global_ns());
}

// every rank's entry of `kind` for seq, summed in rank order (bit-identical on all ranks);
// the first pass issues all ranks' acquire loads back to back (one round trip when
// every rank has already posted), stragglers are then waited for one by one
__device__ __forceinline__ bool mail_collect(const PeerTab *T, int kind, unsigned long long seq,
                                             Scalars *S, double &s0, double &s1) {
  const Mailbox *mb = T->mail[T->rank];
  const int n = T->nranks;
  unsigned long long got[MAXR];
#pragma unroll
  for (int r = 0; r < MAXR; r++)
    if (r < n) got[r] = ld_acquire_sys(&mb->e[kind][r].seq);
  s0 = 0.0;
  s1 = 0.0;
#pragma unroll
  for (int r = 0; r < MAXR; r++) {
    if (r >= n) break;
    const MailEntry *e = &mb->e[kind][r];
    if (got[r] != seq && !xfer_wait(&e->seq, seq, S)) return false;
    s0 += *reinterpret_cast<const volatile double *>(&e->v0);
    s1 += *reinterpret_cast<const volatile double *>(&e->v1);
  }
  return true;
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


// The Jacobi diagonal of a cell, in one fixed evaluation order for every kernel
// (pass A, pass B, the edge-shell kernel, the init dots): diag = dp_k a + b (app_k + apm_k).
__device__ __forceinline__ double diag_at(double dpk, const DiagRow &d, double appk, double apmk) {
  return fma(dpk, d.a, d.b * (appk + apmk));
}
// r / d for d > 0 (normal): approximate reciprocal (MUFU.RCP64H, ~2^-20), one
// Newton step (~2^-40), product, then one remainder correction
// q1 = q0 + y (r - d q0), which leaves the quotient within ~1 ulp of the
// correctly rounded r/d at 6 fp64 operations instead of the DDIV sequence.
__device__ __forceinline__ double fdiv(double r, double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  double q = r * y;
  double rem = fma(-d, q, r);
  return fma(y, rem, q);
}

// z = D^-1 r, the same corrected quotient in every kernel (pass A, pass B, the
// edge-shell kernel, the init dots), so a ghost copy equals the owner's value bitwise
__device__ __forceinline__ double jacobi(double r, double dk) { return fdiv(r, dk); }

// cp.async (LDGSTS) with zero-fill: copies src_bytes of 16 (8) and fills the
// rest of the destination with zeros; src_bytes = 0 reads nothing.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16s(unsigned s, const void *gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8s(unsigned s, const void *gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// ---- mbarrier + TMA (cp.async.bulk.tensor) ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 3-D tiled TMA load of the box at (c0 inner, c1, c2 outer) into smem; bytes land
// on `bar` (complete_tx).  Out-of-bounds elements are zero-filled.
// Programmatic dependent launch: a kernel launched with the PDL attribute may start
// while its predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op without the attribute), and
// pdl_trigger() lets this grid's successor launch once every block has called it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void *smem_dst, const void *map, uint64_t *bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];\n" ::"r"(smem_u32(smem_dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The two edge shells of p_k = z + beta p_{k-1} (z the stored preconditioned
// residual: PC1's D^-1 r buffer or PC2's sweep output) by aligned column pairs (physical
// 2m, 2m+1 = logical k = 2m-1, 2m; 16-B loads and stores), stored locally and into
// the neighbours' ghost shells (peer memory, same [il+1][j][c] layout shifted by
// whole planes); the ghost columns (k = -1, np) are computed like cells from their
// duplicated inputs, exactly as pass A does.  Block-wide call over blocks
// bid = 0 .. nblocks-1; returns true in the block that completed last (after every
// block's stores were released system-wide), which then raises the halo flags.
__device__ __forceinline__ bool edge_shells(const Grid &G, const Metrics &M, Scalars *S,
                                            const double *src, const double *p_old, double *p_new,
                                            const PeerTab *peers, int parity_new,
                                            double beta, int bid, int nblocks, bool work = true) {
  // peers == nullptr (NCCL exchange): local stores only, the caller sends the shells
  double *lo = peers ? peers->p_lo[parity_new] : nullptr, *hi = peers ? peers->p_hi[parity_new] : nullptr;
  if (lo) lo += (long long)peers->nr_lo * G.plane;
  if (hi) hi -= (long long)G.nr_loc * G.plane;
  const int npair = (G.np + 2 + 1) / 2;  // pairs covering physical columns 0 .. np+1
  const long long rows = (long long)G.nt * npair;
  const long long npairs = work ? 2 * rows : 0;
  for (long long c = bid * (long long)blockDim.x + threadIdx.x; c < npairs;
       c += (long long)nblocks * blockDim.x) {
    const int sidx = (int)(c / rows);
    const long long t = c - sidx * rows;
    const int j = (int)(t / npair), m = (int)(t - (long long)j * npair);
    const int il = sidx == 0 ? 0 : G.nr_loc - 1;
    const long long o = (long long)(il + 1) * G.plane + (long long)j * G.PK + 2 * m;  // physical 2m
    const double2 sv = *reinterpret_cast<const double2 *>(src + o);
    const double2 pv = *reinterpret_cast<const double2 *>(p_old + o);
    double v[2];
    v[0] = fma(beta, pv.x, sv.x);  // the same arithmetic as pass A
    v[1] = fma(beta, pv.y, sv.y);
    const bool both = 2 * m + 1 <= G.np + 1;  // physical 2m+1 still a ghost or a cell
    double *rem = sidx == 0 ? lo : hi;
    // the neighbour's ghost shell: rank-1's top ghost (its shell nr_lo), rank+1's bottom (0)
    POT3D_CHK(S, !rem || (sidx == 0 ? in_range(rem + o, peers->p_lo[parity_new] + (long long)(peers->nr_lo + 1) * G.plane, G.plane)
                                    : in_range(rem + o, peers->p_hi[parity_new], G.plane)), CHK_PEER_STORE);
    if (both) {
      *reinterpret_cast<double2 *>(p_new + o) = make_double2(v[0], v[1]);
      if (rem) *reinterpret_cast<double2 *>(rem + o) = make_double2(v[0], v[1]);
    } else {
      p_new[o] = v[0];
      if (rem) rem[o] = v[0];
    }
  }
  if (!peers) return false;
  __shared__ bool s_edge_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this block's peer stores, before the count
    s_edge_last = atomicAdd(&S->counter[4], 1u) == (unsigned)nblocks - 1;
  }
  __syncthreads();
  return s_edge_last;
}
// spin until *flag >= seq (a sequence that only grows: PC3's d halo flags)
__device__ __forceinline__ bool xfer_wait_ge(const unsigned long long *flag, unsigned long long seq,
                                             Scalars *S) {
  if (ld_acquire_sys(flag) >= seq) return true;
  const unsigned long long t0 = global_ns();
  volatile int *err = &S->xfer_error;
  while (ld_acquire_sys(flag) < seq) {
    if (*err || global_ns() - t0 > XFER_TIMEOUT_NS) {
      *err = 1;
      return false;
    }
  }
  return true;
}
// PC3: the neighbours' d-halo flags (caller: the last edge block, one thread)
__device__ __forceinline__ void raise_dhalo_flags(const PeerTab *peers, unsigned long long seq) {
  __threadfence_system();
  if (peers->rank > 0) st_relaxed_sys(&peers->mail[peers->rank - 1]->dhalo[1], seq);
  if (peers->rank < peers->nranks - 1) st_relaxed_sys(&peers->mail[peers->rank + 1]->dhalo[0], seq);
}
// the d-halo sequence of Chebyshev vector d_s of iteration S->iter: grows with both
__device__ __forceinline__ unsigned long long dhalo_seq(const Scalars *S, int s) {
  return mail_seq(S->epoch, S->iter * 8 + s + 1);
}

// neighbours' halo flags for seq (caller: the last block of edge_shells, one thread)
__device__ __forceinline__ void raise_halo_flags(const PeerTab *peers, unsigned long long seq) {
  __threadfence_system();  // + relaxed stores = release of every block's ghost stores
  if (peers->rank > 0) st_relaxed_sys(&peers->mail[peers->rank - 1]->halo[1], seq);
  if (peers->rank < peers->nranks - 1) st_relaxed_sys(&peers->mail[peers->rank + 1]->halo[0], seq);
}

}  // namespace pot3d
