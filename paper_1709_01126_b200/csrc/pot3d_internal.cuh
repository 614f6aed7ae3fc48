// pot3d_internal.cuh -- device data layout and kernel interfaces of libpot3d.
//
// Layout in HBM:
//   cell arrays   [il + 1][j][k], il in [-1, nr_loc] (one ghost shell on each r
//                 side), phi fastest with row pitch PK = round_up(np, 16)
//                 doubles so that every row starts on a 128-byte line.
//                 A theta-phi shell is contiguous: the r-slab halo is one
//                 cudaMemcpy-able / NCCL-sendable block.
//   1-D metrics   per axis, global indices (r) / plain (theta, phi), fp64.
//
// The operator (P:62-77 with the full metric A1, volume-scaled A3, A = -V lap A4)
// is never stored: every coupling is a product of 1-D factors,
//   A^r_{i+1/2,j,k} = arp[i] * g[j] * dp[k]      (arp[i] = rf[i+1]^2 / drh[i+1/2])
//   A^t_{i,j+1/2,k} = dr[i] * atp[j] * dp[k]     (atp[j] = sin tf[j+1] / dth[j+1/2])
//   A^p_{i,j,k+1/2} = dr[i] * q[j] * app[k]      (q[j] = dt[j]/sin tc[j], app[k] = 1/dph[k+1/2])
//   S_{i,j,k}       = ss[i] * g[j] * dp[k]       (source surface, last shell: 2 r1^2/dr)
// with g[j] = sin(tc[j]) dt[j], arm[i] = arp[i-1] (0 at r0: homogeneous Neumann,
// A6), atm[j] = atp[j-1] (0 at the poles, A5), apm[k] = app[k-1] (periodic).
// (A p)_m = sum_f A_f (p_m - p_nbr) + S_m p_m,  diag_m = sum_f A_f + S_m.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pot3d {

// Fused-pass tiling (passes.cu): a block owns TJ interior theta rows x TK phi
// columns and marches along r; one warp per haloed row (TR = TJ + 2 rows:
// the rows above/below the tile are loaded and transformed by warps 0 and
// TR-1), each lane two phi-adjacent cells (128-bit fp64 accesses).
#ifndef POT3D_NS_A
#define POT3D_NS_A 3            // pass A is unrolled by 3: NS_A must be 3
#endif
#ifndef POT3D_NS_B
#define POT3D_NS_B 4
#endif
#ifndef POT3D_MINB
#define POT3D_MINB 2
#endif
constexpr int TK = 64;          // phi columns per tile: lane l owns logical columns
                                // k0-1+2l, k0+2l (k0 = 64 * tile column); the halo columns
                                // k0-2 and k0+63 come with the staged box
#ifndef POT3D_TJ
#define POT3D_TJ 14
#endif
constexpr int TJ = POT3D_TJ;    // interior theta rows per tile
constexpr int TR = TJ + 2;      // haloed rows
// chunks of the fused passes stage their r-metric factors for at most
// POT3D_PLMAX planes (chunk length + 2) in shared memory
#ifndef POT3D_PLMAX
#define POT3D_PLMAX 320
#endif
#ifndef POT3D_RPW
#define POT3D_RPW 2
#endif
constexpr int RPW = POT3D_RPW;  // haloed rows per warp (each lane: RPW rows x 2 phi cells)
constexpr int NWARPS = TR / RPW;
constexpr int NTHREADS = NWARPS * 32;
constexpr int SROW = 68;        // smem row: index i <-> logical column k0-3+i (1..66 used)
constexpr int TKB = 64;         // width of the interior boxes (r, x): logical k0-1 .. k0+62
constexpr int NS_A = POT3D_NS_A; // cp.async stages of pass A (NS_A-1 planes in flight)
constexpr int NS_B = POT3D_NS_B; // cp.async stages of pass B (NS_B-2 planes in flight)
constexpr int PASS_MINB = POT3D_MINB;  // resident blocks per SM the passes are compiled for
// dynamic shared memory of the passes (bytes)
constexpr int SMEM_A = (2 * NS_A + 3) * TR * SROW * 8 + 128;  // + mbarriers
constexpr int SMEM_B = NS_B * (TR * SROW + 2 * TJ * TKB) * 8 + 128;

// single-reduction CG1 passes (cg1.cu): K1 stages the haloed u box and the p, s, x
// interior boxes (NS_C stages, one plane in flight), K2 the haloed u box (NS_D stages)
constexpr int NS_C = 3;
constexpr int NS_D = 4;
constexpr int SMEM_C1 = NS_C * (TR * SROW + 3 * TJ * TKB) * 8 + 128;
constexpr int SMEM_C2 = NS_D * TR * SROW * 8 + 128;
// PC3 Chebyshev steps (poly.cu): the haloed d box and the res, z (and r) interior boxes
constexpr int SMEM_P = NS_C * (TR * SROW + 3 * TJ * TKB) * 8 + 128;
constexpr int POLY_MMAX = 8;  // most Chebyshev steps per PC3 apply

struct Metrics {
  // r (global index, size nr)
  const double *arp, *arm, *dr, *ss;
  // theta (size nt)
  const double *g, *atp, *atm, *q;
  // phi (size np)
  const double *dp, *app, *apm;
};

// Device-resident PCG scalars (A9).  One instance per context.
struct Scalars {
  double rho;        // r.z of the current residual
  double alpha;      // step of the current iteration
  double alpha_prev; // step applied to x lazily in the next pass A
  double beta;       // p_k = z_k + beta p_{k-1}
  double sigma;      // p.Ap
  double rr;         // ||r||^2
  double bnorm;      // ||b||
  double rtol;
  double pad0;
  long long iter;    // completed alpha-updates
  long long maxit;
  int stop;          // 1: loop finished (converged, maxit, error)
  int status;        // 0 ok / 1 not converged / -4 indefinite
  unsigned int counter[6]; // last-block counters
  unsigned long long epoch;  // solve number (peer-memory sequence numbers)
  int xfer_error;    // peer-memory wait expired
  int pend_b;        // peer-memory PC1: pass B posted its sums; the next edge-shell kernel
                     // finalises them (convergence test, beta) before it builds p_k
  unsigned long long *trace;  // POT3D_TRACE: [64 iterations][16] %globaltimer marks, or null
  long long hist_len;         // entries of the residual-history buffer (writes beyond are dropped)
  unsigned int check;         // POT3D_CHECK builds: violated invariants (CHK_* bits)
};

// Checked builds (-DPOT3D_CHECK=1, tests/test_checked_build.py): device-side bounds and
// protocol invariants recorded in Scalars::check, reported by pot3d_solve as an error.
// (compute-sanitizer is not available on the GPU pool; this is its stand-in.)
#ifndef POT3D_CHECK
#define POT3D_CHECK 0
#endif
enum CheckBit {
  CHK_PASS_STORE = 1,    // a fused pass stored outside its cell array
  CHK_SWEEP_STORE = 2,   // a PC2 sweep stored outside z / its edge slots
  CHK_SLOT_REUSE = 4,    // a PC2 producer found its edge slot not yet consumed (re-armed)
  CHK_PEER_STORE = 8,    // an edge shell landed outside the neighbour's ghost shell
  CHK_MAIL_ORDER = 16,   // a mailbox sequence number did not increase
  CHK_CG1_STORE = 32     // a CG1 pass stored outside its arrays
};
#if POT3D_CHECK
#define POT3D_CHK(S, cond, bit)                                   \
  do {                                                            \
    if (!(cond)) atomicOr(&(S)->check, (unsigned)(bit));          \
  } while (0)
#else
#define POT3D_CHK(S, cond, bit) \
  do {                          \
  } while (0)
#endif
// p lies in [base, base + n)
__host__ __device__ inline bool in_range(const double *p, const double *base, long long n) {
  return p >= base && p < base + n;
}

// ---- peer-memory exchange between the rank processes (CUDA IPC over NVLink) ----
constexpr int MAXR = 16;
struct MailEntry {          // one rank's contribution to a reduction
  double v0, v1;
  unsigned long long seq;   // (epoch << 32) | iteration (1-based)
  unsigned long long pad;
};
enum MailKind { MAIL_A = 0, MAIL_B = 1, MAIL_C = 2, MAIL_D = 3 };  // CG1: (A, B) / (C, D) by iteration parity
// slots of the per-iteration kernel timeline (Scalars::trace, [64][16] %globaltimer)
enum TraceSlot { TR_EDGE0 = 0, TR_EDGE1, TR_A0, TR_AHALO, TR_A1, TR_F0, TR_F1, TR_B0, TR_B1, TR_EDGEM };
struct Mailbox {
  MailEntry e[4][MAXR];         // [kind][source rank]
  unsigned long long halo[2];   // ghost shell filled: [0] from rank-1, [1] from rank+1
  unsigned long long dhalo[2];  // PC3: the Chebyshev d's ghost shell filled (sequence grows)
  unsigned long long pad[4];
};
struct PeerTab {
  Mailbox *mail[MAXR];          // every rank's mailbox (own included)
  double *p_lo[2], *p_hi[2];    // P[0], P[1] of rank-1 / rank+1 (nullptr at the ends)
  double *d_lo[2], *d_hi[2];    // PC3: the Chebyshev d buffers of rank-1 / rank+1 (or nullptr)
  int rank, nranks, nr_lo, pad; // nr_lo: nr_loc of rank-1 (its top ghost shell index)
};
__host__ __device__ inline unsigned long long mail_seq(unsigned long long epoch, long long iter1) {
  return (epoch << 32) | (unsigned long long)iter1;
}

struct Grid {
  int nr, nt, np;     // global cells
  int i0, nr_loc;     // slab
  int PK;             // row pitch (doubles)
  long long plane;    // nt * PK
  int nchunks;        // r chunks per fused pass
  int ntj, ntk;       // tiles
  // per-launch split of the fused passes (halo overlap):
  //   part 0: all shells in nchunks chunks; part 1: shells [1, nr_loc-1) in
  //   nchunks chunks; part 2: the two edge shells (blockIdx.y = 0 / 1); part 3:
  //   as part 0 with the two chunks next to the ghost shells scheduled last.
  int part;
  int blk_off, blk_total;  // this launch's blocks within a reduction spanning launches
  int role_rows;           // pass A, peer memory: the first block row builds the edge shells
                           // of p_k and sends them to the neighbours (no edge-shell kernel)
  int cj, ck;              // fused passes: thread-block clusters of cj x ck neighbouring tiles
                           // (0/1: none; pot3d_ctx::pcj/pck, POT3D_CLUSTER)
};

// Tiles of a fused pass launch: blockIdx.x -> (tile row tj, tile column tk).  Without
// clusters tiles run theta-fastest; with cj x ck clusters, consecutive blocks form one
// cluster of neighbouring tiles (the grid is padded to whole clusters: blocks past the
// grid only join the reductions), so tiles sharing halo rows / columns run side by side.
__host__ __device__ inline int pass_tiles(const Grid &G) {
  const int cj = G.cj > 1 ? G.cj : 1, ck = G.ck > 1 ? G.ck : 1;
  return ((G.ntj + cj - 1) / cj) * ((G.ntk + ck - 1) / ck) * cj * ck;
}
__host__ __device__ inline void tile_of(const Grid &G, int b, int &tj, int &tk) {
  const int cj = G.cj > 1 ? G.cj : 1, ck = G.ck > 1 ? G.ck : 1;
  if (cj * ck == 1) {
    tj = b % G.ntj;
    tk = b / G.ntj;
    return;
  }
  const int cs = cj * ck, cid = b / cs, lid = b - cid * cs, nsj = (G.ntj + cj - 1) / cj;
  tj = (cid % nsj) * cj + lid % cj;
  tk = (cid / nsj) * ck + lid / cj;
}

// Physical column of logical phi index k is k + COFF: physical 0 is the
// periodic ghost copy of k = np-1 and physical np+1 the ghost copy of k = 0
// (P:54).  The ghost columns let a TMA box cover the wrap neighbours of every
// tile; every writer of a stencil operand keeps them.
constexpr int COFF = 1;
// Cell (il, j, k) of an array with ghost shells (il in [-1, nr_loc]).
__host__ __device__ inline long long cidx(const Grid &g, int il, int j, int k) {
  return (long long)(il + 1) * g.plane + (long long)j * g.PK + k + COFF;
}
// Start of shell il (whole theta-phi plane incl. pads and ghost columns).
__host__ __device__ inline long long sidx(const Grid &g, int il) { return (long long)(il + 1) * g.plane; }
// (j, k) of a single-plane buffer (bshell, br) with the same row layout.
__host__ __device__ inline long long pidx(const Grid &g, int j, int k) {
  return (long long)j * g.PK + k + COFF;
}

// TMA descriptors of the cell arrays (host-encoded, passed __grid_constant__).
struct TMaps {
  CUtensorMap src_h;    // pass A source: z (PC1: the D^-1 r buffer, PC2: the sweeps' z), haloed box
  CUtensorMap p_h[2];   // P[0], P[1], haloed box
  CUtensorMap r_i;      // pass B: z (PC1) / r (PC2), interior box {TKB, TJ, 1}
  CUtensorMap x_i;      // x, interior box {TKB, TJ, 1}
};


// Arguments of the fused passes (passes.cu).
struct PassArgs {
  Grid G;
  Metrics M;
  Scalars *S;
  const double *r;      // B: the stored residual vector (PC1: z = D^-1 r, PC2: r)
  double *r_out;        // B: its update (same buffer)
  const double *z;      // A: stored z = M^-1 r (PC1: the same buffer as r)
  const double *p_old;  // A
  double *p_new;        // A: write, B: read
  double *x;            // A
  double *partials;
  double *hist;
  int finalize;         // 1: single rank, finalise scalars in the last block
  double *local_sum;    // nranks > 1: this rank's sums for the all-gather
  const PeerTab *peers; // nranks > 1 with peer memory: mailbox / ghost-shell exchange
  int fold;             // peer memory, PC1: pass B posts its sums and leaves their
                        // finalisation (convergence, beta) to the next edge-shell kernel
  double *q_probe;      // k_pass_a_probe only: q = A p_k (cell layout)
  long long pstride;    // batch (gridDim.z > 1): partials / history of RHS z start
  long long hstride;    // z * pstride / z * hstride doubles after partials / hist
};

// CG1 (cg1.cu): TMA descriptors and arguments.  u ping-pongs between U[0], U[1] (K1
// reads U[parity] haloed, writes U[parity^1]); p, s, x are updated cell by cell.
struct Cg1Maps {
  CUtensorMap u_h[2];
  CUtensorMap p_i, s_i, x_i;
};
struct Cg1Args {
  Grid G;
  Metrics M;
  Scalars *S;
  double *u[2];
  double *p, *s, *x;
  double *partials, *hist, *local_sum;
  int finalize;  // single rank: the last block of K2 updates the scalars
  int init;      // K2 of the start: gamma_0, delta_0 -> alpha_0
  const PeerTab *peers;  // rank processes / loopback slabs with peer memory (cg1.cu): K1 stores
                         // u's edge shells into the neighbours' ghost shells and raises their
                         // halo flags, K2 waits for its own and posts its sums to every mailbox
};

// PC3 (poly.cu): TMA descriptors and arguments.  d ping-pongs between d[0], d[1].
struct PolyMaps {
  CUtensorMap d_h[2];
  CUtensorMap res_i, x_i, r_i;
};
struct PolyArgs {
  Grid G;
  Metrics M;
  Scalars *S;
  const double *r;       // the residual the apply starts from
  double *res, *d[2], *x, *z;
  double theta;          // (b + a) / 2
  double c1[POLY_MMAX], c2[POLY_MMAX];  // step k: d_k = c1[k] d_{k-1} + c2[k] res_k
  double *partials, *local_sum;
  int finalize;          // LAST: 1 updates rho/beta, 0 writes local_sum
  int predicated;        // skip when the PCG loop has stopped
  long long pstride;     // a batch (grid z / k_poly_init grid y = the problem): partials stride
  const PeerTab *peers;  // across ranks with peer memory: LAST posts r.z to every mailbox (MAIL_C)
  const PeerTab *hpeers; // ... and the d halo: init / step k store d's edge shells into the
                         // neighbours' ghost shells and raise dhalo; step k waits for d_{k-1}'s
};

// Arguments of the field kernels (a11).
struct FieldArgs {
  Grid G;
  const double *x;
  const double *br;      // device-layout boundary map [j][k]
  const double *mean2;   // closed-wall mean sums or nullptr
  const double *rc, *dr, *drh, *tc, *tf, *dth, *st, *dph;
  const double *poleN, *poleS;  // per local shell
  int bc;
  int nbr;               // r faces on this rank
  double *Br, *Bt, *Bp;  // device layout: [face][j][k], [i][jf][k], [i][j][k] (pitch PK)
};

// cg1.cu
__global__ void k_cg1_update_even(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity);
__global__ void k_cg1_update_odd(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity);
__global__ void k_cg1_dots(const __grid_constant__ Cg1Maps T, Cg1Args A, int parity);
__global__ void k_finalize_cg1(Scalars *S, const double *gathered, int nranks, double *hist, int init);

// poly.cu
__global__ void k_poly_init(PolyArgs A);
__global__ void k_poly_step(const __grid_constant__ PolyMaps T, PolyArgs A, int step);
__global__ void k_poly_last(const __grid_constant__ PolyMaps T, PolyArgs A, int step);

// kernels.cu
__global__ void k_metrics(int nr, int nt, int np, int bc, const double *rf, const double *tf,
                          const double *pf, double *arp, double *arm, double *dr, double *ss,
                          double *g, double *atp, double *atm, double *q, double *dp, double *app,
                          double *apm, double *rc, double *drh, double *tc, double *dth,
                          double *st, double *dph, double *vr);
// parity: P[parity] is p_{k-1}, P[parity^1] receives p_k
__global__ void k_pass_a(const __grid_constant__ TMaps T, PassArgs A, int parity);        // a3
__global__ void k_pass_a_probe(const __grid_constant__ TMaps T, PassArgs A, int parity);  // a3 + q out
// PC1 pass B (a7 + a8): even iterations leave x alone, odd ones apply the pair update (A23)
__global__ void k_pass_b_pc1_even(const __grid_constant__ TMaps T, PassArgs A, int parity);
__global__ void k_pass_b_pc1_odd(const __grid_constant__ TMaps T, PassArgs A, int parity);
__global__ void k_x_finish(Grid G, const Scalars *S, double *x, const double *p);
__global__ void k_pass_b_pc2(const __grid_constant__ TMaps T, PassArgs A, int parity);  // a7
// ghost columns (physical 0 and np+1) of shells [il0, il0 + n) from the interior
__global__ void k_fix_ghost_cols(Grid G, double *a, int il0, int n);
__global__ void k_finalize_alpha(Scalars *S, const double *gathered, int nranks);
__global__ void k_finalize_beta(Scalars *S, const double *gathered, int nranks, double *hist);
__global__ void k_finalize_rr(Scalars *S, const double *gathered, int nranks, double *hist);
__global__ void k_finalize_rho(Scalars *S, const double *gathered, int nranks);
__global__ void k_init_dots(Grid G, Metrics M, Scalars *S, const double *r, double *partials,
                            int finalize, double *local_sum, int use_z, const double *z, int keep_b,
                            double *hist0);
__global__ void k_init_finalize(Scalars *S, const double *gathered, int nranks, int keep_b, double *hist0);
__global__ void k_apply(Grid G, Metrics M, const double *x, double *y, const double *bshell,
                        int b_il, Scalars *S, double *partials, double *local_sum);
__global__ void k_br_mean(Grid G, Metrics M, const double *br, double *out2);
__global__ void k_rhs(Grid G, Metrics M, double r0, const double *br, const double *mean2,
                      double *bshell);
__global__ void k_gauge_sums(Grid G, Metrics M, const double *vr, const double *x, Scalars *S,
                             double *partials, double *local_sum);
__global__ void k_gauge_shift(Grid G, double *x, const double *gathered, int nranks);
__global__ void k_transpose(int ni, int nt, int np, long long stride_i, int PK, int coff,
                            const double *src, double *dst, int to_dev, int ld);
__global__ void k_field_r(FieldArgs F);
__global__ void k_field_t(FieldArgs F);
__global__ void k_field_p(FieldArgs F);
__global__ void k_pole_avg(Grid G, const double *x, const double *dp, double period, double *poleN,
                           double *poleS);
// mode -1: z = D^-1 src on every plane (PC1 apply); 0: p_new = D^-1 src + beta p_old on the
// two edge shells (PC1); 1: p_new = src + beta p_old on the edge shells (PC2, src = z)
__global__ void k_edge_p(Grid G, Metrics M, Scalars *S, const double *src, const double *p_old,
                         double *p_new, int mode, const PeerTab *peers, int parity_new,
                         double *hist, int fold);
// peer-memory finalisation: poll every rank's mailbox entry of `kind` for this
// iteration, sum in rank order, update the scalars (what = 0 alpha, 1 beta, 2 rr, 3 rho)
__global__ void k_finalize_mail(Scalars *S, const PeerTab *peers, int kind, int what, double *hist);
// CG1 over peer memory: gamma, delta (MAIL_A) and ||r||^2 (MAIL_B) of every rank in rank order
__global__ void k_finalize_cg1_mail(Scalars *S, const PeerTab *peers, double *hist);

// pc2.cu -- PC2 (block ILU0 = D-ILU, A11) with tiled sync-free wavefront sweeps
struct Pc2;
// nrhs > 1: the sweeps of a batch leader cover nrhs problems per launch (edge slots per
// problem; pot3d_runtime.nrhs, abi.cu setup_batch)
int pc2_create(Pc2 **out, const Grid &G, int nblocks_local, const int *block_l0,
               void *(*alloc)(size_t, void *), void *actx, cudaStream_t s, int nrhs = 1);
int pc2_factor(Pc2 *P, const Metrics &M, cudaStream_t s, double *min_pivot_host);
// z = M^-1 r; partial r.z -> finalize (single rank: rho/beta update, mode iteration) or
// local_sum[0]; `iteration` selects the predicated in-loop variant.
// A batch (nrhs > 1, the Pc2 created for it): problem q's r, z start q * vstride doubles
// on, its scalars are S[q], its partials q * pstride doubles on.
int pc2_apply(Pc2 *P, const Metrics &M, Scalars *S, const double *r, double *z, double *partials,
              int finalize, double *local_sum, cudaStream_t s, bool iteration,
              const PeerTab *peers = nullptr, int nrhs = 1, long long vstride = 0, long long pstride = 0);
void pc2_destroy(Pc2 *P, void (*fr)(void *, void *), void *actx);
int pc2_status(Pc2 *P, cudaStream_t s);
size_t pc2_bytes(const Pc2 *P);
int pc2_kernels_per_apply(const Pc2 *P);
const char *pc2_last_error();

}  // namespace pot3d
