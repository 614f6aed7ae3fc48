/*
 * pot3d.h -- C ABI of libpot3d.so, the B200 (sm_100a) fp64 PCG solve of the
 * POT3D potential-field problem of arXiv 1709.01126.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; A<n> = the reading
 * A<n> listed in DESIGN.md ("Readings of the paper").
 *
 * The problem: Phi on a nonuniform logically-rectangular spherical
 * (r, theta, phi) grid with
 *   lap Phi = 0                                   (Eq.1)
 *   dPhi/dr = Br0 at r = r0                        (Eq.2)
 *   Phi = 0 (source surface) or dPhi/dr = 0 (closed wall) at r = r1
 *   periodic in phi; polar values = phi-average of the adjacent ring  (Eq.3)
 * discretised by the second-order flux-difference stencil (with the
 * full spherical metric, A1) on cell-centred unknowns (A2), volume-scaled to a
 * symmetric positive (semi)definite matrix A (A3/A4), and solved by
 * preconditioned conjugate gradients with PC1 = inverse diagonal or
 * PC2 = zero-fill ILU of each r-slab block, to ||r||/||b|| <= rtol
 * (A9).  B = grad Phi is derived on staggered faces (A16).
 *
 * Layouts (all float64, C order):
 *   faces         1-D, nr+1 / nt+1 / np+1 entries, strictly increasing;
 *                 r_faces[0] = r0 > 0, t_faces[0] = 0, t_faces[nt] = pi,
 *                 p_faces[np] - p_faces[0] = 2 pi.
 *   br0           nt*np values, theta fastest: br0[j + nt*k]   (Fortran br0(j,k))
 *   phi, x, y, r  this rank's r-slab, r fastest: a[il + nr_loc*(j + nt*k)]
 *                 (Fortran x(i,j,k)), il = i - i0 (see pot3d_info).
 *   br            (nr_loc + last) x nt x np, r fastest: faces i0 .. i1-1, plus
 *                 face nr on the last rank (face i lies between cells i-1, i;
 *                 face 0 is the photosphere r0).
 *   bt            nr_loc x (nt+1) x np, r fastest (theta faces 0..nt; 0 and nt
 *                 are the poles).
 *   bp            nr_loc x nt x np, r fastest, at phi faces k+1/2 (periodic).
 *
 * Pointers: every array argument may be a host pointer (pageable or pinned)
 * or a device pointer of the context's device; the library detects which
 * with cudaPointerGetAttributes and copies accordingly.  Inputs are copied
 * before the call returns; the caller keeps ownership of every buffer.
 *
 * Multi-GPU: one process per GPU.  The grid is split into contiguous r-slabs
 * (leading ranks take the remainder shells).  pot3d_setup maps the
 * neighbours' p buffers and every rank's 1-KB mailbox through CUDA IPC (handles
 * exchanged over NCCL): the kernels store the halo of one theta-phi shell per
 * face straight into the neighbours' ghost shells over NVLink and post each
 * rank's dot-product partials into every mailbox; all ranks sum them in rank
 * order, so every rank holds bit-identical scalars.  If any rank cannot
 * map the peers, the same steps run over NCCL (send/recv, all-gather).  Peer
 * waits are bounded (20 s; the solve then fails with POT3D_ERR_CUDA).  Every call
 * is collective: all ranks call it with identical scalar arguments.
 *
 * Errors: functions return a pot3d_status; on a negative status
 * pot3d_last_error(ctx) describes the failure.  No function aborts.
 */
#ifndef POT3D_H
#define POT3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pot3d_ctx pot3d_ctx; /* opaque; owns all device state */

typedef enum {
  POT3D_OK = 0,
  POT3D_NOT_CONVERGED = 1,       /* maxit reached; outputs valid */
  POT3D_PC2_FELL_BACK = 2,       /* ILU pivot <= 1e-300: PC1 used instead and the solve
                                    converged; a fallen-back solve that
                                    hit maxit returns POT3D_NOT_CONVERGED (pot3d_info().pc
                                    still shows the fallback) */
  POT3D_ERR_INVALID = -1,        /* bad grid / sizes / arguments */
  POT3D_ERR_CUDA = -2,
  POT3D_ERR_NCCL = -3,
  POT3D_ERR_INDEFINITE = -4,     /* p.Ap <= 0 */
  POT3D_ERR_OOM = -5,
  POT3D_ERR_STATE = -6           /* call out of order (e.g. field before solve) */
} pot3d_status;

typedef enum { POT3D_SOURCE_SURFACE = 0, POT3D_CLOSED_WALL = 1 } pot3d_outer_bc;
typedef enum { POT3D_PC1 = 1, POT3D_PC2 = 2,
               POT3D_PC3 = 3 /* Chebyshev-accelerated Jacobi */ } pot3d_pc;

typedef struct {
  int32_t nr, nt, np;            /* cell counts (ghosts excluded, A12); each >= 2 */
  const double *r_faces;         /* host, nr+1 */
  const double *t_faces;         /* host, nt+1 */
  const double *p_faces;         /* host, np+1 */
} pot3d_grid;

typedef struct {
  int32_t rank, nranks;          /* this process and the world size (1 = single GPU) */
  const void *nccl_unique_id;    /* host, 128 bytes (ncclUniqueId) from rank 0; NULL if nranks == 1 */
  void *cuda_stream;             /* cudaStream_t all work is ordered on; NULL = the library's own */
  void *(*alloc)(size_t bytes, void *alloc_ctx); /* device allocator; NULL = cudaMalloc */
  void (*free)(void *ptr, void *alloc_ctx);
  void *alloc_ctx;
  int32_t pc2_blocks;            /* PC2 ILU0 blocks per rank (r sub-slabs); 0 -> 1 (A11) */
  int32_t device;                /* CUDA ordinal; -1 = current device */
  int32_t unroll;                /* PCG iterations per captured CUDA graph; 0 -> 32 */
  int32_t loopback_slabs;        /* > 1 (with nranks == 1): split the grid into this many
                                    r-slabs on ONE device and run the multi-GPU peer-memory
                                    exchange between them (halo stores into the siblings'
                                    ghost shells, mailbox reductions in rank order)
                                    ordered on one stream -- the multi-GPU path testable on
                                    one GPU.  Arrays are then the whole grid. 0/1: off */
  int32_t variant;               /* PCG recurrences: 0 standard (two reductions per
                                    iteration), 1 single-reduction CG1
                                    (Chronopoulos-Gear) */
  int32_t poly_degree;           /* PC3: Chebyshev steps m per apply (2..8); 0 -> 4 */
  double poly_ratio;             /* PC3: the polynomial targets [2/ratio, 2] of D^-1 A's
                                    spectrum (Saad Alg. 12.1); 0 -> 100 */
  int32_t nrhs;                  /* > 1: a multi-RHS batch (MAS repeats
                                    equivalent PCG solves): nrhs independent problems
                                    on the same grid and BC (one boundary map each), solved
                                    in ONE loop whose fused passes cover all of them per
                                    launch (grid z = the problem), each with its own scalars
                                    and convergence test; the loop ends when every problem
                                    has stopped (PC2: the k problems' ILU sweeps share one
                                    launch per sweep, their wavefronts interleaved; PC3: the
                                    Chebyshev steps too).  One rank, no loopback slabs,
                                    standard PCG (else POT3D_ERR_INVALID).  br0, phi, br, bt, bp then
                                    hold nrhs consecutive items of the single-problem layout
                                    (item q at offset q * its size); iters, rel_residual,
                                    true_rel_residual hold nrhs values; pot3d_history returns
                                    problem 0's; the diagnostic applies are refused.
                                    0/1: one problem */
} pot3d_runtime;

typedef struct {
  int32_t i0, i1;                /* this rank's shells [i0, i1) of 0..nr */
  int32_t nr_loc;                /* i1 - i0 */
  int32_t br_shells;             /* r faces returned by pot3d_field on this rank */
  int32_t pc;                    /* preconditioner in use (after any PC2 fallback) */
  int32_t pc2_blocks_total;      /* ILU blocks over all ranks */
  int64_t graph_kernels_per_iter;/* kernels launched per PCG iteration (for gpu_launches) */
  int64_t bytes_per_iter;        /* algorithmic HBM bytes per iteration on this rank */
  int64_t device_bytes;          /* device memory held by the context */
  int64_t kernel_launches;       /* cumulative count of this library's kernels launched
                                    (graph launches counted per kernel node) */
  int32_t exchange;              /* inter-rank exchange of the PCG loop: 0 single rank,
                                    1 NCCL (send/recv halo + all-gather of the sums),
                                    2 peer memory (CUDA IPC over NVLink: the kernels store
                                    halo shells and sums straight into the peers' buffers),
                                    3 the same exchange between the slabs of a loopback
                                    group on one device */
  int32_t chunks_a, chunks_b;    /* r-chunks per tile column of the two fused passes */
  int32_t nrhs;                  /* problems per solve (pot3d_runtime.nrhs; 1 unless a batch);
                                    bytes_per_iter then counts all of them */
} pot3d_info_t;

/* Build the context: metric coefficients (a1), r-slab partition, RHS from
 * br0 (a2; br0 is read on every rank, only the rank owning shell 0 uses it),
 * buffers, the PC2 factorisation if requested, the CUDA graphs.  *out is set
 * to NULL on error. */
int pot3d_setup(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                const pot3d_runtime *rt, pot3d_ctx **out);

/* Replace the boundary map (a2 re-run); the next pot3d_solve uses it. */
int pot3d_set_br0(pot3d_ctx *ctx, const double *br0);

/* PCG solve from x0 = 0 (A9).  phi (nullable): this rank's slab, layout above
 * (a batch: nrhs consecutive slabs, and iters / rel_residual / true_rel_residual
 * arrays of nrhs; the status is the first error, else NOT_CONVERGED if any problem
 * hit maxit).
 * iters: completed alpha-updates; rel_residual: recurrence ||r||/||b||;
 * true_rel_residual (nullable): ||b - A x|| / ||b|| recomputed after the
 * solve.  maxit >= 1.  Returns POT3D_OK, POT3D_NOT_CONVERGED,
 * POT3D_PC2_FELL_BACK or an error.  b = 0 returns Phi = 0, iters = 0.
 * Closed wall: Phi is returned in the zero volume-weighted-mean gauge. */
int pot3d_solve(pot3d_ctx *ctx, double rtol, int64_t maxit, double *phi, int64_t *iters,
                double *rel_residual, double *true_rel_residual);

/* Warm start -- repeated solves (MAS repeats equivalent PCG solves,
 * P:33): the same PCG from a given x0 instead of 0 (r_0 = b - A x0; the stopping test
 * stays ||r_k|| <= rtol ||b||, A9; iters counts this solve's iterations, 0 if x0
 * already meets it; hist[0] = ||r_0|| / ||b||).  x0: the layout of phi (a batch: nrhs
 * items), host or device, copied in; NULL = start from the context's last solution
 * (kept across pot3d_set_br0 and pot3d_field -- the time-series use: a new map, the
 * previous Phi; POT3D_ERR_STATE if a diagnostic call has run since).  Across ranks
 * (collective) x0 is this rank's slab and the start takes two reductions (||b||,
 * then r_0's sums) and the halo of x0; a loopback group takes the whole grid.  b = 0
 * still returns Phi = 0.  Outputs and status as pot3d_solve. */
int pot3d_solve_from(pot3d_ctx *ctx, const double *x0, double rtol, int64_t maxit, double *phi,
                     int64_t *iters, double *rel_residual, double *true_rel_residual);

/* B = grad Phi of the last solution on staggered faces (a11, A16); nullable
 * outputs are skipped.  POT3D_ERR_STATE before a successful solve. */
int pot3d_field(pot3d_ctx *ctx, double *br, double *bt, double *bp);

/* Diagnostics used by the parity tests.  They run the production kernels of
 * the solve loop with scalars that turn them into plain applies (this rank's
 * slab, layout as phi; x, y host or device; every rank calls them together):
 *   pot3d_apply_fused(which = 0): y = A x (homogeneous operator, A6)
 *       through pass B (PC2 instantiation: r_out = 0 - (-1) q = q exactly);
 *   which = 1 (PC1 contexts): y = D^-1 A x through PC1's pass B
 *       (z_out = 0 - (-1) D^-1 q, the Jacobi division of the loop);
 *   which = 2: y = A x from pass A's stencil (a diagnostic instantiation of
 *       the same code that also stores q).
 * pot3d_apply = pot3d_apply_fused(which = 0).  pot3d_precond: z = M^-1 r
 * (PC1: the init kernel that forms z_0 = D^-1 b; PC2: the D-ILU sweeps).
 * Each invalidates the last solution.  POT3D_ERR_INVALID for a bad `which`. */
int pot3d_apply(pot3d_ctx *ctx, const double *x, double *y);
int pot3d_apply_fused(pot3d_ctx *ctx, const double *x, double *y, int32_t which);
int pot3d_precond(pot3d_ctx *ctx, const double *r, double *z);

/* Residual history of the last solve: hist[k] = ||r_k||/||b||, k = 0..n-1,
 * n = min(len, iters+1, 2^24) (the device buffer keeps the first 2^24 entries;
 * maxit itself is not capped). Returns n or an error. */
int64_t pot3d_history(pot3d_ctx *ctx, double *hist, int64_t len);

int pot3d_info(const pot3d_ctx *ctx, pot3d_info_t *info);

/* Diagnostics for the roofline report: continue the PCG recurrences of the
 * current state for `iters` iterations (rtol = 0) launching each pass
 * separately between CUDA events on the context's stream; returns the mean
 * device time per launch of pass A, pass B (and the PC2 sweeps, 0 for PC1)
 * in milliseconds.  Invalidates the last solution (call pot3d_solve again). */
int pot3d_profile(pot3d_ctx *ctx, int32_t iters, double *ms_pass_a, double *ms_pass_b,
                  double *ms_precond);

/* Diagnostics: one PCG iteration at a time (no graph) with CUDA events on the
 * context stream after every sub-step (kernels and collectives); returns the
 * number n of sub-steps, ms[q] their mean duration and `names` (>= 1024 bytes)
 * their ';'-separated names.  Invalidates the last solution. */
int pot3d_profile_iteration(pot3d_ctx *ctx, int32_t iters, double *ms, char *names, int32_t nmax);

/* In-situ kernel timing of the solve loop itself (no extra launches): with
 * tracing enabled before pot3d_solve, every fused pass records %globaltimer when
 * its first block starts (after its dependency wait) and when its last block
 * finishes, in a ring of the last 64 iterations.  pot3d_kernel_times returns the
 * mean pass A and pass B durations (microseconds) over the ring and the number
 * of iterations averaged (n).  POT3D_ERR_STATE if tracing was not enabled. */
int pot3d_trace_enable(pot3d_ctx *ctx, int32_t on);
int pot3d_kernel_times(pot3d_ctx *ctx, double *us_pass_a, double *us_pass_b, int32_t *n);
/* The same ring per iteration: for up to `len` of the last <= 64 iterations of
 * the last solve, the iteration index (0-based; PC1's pass B differs between
 * even and odd iterations, A23) and the pass A / pass B durations in
 * microseconds.  Returns the number of entries written or an error. */
int pot3d_kernel_trace(pot3d_ctx *ctx, int64_t *iter, double *us_pass_a, double *us_pass_b, int32_t len);

/* Rank 0 creates the 128-byte NCCL unique id that every rank passes in
 * pot3d_runtime.nccl_unique_id (the caller broadcasts it, e.g. with
 * torch.distributed).  Returns 0 or POT3D_ERR_NCCL. */
int pot3d_nccl_unique_id(void *out128);
int pot3d_destroy(pot3d_ctx *ctx);
const char *pot3d_last_error(const pot3d_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* POT3D_H */
