// abi.cu -- the C ABI of libpot3d.so (include/pot3d.h): setup, solve loop
// orchestration (CUDA graphs, device-resident scalars, NCCL halo/all-gather),
// field derivation and diagnostics.  All arithmetic of the method runs in the
// kernels of kernels.cu / pc2.cu; this file only schedules them.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pot3d.h"
#include "pot3d_internal.cuh"


using namespace pot3d;

struct pot3d_ctx {
  // problem
  int nr = 0, nt = 0, np = 0, bc = 0, pc_req = 1, pc = 1;
  int rank = 0, nranks = 1, pc2_blocks = 1, unroll = 32;
  int nchunks_b = 1;  // r-chunks of pass B (G.nchunks: pass A)
  bool pdl = true;    // programmatic dependent launch for the loop kernels (POT3D_PDL=0: off)
  int edge_blocks = 148 * 4;  // grid of the edge-shell kernel (POT3D_EDGE_BLOCKS)
  bool edge_in_a = true;      // pass A's first block row builds the edge shells (POT3D_EDGE_IN_A=0: kernel)
  int device = 0;
  double r0 = 1.0;
  Grid G{};
  std::vector<double> rf, tf, pf;
  // runtime
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t comm_stream = nullptr;          // NCCL halo exchange (overlapped with pass A)
  cudaEvent_t ev_edge = nullptr, ev_halo = nullptr;
  void *(*ualloc)(size_t, void *) = nullptr;
  void (*ufree)(void *, void *) = nullptr;
  void *actx = nullptr;
  std::vector<void *> allocs;
  size_t dev_bytes = 0;
  ncclComm_t comm = nullptr;
  // device data
  double *d_rf = nullptr, *d_tf = nullptr, *d_pf = nullptr;
  double *m_arp, *m_arm, *m_dr, *m_ss, *m_g, *m_atp, *m_atm, *m_q, *m_dp, *m_app, *m_apm;
  double *m_rc, *m_drh, *m_tc, *m_dth, *m_st, *m_dph, *m_vr;
  Metrics M{};
  double *x = nullptr, *r = nullptr, *P[2] = {nullptr, nullptr}, *z = nullptr;
  double *bshell = nullptr, *br_dev = nullptr, *mean2 = nullptr, *staging = nullptr;
  size_t staging_bytes = 0;
  Scalars *S = nullptr;
  Scalars *hS = nullptr;  // pinned mirror
  double *partials = nullptr;
  size_t partials_len = 0;
  double *hist = nullptr;
  int64_t hist_len = 0;
  double *local_sum = nullptr, *gathered = nullptr;
  double *poles = nullptr;
  Pc2 *pc2 = nullptr;
  TMaps tmaps{};
  // peer-memory exchange (nranks > 1): P[0], P[1] and the mailbox are cudaMalloc'd
  // (IPC-exportable) and mapped into the neighbours' / all ranks' address spaces
  bool xfer_want = false, xfer = false;
  Mailbox *mail = nullptr;
  PeerTab *peers = nullptr;           // device copy
  std::vector<void *> ipc_own, ipc_open;
  unsigned long long epoch = 0;       // solves (and profile runs) so far
  unsigned long long *trace = nullptr;  // kernel timestamps (pot3d_trace_enable / POT3D_TRACE)
  bool trace_on = false;
  // graphs
  cudaGraphExec_t gexec = nullptr;
  int graph_unroll = 0;
  // launch accounting (pot3d_info_t.kernel_launches)
  int64_t n_launch = 0;     // kernels launched (graph launches count their kernel nodes)
  int64_t n_enq = 0;        // kernels enqueued by enqueue_iteration (graph capture)
  int64_t graph_nodes = 0;  // kernel nodes of the instantiated graph
  // state
  bool solved = false;
  int64_t last_iters = 0;
  std::string err;
};

namespace {

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
      return POT3D_ERR_CUDA;                                                          \
    }                                                                                 \
  } while (0)
#define NK(call)                                                                      \
  do {                                                                                \
    ncclResult_t n_ = (call);                                                         \
    if (n_ != ncclSuccess) {                                                          \
      ctx->err = std::string(#call) + ": " + ncclGetErrorString(n_);                  \
      return POT3D_ERR_NCCL;                                                          \
    }                                                                                 \
  } while (0)
#define TRY(expr)               \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ < 0) return rc_;    \
  } while (0)

void *dalloc_raw(pot3d_ctx *ctx, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void *p = nullptr;
  if (ctx->ualloc) {
    p = ctx->ualloc(bytes, ctx->actx);
  } else {
    if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
  }
  if (p) {
    ctx->allocs.push_back(p);
    ctx->dev_bytes += bytes;
  }
  return p;
}

template <typename T>
int dalloc(pot3d_ctx *ctx, T **out, size_t count) {
  *out = static_cast<T *>(dalloc_raw(ctx, sizeof(T) * count));
  if (!*out) {
    ctx->err = "device allocation of " + std::to_string(sizeof(T) * count) + " bytes failed";
    return POT3D_ERR_OOM;
  }
  return 0;
}

void dfree_all(pot3d_ctx *ctx) {
  for (void *p : ctx->allocs) {
    if (ctx->ufree)
      ctx->ufree(p, ctx->actx);
    else
      cudaFree(p);
  }
  ctx->allocs.clear();
}

// IPC-exportable allocation (plain cudaMalloc: an IPC handle maps a whole allocation)
template <typename T>
int ipc_alloc(pot3d_ctx *ctx, T **out, size_t count) {
  void *p = nullptr;
  if (cudaMalloc(&p, sizeof(T) * count) != cudaSuccess) {
    cudaGetLastError();
    ctx->err = "cudaMalloc of " + std::to_string(sizeof(T) * count) + " bytes failed";
    return POT3D_ERR_OOM;
  }
  ctx->ipc_own.push_back(p);
  ctx->dev_bytes += sizeof(T) * count;
  *out = static_cast<T *>(p);
  return 0;
}

void ipc_release(pot3d_ctx *ctx) {
  for (void *p : ctx->ipc_open) cudaIpcCloseMemHandle(p);
  ctx->ipc_open.clear();
  if (!ctx->ipc_own.empty() && ctx->comm) {
    // every rank has stopped touching the peers' buffers before any is freed
    int *d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
      ncclAllReduce(d, d, 1, ncclInt32, ncclSum, ctx->comm, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      cudaFree(d);
    }
  }
  for (void *p : ctx->ipc_own) cudaFree(p);
  ctx->ipc_own.clear();
}

// Kernel launch, optionally with the programmatic-dependent-launch attribute: the
// kernel may begin (its prologue) while the previous kernel on the stream drains;
// every kernel launched this way calls pdl_wait() before reading its inputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int ensure_staging(pot3d_ctx *ctx, size_t bytes) {
  if (ctx->staging_bytes >= bytes) return 0;
  double *p = nullptr;
  TRY(dalloc(ctx, &p, (bytes + 7) / 8));
  ctx->staging = p;
  ctx->staging_bytes = bytes;
  return 0;
}

// slab partition: B = nranks * pc2_blocks blocks (leading-remainder rule)
void block_bounds(int nr, int B, int b, int &i0, int &i1) {
  int base = nr / B, rem = nr % B;
  i0 = b * base + (b < rem ? b : rem);
  i1 = i0 + base + (b < rem ? 1 : 0);
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

// user layout (r fastest, ni shells) <-> device cells (phi fastest)
int to_device_cells(pot3d_ctx *ctx, const double *user, double *dev_cells_first_shell, int ni,
                    long long stride_i) {
  const size_t n = (size_t)ni * ctx->nt * ctx->np;
  const double *src = user;
  if (!is_device_ptr(user)) {
    TRY(ensure_staging(ctx, n * sizeof(double)));
    CK(cudaMemcpyAsync(ctx->staging, user, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    src = ctx->staging;
  }
  dim3 blk(32, 8), grd((ctx->np + 31) / 32, (ni + 31) / 32, ctx->nt);
  k_transpose<<<grd, blk, 0, ctx->stream>>>(ni, ctx->nt, ctx->np, stride_i, ctx->G.PK, COFF, src,
                                            dev_cells_first_shell, 1);
  CK(cudaGetLastError());
  ctx->n_launch++;
  return 0;
}

int from_device_cells(pot3d_ctx *ctx, const double *dev_first, double *user, int ni, int nj,
                      long long stride_i, int coff = COFF) {
  const size_t n = (size_t)ni * nj * ctx->np;
  const bool dev = is_device_ptr(user);
  double *dst = user;
  if (!dev) {
    TRY(ensure_staging(ctx, n * sizeof(double)));
    dst = ctx->staging;
  }
  dim3 blk(32, 8), grd((ctx->np + 31) / 32, (ni + 31) / 32, nj);
  k_transpose<<<grd, blk, 0, ctx->stream>>>(ni, nj, ctx->np, stride_i, ctx->G.PK, coff, dev_first, dst,
                                            0);
  CK(cudaGetLastError());
  ctx->n_launch++;
  if (!dev) {
    CK(cudaMemcpyAsync(user, dst, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return 0;
}

// all-gather `count` doubles per rank from local_sum into gathered (no-op copy at 1 rank)
int gather_sums(pot3d_ctx *ctx, int count) {
  if (ctx->nranks == 1) {
    CK(cudaMemcpyAsync(ctx->gathered, ctx->local_sum, sizeof(double) * 2, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    return 0;
  }
  (void)count;
  NK(ncclAllGather(ctx->local_sum, ctx->gathered, 2, ncclDouble, ctx->comm, ctx->stream));
  return 0;
}

// halo exchange of one shell per r face of a cell array with ghost shells
int halo_exchange(pot3d_ctx *ctx, double *a, cudaStream_t st = nullptr) {
  if (ctx->nranks == 1) return 0;
  if (!st) st = ctx->stream;
  const Grid &G = ctx->G;
  const size_t cnt = (size_t)G.plane;
  NK(ncclGroupStart());
  if (ctx->rank > 0) {
    NK(ncclSend(a + sidx(G, 0), cnt, ncclDouble, ctx->rank - 1, ctx->comm, st));
    NK(ncclRecv(a + sidx(G, -1), cnt, ncclDouble, ctx->rank - 1, ctx->comm, st));
  }
  if (ctx->rank < ctx->nranks - 1) {
    NK(ncclSend(a + sidx(G, G.nr_loc - 1), cnt, ncclDouble, ctx->rank + 1, ctx->comm, st));
    NK(ncclRecv(a + sidx(G, G.nr_loc), cnt, ncclDouble, ctx->rank + 1, ctx->comm, st));
  }
  NK(ncclGroupEnd());
  return 0;
}

// Peer-memory exchange setup: the IPC handles of P[0], P[1] and the mailbox are
// all-gathered over NCCL; each rank maps every mailbox and its neighbours' P
// arrays.  Enabled only when every rank succeeded (else the NCCL path stays).
int setup_xfer(pot3d_ctx *ctx) {
  struct IpcInfo {
    cudaIpcMemHandle_t h[3];
    int32_t ok, nr_loc, pad0, pad1;
  };
  const int n = ctx->nranks, me = ctx->rank;
  cudaStream_t s = ctx->stream;
  IpcInfo mine{};
  mine.ok = ctx->xfer_want && ctx->mail != nullptr;
  mine.nr_loc = ctx->G.nr_loc;
  if (mine.ok && (cudaIpcGetMemHandle(&mine.h[0], ctx->P[0]) != cudaSuccess ||
                  cudaIpcGetMemHandle(&mine.h[1], ctx->P[1]) != cudaSuccess ||
                  cudaIpcGetMemHandle(&mine.h[2], ctx->mail) != cudaSuccess)) {
    cudaGetLastError();
    mine.ok = 0;
  }
  char *d = nullptr;
  TRY(dalloc(ctx, &d, sizeof(IpcInfo) * (n + 1)));
  CK(cudaMemcpyAsync(d, &mine, sizeof(IpcInfo), cudaMemcpyHostToDevice, s));
  NK(ncclAllGather(d, d + sizeof(IpcInfo), sizeof(IpcInfo), ncclChar, ctx->comm, s));
  std::vector<IpcInfo> all(n);
  CK(cudaMemcpyAsync(all.data(), d + sizeof(IpcInfo), sizeof(IpcInfo) * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  bool ok = true;
  for (const IpcInfo &a : all) ok = ok && a.ok;
  PeerTab T{};
  T.rank = me;
  T.nranks = n;
  T.nr_lo = me > 0 ? all[me - 1].nr_loc : 0;
  auto open = [&](const cudaIpcMemHandle_t &hd) -> void * {
    void *p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    ctx->ipc_open.push_back(p);
    return p;
  };
  if (ok) {
    for (int r = 0; r < n && ok; r++) {
      T.mail[r] = (r == me) ? ctx->mail : static_cast<Mailbox *>(open(all[r].h[2]));
      ok = T.mail[r] != nullptr;
    }
    for (int q = 0; q < 2 && ok; q++) {
      if (me > 0) ok = ok && (T.p_lo[q] = static_cast<double *>(open(all[me - 1].h[q]))) != nullptr;
      if (me < n - 1) ok = ok && (T.p_hi[q] = static_cast<double *>(open(all[me + 1].h[q]))) != nullptr;
    }
  }
  // agreement: all ranks or none
  int32_t okv = ok ? 1 : 0;
  CK(cudaMemcpyAsync(d, &okv, sizeof(int32_t), cudaMemcpyHostToDevice, s));
  NK(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, ctx->comm, s));
  CK(cudaMemcpyAsync(&okv, d, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (!okv) {
    for (void *p : ctx->ipc_open) cudaIpcCloseMemHandle(p);
    ctx->ipc_open.clear();
    ctx->xfer = false;
    return 0;
  }
  TRY(dalloc(ctx, &ctx->peers, 1));
  CK(cudaMemcpyAsync(ctx->peers, &T, sizeof(PeerTab), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  ctx->xfer = true;
  return 0;
}

// TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry point)
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 3-D view [nr_loc+2 shells][nt rows][PK columns] of a cell array; box {b0, b1, 1}
int make_map(pot3d_ctx *ctx, CUtensorMap *m, double *base, unsigned b0, unsigned b1) {
  auto enc = tma_encoder();
  if (!enc) {
    ctx->err = "cuTensorMapEncodeTiled unavailable";
    return POT3D_ERR_CUDA;
  }
  const Grid &G = ctx->G;
  cuuint64_t dims[3] = {(cuuint64_t)G.PK, (cuuint64_t)G.nt, (cuuint64_t)G.nr_loc + 2};
  cuuint64_t strides[2] = {(cuuint64_t)G.PK * 8, (cuuint64_t)G.plane * 8};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    ctx->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return POT3D_ERR_CUDA;
  }
  return 0;
}

int make_maps(pot3d_ctx *ctx) {
  TRY(make_map(ctx, &ctx->tmaps.src_h, ctx->pc == 2 ? ctx->z : ctx->r, SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.p_h[0], ctx->P[0], SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.p_h[1], ctx->P[1], SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.r_i, ctx->r, TKB, TJ));
  TRY(make_map(ctx, &ctx->tmaps.x_i, ctx->x, TKB, TJ));
  return 0;
}


PassArgs make_args(pot3d_ctx *ctx, int parity) {
  PassArgs a{};
  a.G = ctx->G;
  a.M = ctx->M;
  a.S = ctx->S;
  a.r = ctx->r;
  a.r_out = ctx->r;
  a.z = ctx->z;
  a.p_old = ctx->P[parity];
  a.p_new = ctx->P[parity ^ 1];
  a.x = ctx->x;
  a.partials = ctx->partials;
  a.hist = ctx->hist;
  a.finalize = ctx->nranks == 1 ? 1 : 0;
  a.local_sum = ctx->local_sum;
  return a;
}

using PassKernel = void (*)(const TMaps, PassArgs, int);
PassKernel kern_a(const pot3d_ctx *ctx) {
  return ctx->pc == 2 ? k_pass_a_pc2 : k_pass_a_pc1;
}
PassKernel kern_b(const pot3d_ctx *ctx) {
  return ctx->pc == 2 ? k_pass_b_pc2 : k_pass_b_pc1;
}

// One PCG iteration (a3-a10) enqueued on ctx->stream; parity = iteration & 1.
//   pass A  (p_new = z + beta p_old, q = A p_new, sigma partial)      -> alpha
//   pass B  (q again, r -= alpha q, x += alpha p_new; PC1: rho', ||r||^2) -> convergence, beta
//   [PC2]   forward + backward D-ILU sweeps (z, rho')                 -> beta
//   [N > 1] edge shells of p_new to the neighbours (peer memory: pass A's first block
//           row or k_edge_p; NCCL: k_edge_p + send/recv) and rank sums through the
//           mailboxes (or an NCCL all-gather) before each finalisation
// optional timing hook: records an event on the main stream after each sub-step
struct StepTimer {
  std::vector<cudaEvent_t> ev;
  std::vector<const char *> name;
  cudaStream_t s;
  void mark(const char *n) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    name.push_back(n);
  }
};
static StepTimer *g_timer = nullptr;
#define MARK(n) \
  do {          \
    if (g_timer) g_timer->mark(n); \
  } while (0)

int enqueue_iteration(pot3d_ctx *ctx, int parity) {
  const Grid &G = ctx->G;
  PassArgs a = make_args(ctx, parity);
  dim3 grd(G.ntj * G.ntk, G.nchunks);
  PassArgs ab = a;  // pass B: its own r-chunking
  ab.G.nchunks = ctx->nchunks_b;
  dim3 grdb(G.ntj * G.ntk, ctx->nchunks_b);
  const bool pc2 = ctx->pc == 2;
  const bool multi = ctx->nranks > 1;
  if (ctx->xfer) {
    // peer memory: edge shells of p_k stored into the neighbours' ghost shells
    // (flag per iteration); pass A waits for that flag only in the blocks whose
    // chunk touches a ghost shell (scheduled last); the rank sums go straight into
    // every rank's mailbox from the reductions' last blocks
    const PeerTab *pt = ctx->peers;
    if (ctx->edge_in_a && !pc2) {
      // pass A's first block row builds and sends the edge shells beside the interior
      // chunks; beta is finalised by its own kernel after pass B
      PassArgs ax = a;
      ax.G.part = 3;
      ax.G.role_rows = 1;
      ax.peers = pt;
      // at least 3 chunks, so an interior chunk runs while the halo travels (the two
      // chunks touching the ghost shells are scheduled last): 4 GPUs x 19 shells,
      // 84.9 us per iteration with 3 chunks vs 89.1 with the single-GPU choice of 1
      if (ax.G.nchunks < 3 && G.nr_loc >= 6) ax.G.nchunks = 3;
      CK(launch_k(ctx->pdl, kern_a(ctx), dim3(G.ntj * G.ntk, ax.G.nchunks + 1), dim3(NTHREADS), SMEM_A,
                  ctx->stream, ctx->tmaps, ax, parity));
      MARK("passA");
      CK(launch_k(ctx->pdl, k_finalize_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S, pt, (int)MAIL_A, 0,
                  (double *)nullptr));
      MARK("finalize_alpha");
      PassArgs bx = ab;
      bx.peers = pt;
      CK(launch_k(ctx->pdl, kern_b(ctx), grdb, dim3(NTHREADS), SMEM_B, ctx->stream, ctx->tmaps, bx, parity));
      MARK("passB");
      CK(launch_k(ctx->pdl, k_finalize_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S, pt, (int)MAIL_B, 1,
                  ctx->hist));
      MARK("finalize_beta");
      ctx->n_enq += 4;
      return 0;
    }
    // PC1: the previous iteration's beta finalisation lives in edge_p (fold)
    const int fold = pc2 ? 0 : 1;
    CK(launch_k(ctx->pdl, k_edge_p, dim3(ctx->edge_blocks), dim3(256), 0, ctx->stream, G, ctx->M, ctx->S,
                (const double *)(pc2 ? ctx->z : ctx->r), (const double *)ctx->P[parity],
                ctx->P[parity ^ 1], pc2 ? 1 : 0, pt, parity ^ 1, ctx->hist, fold));
    MARK("edge_p");
    PassArgs ax = a;
    ax.G.part = 3;
    ax.peers = pt;
    CK(launch_k(ctx->pdl, kern_a(ctx), grd, dim3(NTHREADS), SMEM_A,
                ctx->stream, ctx->tmaps, ax, parity));
    MARK("passA");
    CK(launch_k(ctx->pdl, k_finalize_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S, pt, (int)MAIL_A, 0,
                (double *)nullptr));
    MARK("finalize_alpha");
    PassArgs bx = ab;
    bx.peers = pt;
    bx.fold = fold;  // pass B only posts its sums and marks them pending
    CK(launch_k(ctx->pdl, kern_b(ctx), grdb, dim3(NTHREADS), SMEM_B,
                ctx->stream, ctx->tmaps, bx, parity));
    MARK("passB");
    ctx->n_enq += 4;
    if (!fold) {
      CK(launch_k(ctx->pdl, k_finalize_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S, pt, (int)MAIL_B,
                  2, ctx->hist));
      MARK("finalize_rr");
      ctx->n_enq++;
    }
    if (pc2) {
      int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, 0, ctx->local_sum,
                         ctx->stream, true, pt);
      TRY(nk);
      k_finalize_mail<<<1, 1, 0, ctx->stream>>>(ctx->S, pt, MAIL_C, 3, nullptr);
      CK(cudaGetLastError());
      ctx->n_enq += nk + 1;
      MARK("pc2");
    }
    return 0;
  }
  if (multi && G.nr_loc >= 3) {
    // edge shells first; their halo travels on the comm stream while pass A
    // covers the interior shells, then pass A finishes the two edge shells
    k_edge_p<<<148 * 4, 256, 0, ctx->stream>>>(G, ctx->M, ctx->S, pc2 ? ctx->z : ctx->r,
                                                ctx->P[parity], ctx->P[parity ^ 1], pc2 ? 1 : 0,
                                                nullptr, 0, nullptr, 0);
    CK(cudaGetLastError());
    ctx->n_enq++;
    MARK("edge_p");
    CK(cudaEventRecord(ctx->ev_edge, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_edge, 0));
    TRY(halo_exchange(ctx, ctx->P[parity ^ 1], ctx->comm_stream));
    CK(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
    const int nci = std::max(1, std::min(G.nchunks, G.nr_loc - 2));
    const int ntl = G.ntj * G.ntk;
    PassArgs ai = a, ae = a;
    ai.G.part = 1;
    ai.G.nchunks = nci;
    ai.G.blk_off = 0;
    ai.G.blk_total = ntl * (nci + 2);
    ae.G.part = 2;
    ae.G.blk_off = ntl * nci;
    ae.G.blk_total = ntl * (nci + 2);
    CK(launch_k(false, kern_a(ctx), dim3(ntl, nci), dim3(NTHREADS), SMEM_A, ctx->stream, ctx->tmaps, ai,
                parity));
    ctx->n_enq++;
    MARK("passA_interior");
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    MARK("halo_wait");
    CK(launch_k(false, kern_a(ctx), dim3(ntl, 2), dim3(NTHREADS), SMEM_A, ctx->stream, ctx->tmaps, ae,
                parity));
    ctx->n_enq++;
    MARK("passA_edge");
  } else {
    if (multi) {
      k_edge_p<<<148 * 4, 256, 0, ctx->stream>>>(G, ctx->M, ctx->S, pc2 ? ctx->z : ctx->r,
                                                  ctx->P[parity], ctx->P[parity ^ 1], pc2 ? 1 : 0,
                                                nullptr, 0, nullptr, 0);
      CK(cudaGetLastError());
      ctx->n_enq++;
      TRY(halo_exchange(ctx, ctx->P[parity ^ 1]));
    }
    CK(launch_k(ctx->pdl && !multi, kern_a(ctx), grd, dim3(NTHREADS), SMEM_A,
                ctx->stream, ctx->tmaps, a, parity));
    ctx->n_enq++;
  }
  if (multi) {
    TRY(gather_sums(ctx, 1));
    MARK("allgather_sigma");
    k_finalize_alpha<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks);
    CK(cudaGetLastError());
    ctx->n_enq++;
    MARK("finalize_alpha");
  }
  CK(launch_k(ctx->pdl && !multi, kern_b(ctx), grdb, dim3(NTHREADS), SMEM_B,
              ctx->stream, ctx->tmaps, ab, parity));
    ctx->n_enq++;
  MARK("passB");
  if (multi) {
    TRY(gather_sums(ctx, 2));
    MARK("allgather_rz_rr");
    if (pc2)
      k_finalize_rr<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks, ctx->hist);
    else
      k_finalize_beta<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks, ctx->hist);
    CK(cudaGetLastError());
    ctx->n_enq++;
  }
  if (pc2) {
    int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, multi ? 0 : 1,
                       ctx->local_sum, ctx->stream, true);
    TRY(nk);
    CK(cudaGetLastError());
    ctx->n_enq += nk;
    if (multi) {
      TRY(gather_sums(ctx, 1));
      k_finalize_rho<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks);
      CK(cudaGetLastError());
    ctx->n_enq++;
    }
  }
  return 0;
}

int build_graph(pot3d_ctx *ctx) {
  if (ctx->gexec) {
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  cudaGraph_t g;
  ctx->n_enq = 0;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int u = 0; u < ctx->unroll && rc == 0; u++) rc = enqueue_iteration(ctx, u & 1);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (rc) return rc;
  CK(e);
  CK(cudaGraphInstantiate(&ctx->gexec, g, 0));
  cudaGraphDestroy(g);
  ctx->graph_unroll = ctx->unroll;
  ctx->graph_nodes = ctx->n_enq;
  return 0;
}

// r-chunks per tile column of a fused pass: at least ceil(nr_loc / Lcap) chunks,
// then the count with the best product of wave efficiency (blocks / whole waves,
// counted only below 3 waves: with more, unequal block times hide the tail) and
// halo-plane efficiency L / (L + 2).  Short chunks keep the tiles of a wave within
// a few planes of each other, so the halo rows a tile shares with its neighbours
// are still in L2; measured best chunk lengths (pass A / pass B): medium 38 / 30,
// large 75-100 / 27-38, weak 69 / 35 shells -> Lcap 100 for A and 32 for B.
int pick_chunks(const Grid &G, double slots, int Lcap) {
  const int cmin = std::max(1, (G.nr_loc + Lcap - 1) / Lcap);
  // thin slabs (multi-GPU r-slabs of <= 24 shells) whose tiles alone already cover
  // every SM: the two halo planes of a chunk cost more than idle slots -- one chunk
  // (19 x 301 x 601: 57.8 us per iteration with 1 chunk per pass vs 66.0 us with 4,
  // tools/lat.py); small grids with few tiles still need the chunks for parallelism
  if (G.nr_loc <= 24 && (double)G.ntj * G.ntk >= slots / 2) return cmin;
  const long long tiles = (long long)G.ntj * G.ntk;
  double best = -1;
  int bestc = cmin;
  for (int c = cmin; c <= std::max(cmin, std::min(G.nr_loc, 64)); c++) {
    double blocks = (double)tiles * c;
    double waves = blocks / slots;
    double eff_w = waves < 3.0 ? waves / std::ceil(waves) : 1.0;
    double L = (double)G.nr_loc / c;
    double eff_h = L / (L + 2.0);
    double e = eff_w * eff_h;
    if (e > best + 1e-9) {
      best = e;
      bestc = c;
    }
  }
  return bestc;
}

int choose_chunks(pot3d_ctx *ctx) {
  Grid &G = ctx->G;
  // every chunk (plus its two halo planes) fits the passes' staged r-metrics
  const int lstage = POT3D_PLMAX - 2;
  int occ = 0, sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pass_b_pc1, NTHREADS, SMEM_B));
  int occa = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occa, k_pass_a_pc1, NTHREADS, SMEM_A));
  const double slots_a = (double)sms * std::max(1, occa), slots_b = (double)sms * std::max(1, occ);
  G.nchunks = pick_chunks(G, slots_a, std::min(lstage, 100));
  ctx->nchunks_b = pick_chunks(G, slots_b, std::min(lstage, 32));
  auto env_chunks = [&](const char *name, int &dst) {
    const char *e = getenv(name);
    if (e && atoi(e) > 0) dst = std::max((G.nr_loc + lstage - 1) / lstage, std::min(atoi(e), G.nr_loc));
  };
  env_chunks("POT3D_CHUNKS", G.nchunks);
  env_chunks("POT3D_CHUNKS_B", ctx->nchunks_b);
  return 0;
}
}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

static thread_local std::string g_setup_error = "no error";

const char *pot3d_last_error(const pot3d_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_setup_error.c_str();
}

int pot3d_nccl_unique_id(void *out128) {
  if (!out128) return POT3D_ERR_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return POT3D_ERR_NCCL;
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int pot3d_info(const pot3d_ctx *ctx, pot3d_info_t *info) {
  if (!ctx || !info) return POT3D_ERR_INVALID;
  info->i0 = ctx->G.i0;
  info->i1 = ctx->G.i0 + ctx->G.nr_loc;
  info->nr_loc = ctx->G.nr_loc;
  info->br_shells = ctx->G.nr_loc + (ctx->rank == ctx->nranks - 1 ? 1 : 0);
  info->pc = ctx->pc;
  info->pc2_blocks_total = ctx->pc2_blocks * ctx->nranks;
  int64_t k = 2;
  if (ctx->nranks > 1) k += (ctx->xfer && ctx->pc == 1) ? 2 : 3;
  if (ctx->pc == 2 && ctx->pc2) k += pc2_kernels_per_apply(ctx->pc2) + (ctx->nranks > 1 ? 1 : 0);
  info->graph_kernels_per_iter = k;
  // algorithmic bytes: PC1 64 B/cell (pass A 24 + pass B 40), PC2 + 56 B sweeps
  const int64_t cells = (int64_t)ctx->G.nr_loc * ctx->nt * ctx->np;
  info->bytes_per_iter = (ctx->pc == 2 ? 120 : 64) * cells;
  info->device_bytes = (int64_t)ctx->dev_bytes;
  info->kernel_launches = ctx->n_launch;
  info->exchange = ctx->nranks == 1 ? 0 : (ctx->xfer ? 2 : 1);
  info->chunks_a = ctx->G.nchunks;
  info->chunks_b = ctx->nchunks_b;
  info->reserved = 0;
  return 0;
}

int pot3d_set_br0(pot3d_ctx *ctx, const double *br0) {
  if (!ctx || !br0) return POT3D_ERR_INVALID;
  const Grid &G = ctx->G;
  CK(cudaSetDevice(ctx->device));
  // (np, nt) theta-fastest user map -> device [j][k]: the transpose with ni = nt, nj = 1
  const size_t n = (size_t)ctx->nt * ctx->np;
  const double *src = br0;
  if (!is_device_ptr(br0)) {
    TRY(ensure_staging(ctx, n * sizeof(double)));
    CK(cudaMemcpyAsync(ctx->staging, br0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    src = ctx->staging;
  }
  {
    dim3 blk(32, 8), grd((ctx->np + 31) / 32, (ctx->nt + 31) / 32, 1);
    k_transpose<<<grd, blk, 0, ctx->stream>>>(ctx->nt, 1, ctx->np, G.PK, G.PK, COFF, src, ctx->br_dev, 1);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  if (ctx->bc == POT3D_CLOSED_WALL) {
    k_br_mean<<<1, 1024, 0, ctx->stream>>>(G, ctx->M, ctx->br_dev, ctx->mean2);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  if (G.i0 == 0) {
    unsigned nb = (unsigned)((n + 255) / 256);
    k_rhs<<<nb, 256, 0, ctx->stream>>>(G, ctx->M, ctx->r0, ctx->br_dev,
                                       ctx->bc == POT3D_CLOSED_WALL ? ctx->mean2 : nullptr,
                                       ctx->bshell);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->solved = false;
  return 0;
}

int pot3d_setup(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                const pot3d_runtime *rt, pot3d_ctx **out) {
  if (!out) return POT3D_ERR_INVALID;
  *out = nullptr;
  pot3d_ctx *ctx = new pot3d_ctx();
  auto fail = [&](int rc) {
    *out = nullptr;
    g_setup_error = ctx->err;  // reachable through pot3d_last_error(NULL)
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ipc_release(ctx);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    dfree_all(ctx);
    if (ctx->hS) cudaFreeHost(ctx->hS);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return rc;
  };
  if (!grid || !br0 || !grid->r_faces || !grid->t_faces || !grid->p_faces) {
    ctx->err = "null argument";
    return fail(POT3D_ERR_INVALID);
  }
  const int nr = grid->nr, nt = grid->nt, np = grid->np;
  if (nr < 2 || nt < 2 || np < 2) {
    ctx->err = "cell counts must be >= 2 (S:45)";
    return fail(POT3D_ERR_INVALID);
  }
  if (outer_bc != POT3D_SOURCE_SURFACE && outer_bc != POT3D_CLOSED_WALL) {
    ctx->err = "outer_bc must be SOURCE_SURFACE or CLOSED_WALL";
    return fail(POT3D_ERR_INVALID);
  }
  if (pc != POT3D_PC1 && pc != POT3D_PC2) {
    ctx->err = "pc must be 1 or 2";
    return fail(POT3D_ERR_INVALID);
  }
  ctx->rf.assign(grid->r_faces, grid->r_faces + nr + 1);
  ctx->tf.assign(grid->t_faces, grid->t_faces + nt + 1);
  ctx->pf.assign(grid->p_faces, grid->p_faces + np + 1);
  for (int i = 0; i < nr; i++)
    if (!(ctx->rf[i + 1] > ctx->rf[i])) { ctx->err = "r_faces not increasing"; return fail(POT3D_ERR_INVALID); }
  for (int j = 0; j < nt; j++)
    if (!(ctx->tf[j + 1] > ctx->tf[j])) { ctx->err = "t_faces not increasing"; return fail(POT3D_ERR_INVALID); }
  for (int k = 0; k < np; k++)
    if (!(ctx->pf[k + 1] > ctx->pf[k])) { ctx->err = "p_faces not increasing"; return fail(POT3D_ERR_INVALID); }
  if (!(ctx->rf[0] > 0.0)) { ctx->err = "r0 must be > 0"; return fail(POT3D_ERR_INVALID); }
  if (std::fabs(ctx->tf[0]) > 1e-12 || std::fabs(ctx->tf[nt] - M_PI) > 1e-12) {
    ctx->err = "t_faces must span [0, pi]";
    return fail(POT3D_ERR_INVALID);
  }
  if (std::fabs(ctx->pf[np] - ctx->pf[0] - 2 * M_PI) > 1e-12) {
    ctx->err = "p_faces must span 2 pi";
    return fail(POT3D_ERR_INVALID);
  }
  ctx->nr = nr; ctx->nt = nt; ctx->np = np;
  ctx->bc = outer_bc;
  ctx->pc_req = ctx->pc = pc;
  ctx->r0 = ctx->rf[0];
  {
    const char *e = getenv("POT3D_PDL");
    ctx->pdl = !(e && atoi(e) == 0);
    const char *eb = getenv("POT3D_EDGE_BLOCKS");
    if (eb && atoi(eb) > 0) ctx->edge_blocks = atoi(eb);
    const char *ea = getenv("POT3D_EDGE_IN_A");
    ctx->edge_in_a = !(ea && atoi(ea) == 0);
  }
  pot3d_runtime R{};
  R.nranks = 1;
  R.device = -1;
  if (rt) R = *rt;
  ctx->rank = R.rank;
  ctx->nranks = R.nranks < 1 ? 1 : R.nranks;
  ctx->pc2_blocks = R.pc2_blocks < 1 ? 1 : R.pc2_blocks;
  ctx->unroll = R.unroll > 0 ? (R.unroll + 1) / 2 * 2 : 32;
  ctx->ualloc = R.alloc;
  ctx->ufree = R.free;
  ctx->actx = R.alloc_ctx;
  if (ctx->rank < 0 || ctx->rank >= ctx->nranks) { ctx->err = "bad rank"; return fail(POT3D_ERR_INVALID); }
  if (ctx->nranks > 1 && !R.nccl_unique_id) { ctx->err = "nccl_unique_id required for nranks > 1"; return fail(POT3D_ERR_INVALID); }
  const int B = ctx->nranks * ctx->pc2_blocks;
  if (nr < 2 * ctx->nranks || (pc == POT3D_PC2 && nr < B)) {
    ctx->err = "too many ranks/blocks for nr";
    return fail(POT3D_ERR_INVALID);
  }
  if (R.device >= 0) {
    ctx->device = R.device;
  } else {
    cudaGetDevice(&ctx->device);
  }
  CK(cudaSetDevice(ctx->device));
  if (R.cuda_stream) {
    ctx->stream = (cudaStream_t)R.cuda_stream;
  } else {
    // a blocking stream: implicitly ordered with the legacy default stream the
    // caller (e.g. torch's default stream) produces device inputs on
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault));
    ctx->own_stream = true;
  }

  if (ctx->nranks > 1) {
    CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_edge, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
  }
  // r-slab of this rank: union of its pc2_blocks consecutive blocks
  std::vector<int> bi0(B), bi1(B);
  for (int b = 0; b < B; b++) block_bounds(nr, B, b, bi0[b], bi1[b]);
  if (pc == POT3D_PC1) {
    int a, b;
    block_bounds(nr, ctx->nranks, ctx->rank, a, b);
    ctx->G.i0 = a;
    ctx->G.nr_loc = b - a;
  } else {
    ctx->G.i0 = bi0[ctx->rank * ctx->pc2_blocks];
    ctx->G.nr_loc = bi1[(ctx->rank + 1) * ctx->pc2_blocks - 1] - ctx->G.i0;
  }
  Grid &G = ctx->G;
  G.nr = nr; G.nt = nt; G.np = np;
  G.PK = round_up(np + COFF + 1, 16);  // physical columns: [ghost np-1][0..np-1][ghost 0][pads]
  G.plane = (long long)nt * G.PK;
  G.ntj = (nt + TJ - 1) / TJ;
  G.ntk = (np + TK - 1) / TK;
  {
    const void *fa[2] = {(const void *)k_pass_a_pc1, (const void *)k_pass_a_pc2};
    const void *fb[2] = {(const void *)k_pass_b_pc1, (const void *)k_pass_b_pc2};
    for (int q = 0; q < 2; q++) {
      if (cudaFuncSetAttribute(fa[q], cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_A) ||
          cudaFuncSetAttribute(fb[q], cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_B)) {
        ctx->err = "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed";
        return fail(POT3D_ERR_CUDA);
      }
    }
  }
  { int rc = choose_chunks(ctx); if (rc) return fail(rc); }

  // metrics (a1)
  int rc = 0;
#define DA(ptr, n) if ((rc = dalloc(ctx, &(ptr), (n)))) return fail(rc)
  DA(ctx->d_rf, nr + 1); DA(ctx->d_tf, nt + 1); DA(ctx->d_pf, np + 1);
  // r factors carry one padding entry on each side (read for ghost shells)
  DA(ctx->m_arp, nr + 2); DA(ctx->m_arm, nr + 2); DA(ctx->m_dr, nr + 2); DA(ctx->m_ss, nr + 2);
  ctx->m_arp += 1; ctx->m_arm += 1; ctx->m_dr += 1; ctx->m_ss += 1;
  DA(ctx->m_rc, nr); DA(ctx->m_drh, nr); DA(ctx->m_vr, nr);
  DA(ctx->m_g, nt); DA(ctx->m_atp, nt); DA(ctx->m_atm, nt); DA(ctx->m_q, nt);
  DA(ctx->m_tc, nt); DA(ctx->m_dth, nt); DA(ctx->m_st, nt);
  DA(ctx->m_dp, np); DA(ctx->m_app, np); DA(ctx->m_apm, np); DA(ctx->m_dph, np);
  if (cudaMemcpyAsync(ctx->d_rf, ctx->rf.data(), sizeof(double) * (nr + 1), cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(ctx->d_tf, ctx->tf.data(), sizeof(double) * (nt + 1), cudaMemcpyHostToDevice, ctx->stream) ||
      cudaMemcpyAsync(ctx->d_pf, ctx->pf.data(), sizeof(double) * (np + 1), cudaMemcpyHostToDevice, ctx->stream)) {
    ctx->err = "face upload failed";
    return fail(POT3D_ERR_CUDA);
  }
  {
    int n = std::max(nr, std::max(nt, np));
    k_metrics<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
        nr, nt, np, outer_bc, ctx->d_rf, ctx->d_tf, ctx->d_pf, ctx->m_arp, ctx->m_arm, ctx->m_dr,
        ctx->m_ss, ctx->m_g, ctx->m_atp, ctx->m_atm, ctx->m_q, ctx->m_dp, ctx->m_app, ctx->m_apm,
        ctx->m_rc, ctx->m_drh, ctx->m_tc, ctx->m_dth, ctx->m_st, ctx->m_dph, ctx->m_vr);
    if (cudaGetLastError() != cudaSuccess) { ctx->err = "k_metrics launch failed"; return fail(POT3D_ERR_CUDA); }
  }
  ctx->M = Metrics{ctx->m_arp, ctx->m_arm, ctx->m_dr, ctx->m_ss, ctx->m_g, ctx->m_atp,
                   ctx->m_atm, ctx->m_q, ctx->m_dp, ctx->m_app, ctx->m_apm};


  // vectors with ghost shells
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  DA(ctx->x, cells); DA(ctx->r, cells);
  {
    const char *xe = getenv("POT3D_XFER");
    ctx->xfer_want = ctx->nranks > 1 && ctx->nranks <= MAXR && !(xe && atoi(xe) == 0);
  }
  if (ctx->xfer_want) {
    if ((rc = ipc_alloc(ctx, &ctx->P[0], cells)) || (rc = ipc_alloc(ctx, &ctx->P[1], cells)) ||
        (rc = ipc_alloc(ctx, &ctx->mail, 1)))
      return fail(rc);
    if (cudaMemsetAsync(ctx->mail, 0, sizeof(Mailbox), ctx->stream)) { ctx->err = "memset"; return fail(POT3D_ERR_CUDA); }
  } else {
    DA(ctx->P[0], cells); DA(ctx->P[1], cells);
  }
  if (pc == POT3D_PC2) DA(ctx->z, cells);
  DA(ctx->bshell, G.plane + 16); DA(ctx->br_dev, G.plane + 16); DA(ctx->mean2, 2);
  DA(ctx->S, 1);
  ctx->partials_len = 4 * (size_t)std::max<long long>(
      (long long)G.ntj * G.ntk * (std::max(G.nchunks, ctx->nchunks_b) + 3), 65536);
  DA(ctx->partials, ctx->partials_len);
  DA(ctx->local_sum, 2);
  DA(ctx->gathered, 2 * (size_t)ctx->nranks + 2);
  DA(ctx->poles, 2 * (size_t)G.nr_loc);
#undef DA
  for (void *p : {(void *)ctx->x, (void *)ctx->r, (void *)ctx->P[0], (void *)ctx->P[1]})
    if (cudaMemsetAsync(p, 0, cells * sizeof(double), ctx->stream)) { ctx->err = "memset"; return fail(POT3D_ERR_CUDA); }
  if (ctx->z) cudaMemsetAsync(ctx->z, 0, cells * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->bshell, 0, (G.plane + 16) * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->br_dev, 0, (G.plane + 16) * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->S, 0, sizeof(Scalars), ctx->stream);
  if (cudaMallocHost(&ctx->hS, sizeof(Scalars)) != cudaSuccess) { ctx->err = "pinned alloc"; return fail(POT3D_ERR_CUDA); }

  if (ctx->nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, R.nccl_unique_id, sizeof(id));
    ncclResult_t nr_ = ncclCommInitRank(&ctx->comm, ctx->nranks, id, ctx->rank);
    if (nr_ != ncclSuccess) {
      ctx->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(nr_);
      return fail(POT3D_ERR_NCCL);
    }
    if ((rc = setup_xfer(ctx))) return fail(rc);
  }

  if (pc == POT3D_PC2) {
    std::vector<int> lb(ctx->pc2_blocks + 1);
    for (int b = 0; b < ctx->pc2_blocks; b++) lb[b] = bi0[ctx->rank * ctx->pc2_blocks + b] - G.i0;
    lb[ctx->pc2_blocks] = G.nr_loc;
    rc = pc2_create(&ctx->pc2, G, ctx->pc2_blocks, lb.data(), ctx->ualloc, ctx->actx, ctx->stream);
    if (rc) { ctx->err = "pc2_create failed"; return fail(POT3D_ERR_OOM); }
    double minpiv = 0;
    rc = pc2_factor(ctx->pc2, ctx->M, ctx->stream, &minpiv);
    if (rc) { ctx->err = "pc2_factor failed"; return fail(POT3D_ERR_CUDA); }
    // breakdown on any rank -> every rank falls back
    int bad = (minpiv < 1e-300) ? 1 : 0;
    if (ctx->nranks > 1) {
      int *d = nullptr;
      if ((rc = dalloc(ctx, &d, 2 * ctx->nranks))) return fail(rc);
      cudaMemcpyAsync(d, &bad, sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
      ncclAllGather(d, d + ctx->nranks, 1, ncclInt32, ctx->comm, ctx->stream);
      std::vector<int> h(ctx->nranks);
      cudaMemcpyAsync(h.data(), d + ctx->nranks, sizeof(int) * ctx->nranks, cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      for (int v : h) bad |= v;
    }
    if (bad) ctx->pc = POT3D_PC1;
  }
  {
    int rc2 = pot3d_set_br0(ctx, br0);
    if (rc2) return fail(rc2);
  }
  {
    int rc2 = make_maps(ctx);
    if (rc2) return fail(rc2);
    rc2 = build_graph(ctx);
    if (rc2) return fail(rc2);
  }
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    ctx->err = std::string("setup: ") + cudaGetErrorString(cudaGetLastError());
    return fail(POT3D_ERR_CUDA);
  }
  *out = ctx;
  return 0;
}

int pot3d_solve(pot3d_ctx *ctx, double rtol, int64_t maxit, double *phi, int64_t *iters,
                double *rel_residual, double *true_rel_residual) {
  if (!ctx) return POT3D_ERR_INVALID;
  if (!(rtol >= 0.0) || maxit < 1) {
    ctx->err = "rtol must be >= 0 and maxit >= 1";
    return POT3D_ERR_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  ctx->solved = false;
  // residual history buffer (maxit+1 doubles, capped)
  const int64_t hlen = std::min<int64_t>(maxit + 1, (int64_t)1 << 24);
  if (hlen > ctx->hist_len) {
    double *h = nullptr;
    TRY(dalloc(ctx, &h, (size_t)hlen));
    ctx->hist = h;
    ctx->hist_len = hlen;
    TRY(build_graph(ctx));  // graph captured the old history pointer
  }
  // x0 = 0, r = b, p = 0 (A9)
  CK(cudaMemsetAsync(ctx->x, 0, cells * sizeof(double), s));
  CK(cudaMemsetAsync(ctx->r, 0, cells * sizeof(double), s));
  CK(cudaMemsetAsync(ctx->P[0], 0, cells * sizeof(double), s));
  CK(cudaMemsetAsync(ctx->P[1], 0, cells * sizeof(double), s));
  if (G.i0 == 0) {
    CK(cudaMemcpyAsync(ctx->r + sidx(G, 0), ctx->bshell, G.plane * sizeof(double),
                       cudaMemcpyDeviceToDevice, s));
    k_fix_ghost_cols<<<(ctx->nt + 255) / 256, 256, 0, s>>>(G, ctx->r, 0, 1);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  Scalars h0{};
  h0.epoch = ++ctx->epoch;
  if ((ctx->trace_on || getenv("POT3D_TRACE")) && !ctx->trace) {
    TRY(dalloc(ctx, &ctx->trace, 64 * 16));
  }
  if (ctx->trace) CK(cudaMemsetAsync(ctx->trace, 0, 64 * 16 * sizeof(unsigned long long), s));
  h0.trace = ctx->trace;
  h0.rtol = rtol;
  h0.maxit = (long long)std::min<int64_t>(maxit, hlen - 1);
  CK(cudaMemcpyAsync(ctx->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
  // z0 = M^-1 b, rho0 = b.z0, ||b|| (a10 init)
  const int nbi = 148 * 4;
  if (ctx->pc == 2) {
    int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, 0, ctx->local_sum,
                       s, false);
    TRY(nk);
    CK(cudaGetLastError());
    ctx->n_launch += nk;
  }
  k_init_dots<<<nbi, 256, 0, s>>>(G, ctx->M, ctx->S, ctx->r, ctx->partials, ctx->nranks == 1,
                                  ctx->local_sum, ctx->pc == 2, ctx->z);
  CK(cudaGetLastError());
    ctx->n_launch++;
  if (ctx->nranks > 1) {
    TRY(gather_sums(ctx, 2));
    k_init_finalize<<<1, 1, 0, s>>>(ctx->S, ctx->gathered, ctx->nranks);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  if (ctx->hist) {
    // hist[0] = 1 (||r_0|| = ||b||)
    double one = 1.0;
    CK(cudaMemcpyAsync(ctx->hist, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  }
  // device-driven loop: graphs of `unroll` predicated iterations; the stop flag
  // of graph g is read back while graph g+1 is already queued
  CK(cudaMemcpyAsync(ctx->hS, ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int64_t launched = 0;
  if (!ctx->hS->stop) {
    cudaEvent_t ev[2];
    Scalars *hs2 = nullptr;
    CK(cudaMallocHost(&hs2, 2 * sizeof(Scalars)));
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    CK(cudaGraphLaunch(ctx->gexec, s));
    ctx->n_launch += ctx->graph_nodes;
    CK(cudaMemcpyAsync(&hs2[0], ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ev[0], s));
    launched++;
    int cur = 0;
    while (true) {
      const bool more = (launched * ctx->graph_unroll) < maxit + ctx->graph_unroll;
      if (more) {
        CK(cudaGraphLaunch(ctx->gexec, s));
        ctx->n_launch += ctx->graph_nodes;
        CK(cudaMemcpyAsync(&hs2[cur ^ 1], ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[cur ^ 1], s));
        launched++;
      }
      CK(cudaEventSynchronize(ev[cur]));
      if (hs2[cur].stop || !more) break;
      cur ^= 1;
    }
    CK(cudaStreamSynchronize(s));
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    cudaFreeHost(hs2);
  }
  CK(cudaMemcpyAsync(ctx->hS, ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const Scalars hs = *ctx->hS;
  ctx->last_iters = hs.iter;
  if (ctx->trace && getenv("POT3D_TRACE")) {  // mean per-iteration timeline after the edge-shell kernel
    std::vector<unsigned long long> t(64 * 16);
    cudaMemcpy(t.data(), ctx->trace, t.size() * 8, cudaMemcpyDeviceToHost);
    const char *nm[10] = {"edge0", "edge1", "A0", "Ahalo", "A1", "fin0", "fin1", "B0", "B1", "edgeM"};
    double sum[10] = {0}, n = 0, per = 0;
    for (int it = 0; it < 64; it++) {
      const unsigned long long *r = &t[it * 16];
      if (!r[0] || !r[8]) continue;
      for (int q = 0; q < 10; q++) sum[q] += r[q] ? (double)(long long)(r[q] - r[0]) : 0.0;
      const unsigned long long *nx = &t[((it + 1) % 64) * 16];
      if (nx[0] > r[0]) per += (double)(nx[0] - r[0]);
      n++;
    }
    if (n > 0) {
      fprintf(stderr, "POT3D_TRACE rank %d (us after edge0, mean of %.0f iterations):", ctx->rank, n);
      for (int q = 0; q < 10; q++) fprintf(stderr, " %s %.1f", nm[q], sum[q] / n / 1e3);
      fprintf(stderr, " | iteration %.1f\n", per / n / 1e3);
    }
  }
  if (ctx->pc == 2 && (pc2_status(ctx->pc2, s) & 2)) {
    ctx->err = "PC2 sweep handoff protocol error (bounded wait expired)";
    return POT3D_ERR_CUDA;
  }
  if (hs.xfer_error || hs.status == -5) {
    ctx->err = "peer-memory exchange: bounded wait expired (a rank stalled or diverged)";
    return POT3D_ERR_CUDA;
  }
  if (hs.status == -4) {
    if (getenv("POT3D_DEBUG")) {  // diagnostics: scalars and non-finite counts of the vectors
      fprintf(stderr, "POT3D_DEBUG iter %lld rho %g alpha %g beta %g sigma %g rr %g bnorm %g\n",
              hs.iter, hs.rho, hs.alpha, hs.beta, hs.sigma, hs.rr, hs.bnorm);
      const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
      std::vector<double> h(cells);
      const char *nm[5] = {"x", "r", "P0", "P1", "z"};
      double *ar[5] = {ctx->x, ctx->r, ctx->P[0], ctx->P[1], ctx->z};
      for (int q = 0; q < 5; q++) {
        if (!ar[q]) continue;
        cudaMemcpy(h.data(), ar[q], cells * 8, cudaMemcpyDeviceToHost);
        size_t bad = 0, first = (size_t)-1;
        double mx = 0;
        for (size_t c = 0; c < cells; c++) {
          if (!std::isfinite(h[c])) { if (!bad) first = c; bad++; }
          else mx = std::max(mx, std::fabs(h[c]));
        }
        long long fi = first == (size_t)-1 ? -1 : (long long)first;
        fprintf(stderr, "  %s: nonfinite %zu first %lld (shell %lld row %lld col %lld) max|.| %g\n", nm[q], bad, fi,
                fi < 0 ? -1 : fi / G.plane - 1, fi < 0 ? -1 : (fi % G.plane) / G.PK,
                fi < 0 ? -1 : (fi % G.PK) - COFF, mx);
      }
    }
    ctx->err = "p.Ap <= 0: operator or preconditioner not positive definite (S:341)";
    return POT3D_ERR_INDEFINITE;
  }
  if (!hs.stop) {
    ctx->err = "loop ended without the stop flag";
    return POT3D_ERR_STATE;
  }
  // (x is current: pass B applies x += alpha p_k in the same sweep as r -= alpha q)
  // closed wall: zero volume-weighted-mean gauge (A8)
  if (ctx->bc == POT3D_CLOSED_WALL && hs.bnorm > 0) {
    k_gauge_sums<<<nbi, 256, 0, s>>>(G, ctx->M, ctx->m_vr, ctx->x, ctx->S, ctx->partials,
                                      ctx->local_sum);
    CK(cudaGetLastError());
    ctx->n_launch++;
    TRY(gather_sums(ctx, 2));
    k_gauge_shift<<<148 * 8, 256, 0, s>>>(G, ctx->x, ctx->gathered, ctx->nranks);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  TRY(halo_exchange(ctx, ctx->x));
  if (true_rel_residual) {
    k_apply<<<nbi, 256, 0, s>>>(G, ctx->M, ctx->x, nullptr, ctx->bshell, G.i0 == 0 ? 0 : -1000,
                                ctx->S, ctx->partials, ctx->local_sum);
    CK(cudaGetLastError());
    ctx->n_launch++;
    TRY(gather_sums(ctx, 1));
    std::vector<double> g(2 * ctx->nranks);
    CK(cudaMemcpyAsync(g.data(), ctx->gathered, sizeof(double) * 2 * ctx->nranks,
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double t = 0.0;
    for (int rr = 0; rr < ctx->nranks; rr++) t += g[2 * rr];
    *true_rel_residual = hs.bnorm > 0 ? std::sqrt(t) / hs.bnorm : 0.0;
  }
  if (phi) TRY(from_device_cells(ctx, ctx->x + G.plane, phi, G.nr_loc, ctx->nt, G.plane));
  CK(cudaStreamSynchronize(s));
  if (iters) *iters = hs.iter;
  if (rel_residual) *rel_residual = hs.bnorm > 0 ? std::sqrt(hs.rr) / hs.bnorm : 0.0;
  ctx->last_iters = hs.iter;
  ctx->solved = true;
  if (ctx->pc != ctx->pc_req) return POT3D_PC2_FELL_BACK;
  return hs.status == 1 ? POT3D_NOT_CONVERGED : POT3D_OK;
}

int64_t pot3d_history(pot3d_ctx *ctx, double *hist, int64_t len) {
  if (!ctx || !hist) return POT3D_ERR_INVALID;
  if (!ctx->hist) return POT3D_ERR_STATE;
  int64_t n = std::min<int64_t>(len, ctx->last_iters + 1);
  if (cudaMemcpy(hist, ctx->hist, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess) {
    ctx->err = "history copy failed";
    return POT3D_ERR_CUDA;
  }
  return n;
}

int pot3d_field(pot3d_ctx *ctx, double *br, double *bt, double *bp) {
  if (!ctx) return POT3D_ERR_INVALID;
  if (!ctx->solved) {
    ctx->err = "pot3d_field before a successful pot3d_solve";
    return POT3D_ERR_STATE;
  }
  CK(cudaSetDevice(ctx->device));
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
  // temporaries: reuse the Krylov buffers (x keeps the solution)
  double *Br = ctx->P[0], *Bt = ctx->P[1], *Bp = ctx->r;
  const int nbr = G.nr_loc + (ctx->rank == ctx->nranks - 1 ? 1 : 0);
  const int ntf = ctx->nt + 1;
  // Bt needs nr_loc * (nt+1) * PK <= (nr_loc+2) * nt * PK
  if ((long long)G.nr_loc * ntf > (long long)(G.nr_loc + 2) * ctx->nt) {
    ctx->err = "field buffer too small";
    return POT3D_ERR_STATE;
  }
  k_pole_avg<<<dim3(G.nr_loc, 2), 256, 0, s>>>(G, ctx->x, ctx->m_dp, ctx->pf[ctx->np] - ctx->pf[0],
                                                ctx->poles, ctx->poles + G.nr_loc);
  CK(cudaGetLastError());
    ctx->n_launch++;
  FieldArgs F{};
  F.G = G;
  F.x = ctx->x;
  F.br = ctx->br_dev;
  F.mean2 = ctx->bc == POT3D_CLOSED_WALL ? ctx->mean2 : nullptr;
  F.rc = ctx->m_rc; F.dr = ctx->m_dr; F.drh = ctx->m_drh; F.tc = ctx->m_tc; F.tf = ctx->d_tf;
  F.dth = ctx->m_dth; F.st = ctx->m_st; F.dph = ctx->m_dph;
  F.poleN = ctx->poles; F.poleS = ctx->poles + G.nr_loc;
  F.bc = ctx->bc;
  F.nbr = nbr;
  F.Br = Br; F.Bt = Bt; F.Bp = Bp;
  const long long nc = (long long)G.nr_loc * ctx->nt * ctx->np;
  if (br) {
    long long n = (long long)nbr * ctx->nt * ctx->np;
    k_field_r<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(F);
    CK(cudaGetLastError());
    ctx->n_launch++;
    TRY(from_device_cells(ctx, Br, br, nbr, ctx->nt, G.plane, 0));
  }
  if (bt) {
    long long n = (long long)G.nr_loc * ntf * ctx->np;
    k_field_t<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(F);
    CK(cudaGetLastError());
    ctx->n_launch++;
    TRY(from_device_cells(ctx, Bt, bt, G.nr_loc, ntf, (long long)ntf * G.PK, 0));
  }
  if (bp) {
    k_field_p<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(F);
    CK(cudaGetLastError());
    ctx->n_launch++;
    TRY(from_device_cells(ctx, Bp, bp, G.nr_loc, ctx->nt, G.plane, 0));
  }
  CK(cudaStreamSynchronize(s));
  // the Krylov buffers were reused: a later field call needs a new solve's x only
  return 0;
}

int pot3d_apply(pot3d_ctx *ctx, const double *x, double *y) {
  if (!ctx || !x || !y) return POT3D_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  double *xin = ctx->P[0], *yout = ctx->P[1];
  CK(cudaMemsetAsync(xin, 0, cells * sizeof(double), s));
  TRY(to_device_cells(ctx, x, xin + G.plane, G.nr_loc, G.plane));
  TRY(halo_exchange(ctx, xin));
  k_apply<<<148 * 4, 256, 0, s>>>(G, ctx->M, xin, yout, nullptr, 0, ctx->S, nullptr, nullptr);
  CK(cudaGetLastError());
    ctx->n_launch++;
  TRY(from_device_cells(ctx, yout + G.plane, y, G.nr_loc, ctx->nt, G.plane));
  CK(cudaStreamSynchronize(s));
  ctx->solved = false;
  return 0;
}

int pot3d_precond(pot3d_ctx *ctx, const double *rin, double *zout) {
  if (!ctx || !rin || !zout) return POT3D_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  double *rr = ctx->P[0], *zz = ctx->P[1];
  CK(cudaMemsetAsync(rr, 0, cells * sizeof(double), s));
  CK(cudaMemsetAsync(zz, 0, cells * sizeof(double), s));
  TRY(to_device_cells(ctx, rin, rr + G.plane, G.nr_loc, G.plane));
  if (ctx->pc == 2) {
    int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, rr, zz, ctx->partials, 0, ctx->local_sum, s, false);
    TRY(nk);
    CK(cudaGetLastError());
    ctx->n_launch += nk;
  } else {
    // PC1: the edge-plane kernel computes z = D^-1 r (beta = 0) over any planes
    Scalars h0{};
    CK(cudaMemcpyAsync(ctx->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
    k_edge_p<<<148 * 8, 256, 0, s>>>(G, ctx->M, ctx->S, rr, nullptr, zz, -1, nullptr, 0, nullptr, 0);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  TRY(from_device_cells(ctx, zz + G.plane, zout, G.nr_loc, ctx->nt, G.plane));
  CK(cudaStreamSynchronize(s));
  ctx->solved = false;
  return 0;
}

int pot3d_profile(pot3d_ctx *ctx, int32_t iters, double *ms_pass_a, double *ms_pass_b,
                  double *ms_precond) {
  if (!ctx || iters < 1) return POT3D_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const Grid &G = ctx->G;
  // continue the recurrences of the current state without a stopping test
  CK(cudaMemcpyAsync(ctx->hS, ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  Scalars h = *ctx->hS;
  h.stop = 0;
  h.status = 0;
  h.rtol = 0.0;
  h.maxit = h.iter + iters + 1;
  if (!(h.rho != 0.0)) h.rho = 1.0;
  if (!(h.bnorm > 0.0)) h.bnorm = 1.0;
  *ctx->hS = h;
  CK(cudaMemcpyAsync(ctx->S, ctx->hS, sizeof(Scalars), cudaMemcpyHostToDevice, s));
  cudaEvent_t ev[4];
  for (auto &e : ev) CK(cudaEventCreate(&e));
  double ta = 0, tb = 0, tp = 0;
  const bool pc2 = ctx->pc == 2;
  dim3 grd(G.ntj * G.ntk, G.nchunks);
  for (int it = 0; it < iters; it++) {
    const int par = (int)((h.iter + it) & 1);
    PassArgs a = make_args(ctx, par);
    a.hist = nullptr;
    a.finalize = 1;
    CK(cudaEventRecord(ev[0], s));
    CK(launch_k(false, kern_a(ctx), grd, dim3(NTHREADS), SMEM_A, s, ctx->tmaps, a, par));
    CK(cudaEventRecord(ev[1], s));
    PassArgs ab = a;
    ab.G.nchunks = ctx->nchunks_b;
    dim3 grdb(G.ntj * G.ntk, ctx->nchunks_b);
    CK(launch_k(false, kern_b(ctx), grdb, dim3(NTHREADS), SMEM_B, s, ctx->tmaps, ab, par));
    CK(cudaEventRecord(ev[2], s));
    ctx->n_launch += 2;
    if (pc2) {
      int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, 1, ctx->local_sum,
                         s, true);
      TRY(nk);
      ctx->n_launch += nk;
    }
    CK(cudaEventRecord(ev[3], s));
    CK(cudaEventSynchronize(ev[3]));
    float f;
    CK(cudaEventElapsedTime(&f, ev[0], ev[1])); ta += f;
    CK(cudaEventElapsedTime(&f, ev[1], ev[2])); tb += f;
    CK(cudaEventElapsedTime(&f, ev[2], ev[3])); tp += f;
  }
  for (auto &e : ev) cudaEventDestroy(e);
  if (ms_pass_a) *ms_pass_a = ta / iters;
  if (ms_pass_b) *ms_pass_b = tb / iters;
  if (ms_precond) *ms_precond = tp / iters;
  ctx->solved = false;
  return 0;
}

int pot3d_profile_iteration(pot3d_ctx *ctx, int32_t iters, double *ms, char *names, int32_t nmax) {
  if (!ctx || iters < 1 || !ms || !names || nmax < 1) return POT3D_ERR_INVALID;
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(ctx->hS, ctx->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  Scalars h = *ctx->hS;
  h.stop = 0;
  h.status = 0;
  h.rtol = 0.0;
  h.maxit = h.iter + iters + 2;
  h.epoch = ++ctx->epoch;
  if (!(h.rho != 0.0)) h.rho = 1.0;
  if (!(h.bnorm > 0.0)) h.bnorm = 1.0;
  *ctx->hS = h;
  CK(cudaMemcpyAsync(ctx->S, ctx->hS, sizeof(Scalars), cudaMemcpyHostToDevice, s));
  std::vector<double> acc;
  std::vector<const char *> nm;
  for (int it = 0; it < iters; it++) {
    StepTimer T;
    T.s = s;
    g_timer = &T;
    T.mark("start");
    int rc = enqueue_iteration(ctx, (int)((h.iter + it) & 1));
    g_timer = nullptr;
    if (rc < 0) return rc;
    CK(cudaStreamSynchronize(s));
    if (acc.empty()) {
      acc.assign(T.ev.size(), 0.0);
      nm = T.name;
    }
    for (size_t q = 1; q < T.ev.size() && q < acc.size(); q++) {
      float f = 0;
      cudaEventElapsedTime(&f, T.ev[q - 1], T.ev[q]);
      acc[q] += f;
    }
    for (auto e : T.ev) cudaEventDestroy(e);
  }
  int n = (int)std::min<size_t>(acc.size() - 1, (size_t)nmax);
  std::string all;
  for (int q = 0; q < n; q++) {
    ms[q] = acc[q + 1] / iters;
    all += nm[q + 1];
    all += ";";
  }
  strncpy(names, all.c_str(), 1023);
  names[1023] = 0;
  ctx->solved = false;
  return n;
}

int pot3d_trace_enable(pot3d_ctx *ctx, int32_t on) {
  if (!ctx) return POT3D_ERR_INVALID;
  ctx->trace_on = on != 0;
  return 0;
}

int pot3d_kernel_times(pot3d_ctx *ctx, double *us_pass_a, double *us_pass_b, int32_t *n) {
  if (!ctx || !us_pass_a || !us_pass_b || !n) return POT3D_ERR_INVALID;
  *n = 0;
  if (!ctx->trace) {
    ctx->err = "tracing not enabled (pot3d_trace_enable before pot3d_solve)";
    return POT3D_ERR_STATE;
  }
  CK(cudaSetDevice(ctx->device));
  std::vector<unsigned long long> t(64 * 16);
  CK(cudaMemcpy(t.data(), ctx->trace, t.size() * 8, cudaMemcpyDeviceToHost));
  double sa = 0, sb = 0;
  int cnt = 0;
  for (int it = 0; it < 64; it++) {
    const unsigned long long *r = &t[it * 16];
    if (!r[TR_A0] || !r[TR_A1] || !r[TR_B0] || !r[TR_B1] || r[TR_A1] < r[TR_A0] || r[TR_B1] < r[TR_B0]) continue;
    sa += (double)(r[TR_A1] - r[TR_A0]);
    sb += (double)(r[TR_B1] - r[TR_B0]);
    cnt++;
  }
  if (cnt) {
    *us_pass_a = sa / cnt / 1e3;
    *us_pass_b = sb / cnt / 1e3;
  }
  *n = cnt;
  return 0;
}

int pot3d_destroy(pot3d_ctx *ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->pc2) pc2_destroy(ctx->pc2, ctx->ufree, ctx->actx);
  ipc_release(ctx);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  dfree_all(ctx);
  if (ctx->hS) cudaFreeHost(ctx->hS);
  if (ctx->ev_edge) cudaEventDestroy(ctx->ev_edge);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return 0;
}

}  // extern "C"
