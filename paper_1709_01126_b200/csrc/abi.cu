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
#include <functional>
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
  int variant = 0;    // 0 standard PCG, 1 single-reduction CG1 (cg1.cu)
  int nchunks_b = 1;  // r-chunks of pass B (G.nchunks: pass A)
  bool pdl = true;    // programmatic dependent launch for the loop kernels (POT3D_PDL=0: off)
  int edge_blocks = 148 * 4;  // grid of the edge-shell kernel (POT3D_EDGE_BLOCKS)
  bool edge_in_a = true;      // pass A's first block row builds the edge shells (POT3D_EDGE_IN_A=0: kernel)
  int pcj = 1, pck = 1;       // fused passes: clusters of pcj x pck neighbouring tiles (POT3D_CLUSTER)
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
  Cg1Maps cmaps{};          // CG1: U[0] = P[0], U[1] = P[1] (peer-mapped), p = r, s = s_cg
  double *s_cg = nullptr;
  // PC3 (poly.cu): Chebyshev steps, their coefficients and work vectors
  int poly_m = 4;
  double poly_ratio = 100.0;
  PolyMaps pmaps{};
  double *p_res = nullptr, *p_d[2] = {nullptr, nullptr}, *p_x = nullptr;
  double p_theta = 0.0, p_c1[POLY_MMAX] = {0.0}, p_c2[POLY_MMAX] = {0.0};
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
  // loopback group (pot3d_runtime.loopback_slabs = k > 1): this context is the group's
  // handle (stream, graph, staging) and `slabs` are k slab contexts on the same device,
  // ranks 0..k-1 of a peer-memory exchange wired with plain device pointers
  std::vector<pot3d_ctx *> slabs;
  bool member = false;  // a slab context of a loopback group (no NCCL)
  std::vector<pot3d_ctx *> *group = nullptr;  // member: the group's slab list
  // multi-RHS batch (pot3d_runtime.nrhs = k > 1): this context is the
  // batch handle and `rhs` are k single-problem contexts on its stream whose x, r, p
  // vectors and scalars are stacked (rhs[q] at offset q), so one TMA descriptor and one
  // launch of each fused pass cover the batch (blockIdx.z = RHS).  rhs[0] (nrhs = k)
  // owns the graph, the per-RHS partials of the batched passes and the stacked histories.
  std::vector<pot3d_ctx *> rhs;
  int nrhs = 1;
  double *zpartials = nullptr;
  size_t zpart_len = 0;
  // state
  bool solved = false;
  bool has_x = false;  // x holds the last solve's Phi (a warm start may begin from it)
  bool warm = false;   // the next solve_begin starts from x0 = the current x (pot3d_solve_from)
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

// A fused pass (k_pass_a*, k_pass_b_*): grid.x becomes the tile count of a.G (padded to
// whole clusters) and the launch carries the cluster dimension a.G.cj * a.G.ck.
cudaError_t launch_pass(bool pdl, void (*k)(const TMaps, PassArgs, int), dim3 grid, size_t smem,
                        cudaStream_t s, const TMaps &T, const PassArgs &a, int parity) {
  cudaLaunchConfig_t cfg = {};
  grid.x = pass_tiles(a.G);
  cfg.gridDim = grid;
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    n++;
  }
  const int cs = std::max(a.G.cj, 1) * std::max(a.G.ck, 1);
  if (cs > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cs;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    n++;
  }
  cfg.attrs = n ? at : nullptr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, T, a, parity);
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

// user layout (r fastest, ni shells) <-> device cells (phi fastest).  ld > 0: the
// user array is a slab of an r-fastest array with ld shells (a device pointer at the
// slab's first shell: loopback groups stage the whole array on the device first).
int to_device_cells(pot3d_ctx *ctx, const double *user, double *dev_cells_first_shell, int ni,
                    long long stride_i, int ld = 0) {
  const size_t n = (size_t)ni * ctx->nt * ctx->np;
  const double *src = user;
  if (ld <= 0) ld = ni;
  if (ld == ni && !is_device_ptr(user)) {
    TRY(ensure_staging(ctx, n * sizeof(double)));
    CK(cudaMemcpyAsync(ctx->staging, user, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    src = ctx->staging;
  }
  dim3 blk(32, 8), grd((ctx->np + 31) / 32, (ni + 31) / 32, ctx->nt);
  k_transpose<<<grd, blk, 0, ctx->stream>>>(ni, ctx->nt, ctx->np, stride_i, ctx->G.PK, COFF, src,
                                            dev_cells_first_shell, 1, ld);
  CK(cudaGetLastError());
  ctx->n_launch++;
  return 0;
}

int from_device_cells(pot3d_ctx *ctx, const double *dev_first, double *user, int ni, int nj,
                      long long stride_i, int coff = COFF, int ld = 0) {
  const size_t n = (size_t)ni * nj * ctx->np;
  if (ld <= 0) ld = ni;
  const bool dev = ld != ni || is_device_ptr(user);
  double *dst = user;
  if (!dev) {
    TRY(ensure_staging(ctx, n * sizeof(double)));
    dst = ctx->staging;
  }
  dim3 blk(32, 8), grd((ctx->np + 31) / 32, (ni + 31) / 32, nj);
  k_transpose<<<grd, blk, 0, ctx->stream>>>(ni, nj, ctx->np, stride_i, ctx->G.PK, coff, dev_first, dst,
                                            0, ld);
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
    cudaIpcMemHandle_t h[5];  // P[0], P[1], the mailbox; PC3: the Chebyshev d[0], d[1]
    int32_t ok, nr_loc, pad0, pad1;
  };
  const int n = ctx->nranks, me = ctx->rank;
  cudaStream_t s = ctx->stream;
  IpcInfo mine{};
  mine.ok = ctx->xfer_want && ctx->mail != nullptr;
  mine.nr_loc = ctx->G.nr_loc;
  if (mine.ok && (cudaIpcGetMemHandle(&mine.h[0], ctx->P[0]) != cudaSuccess ||
                  cudaIpcGetMemHandle(&mine.h[1], ctx->P[1]) != cudaSuccess ||
                  cudaIpcGetMemHandle(&mine.h[2], ctx->mail) != cudaSuccess ||
                  (ctx->pc == POT3D_PC3 && (cudaIpcGetMemHandle(&mine.h[3], ctx->p_d[0]) != cudaSuccess ||
                                            cudaIpcGetMemHandle(&mine.h[4], ctx->p_d[1]) != cudaSuccess)))) {
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
    for (int q = 0; q < 2 && ok && ctx->pc == POT3D_PC3; q++) {
      if (me > 0) ok = ok && (T.d_lo[q] = static_cast<double *>(open(all[me - 1].h[3 + q]))) != nullptr;
      if (me < n - 1) ok = ok && (T.d_hi[q] = static_cast<double *>(open(all[me + 1].h[3 + q]))) != nullptr;
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
  // a batch leader's descriptors span the k stacked vectors (nr_loc + 2 planes each)
  cuuint64_t dims[3] = {(cuuint64_t)G.PK, (cuuint64_t)G.nt, (cuuint64_t)(G.nr_loc + 2) * ctx->nrhs};
  cuuint64_t strides[2] = {(cuuint64_t)G.PK * 8, (cuuint64_t)G.plane * 8};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  // L2 promotion of the boxes' misses: 64 B for the haloed boxes (their halo columns
  // straddle the neighbour tiles' sectors; large pass A: ncu DRAM reads 4.3 -> 3.9 GB,
  // 1004 -> 978 us live), 128 B for the interior boxes.  POT3D_L2PROMO = 0 / 64 / 128 /
  // 256 overrides the haloed boxes' choice (A/B only).
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (b0 == SROW) {
    const char *e = getenv("POT3D_L2PROMO");
    const int v = e ? atoi(e) : 64;
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                   : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                             : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    ctx->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return POT3D_ERR_CUDA;
  }
  return 0;
}

int make_maps(pot3d_ctx *ctx) {
  TRY(make_map(ctx, &ctx->tmaps.src_h, ctx->pc >= 2 ? ctx->z : ctx->r, SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.p_h[0], ctx->P[0], SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.p_h[1], ctx->P[1], SROW, TR));
  TRY(make_map(ctx, &ctx->tmaps.r_i, ctx->r, TKB, TJ));
  TRY(make_map(ctx, &ctx->tmaps.x_i, ctx->x, TKB, TJ));
  if (ctx->pc == 3) {
    TRY(make_map(ctx, &ctx->pmaps.d_h[0], ctx->p_d[0], SROW, TR));
    TRY(make_map(ctx, &ctx->pmaps.d_h[1], ctx->p_d[1], SROW, TR));
    TRY(make_map(ctx, &ctx->pmaps.res_i, ctx->p_res, TKB, TJ));
    TRY(make_map(ctx, &ctx->pmaps.x_i, ctx->p_x, TKB, TJ));
    TRY(make_map(ctx, &ctx->pmaps.r_i, ctx->r, TKB, TJ));
  }
  if (ctx->variant == 1) {
    TRY(make_map(ctx, &ctx->cmaps.u_h[0], ctx->P[0], SROW, TR));
    TRY(make_map(ctx, &ctx->cmaps.u_h[1], ctx->P[1], SROW, TR));
    TRY(make_map(ctx, &ctx->cmaps.p_i, ctx->r, TKB, TJ));
    TRY(make_map(ctx, &ctx->cmaps.s_i, ctx->s_cg, TKB, TJ));
    TRY(make_map(ctx, &ctx->cmaps.x_i, ctx->x, TKB, TJ));
  }
  return 0;
}


PassArgs make_args(pot3d_ctx *ctx, int parity) {
  PassArgs a{};
  a.G = ctx->G;
  a.G.cj = ctx->pcj;
  a.G.ck = ctx->pck;
  a.M = ctx->M;
  a.S = ctx->S;
  a.r = ctx->r;
  a.r_out = ctx->r;
  a.z = ctx->pc >= 2 ? ctx->z : ctx->r;  // PC1 stores z = D^-1 r in ctx->r (A22)
  a.p_old = ctx->P[parity];
  a.p_new = ctx->P[parity ^ 1];
  a.x = ctx->x;
  a.partials = ctx->partials;
  a.hist = ctx->hist;
  a.finalize = ctx->nranks == 1 ? 1 : 0;
  a.local_sum = ctx->local_sum;
  if (ctx->nrhs > 1) {  // batch leader: per-RHS partials and histories (pass_common.cuh)
    a.partials = ctx->zpartials;
    a.pstride = (long long)ctx->zpart_len;
    a.hstride = ctx->hist_len;
  }
  return a;
}

using PassKernel = void (*)(const TMaps, PassArgs, int);
PassKernel kern_a(const pot3d_ctx *) { return k_pass_a; }
// parity = iteration index & 1 (every solve starts at iteration 0; graphs hold an even
// number of iterations): PC1 updates x on odd iterations only (A23)
PassKernel kern_b(const pot3d_ctx *ctx, int parity) {
  if (ctx->pc >= 2) return k_pass_b_pc2;
  return parity ? k_pass_b_pc1_odd : k_pass_b_pc1_even;
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

// The kernels of one peer-memory iteration as separate launch steps.  A process
// with one context runs them in order; a loopback group (several slab contexts on
// one device, pot3d_runtime.loopback_slabs) runs step q of every slab before step
// q+1 of any, so every wait of the exchange protocol (halo flags, mailboxes) is on
// work that an earlier launch of the same stream already finished.
using Step = std::function<int()>;
// ---------------------------------------------------------------------------
// CG1 (single-reduction PCG, cg1.cu): per iteration K1 (vector update, u from
// U[parity] into U[parity^1]), the halo of the new u, K2 (w = A u and the three
// inner products), one reduction.  With peer memory (rank processes whose peers
// are mapped, loopback slabs) K1 stores the halo into the neighbours' ghost shells
// and K2 posts the sums to every mailbox (cg1.cu); otherwise NCCL send/recv and an
// all-gather.  The u vectors live in P[0], P[1] (the peer-mapped buffers), p in r.
// ---------------------------------------------------------------------------
double *cg1_u(pot3d_ctx *c, int b) { return c->P[b]; }
bool cg1_peer(const pot3d_ctx *c) { return c->nranks > 1 && c->xfer && c->peers && !getenv("POT3D_CG1_NCCL"); }

Cg1Args cg1_args(pot3d_ctx *ctx, int init) {
  Cg1Args a{};
  a.G = ctx->G;
  a.M = ctx->M;
  a.S = ctx->S;
  a.u[0] = cg1_u(ctx, 0);
  a.u[1] = cg1_u(ctx, 1);
  a.p = ctx->r;
  a.peers = cg1_peer(ctx) ? ctx->peers : nullptr;
  a.s = ctx->s_cg;
  a.x = ctx->x;
  a.partials = ctx->partials;
  a.hist = ctx->hist;
  a.local_sum = ctx->local_sum;
  a.finalize = (ctx->nranks == 1) ? 1 : 0;
  a.init = init;
  return a;
}

// the steps of one CG1 iteration (parity: u is read from U[parity]); init: only the
// dots of u_0 (alpha_0) from U[0]
std::vector<Step> cg1_steps(pot3d_ctx *ctx, int parity, bool init) {
  std::vector<Step> st;
  const Grid &G = ctx->G;
  const int b = init ? 0 : (parity ^ 1);  // the u the dots read
  if (!init) {
    st.push_back([=]() -> int {
      Cg1Args a = cg1_args(ctx, 0);
      a.G.nchunks = ctx->nchunks_b;
      CK(launch_k(ctx->pdl, parity ? k_cg1_update_odd : k_cg1_update_even, dim3(G.ntj * G.ntk, ctx->nchunks_b),
                  dim3(NTHREADS), SMEM_C1, ctx->stream, ctx->cmaps, a, parity));
      MARK("cg1_update");
      ctx->n_enq++;
      return 0;
    });
  }
  const bool peer = cg1_peer(ctx) && !init;  // the start's halo and sums go the copy way
  if (ctx->nranks > 1 && !peer) {  // the halo of the u the dots (and the next update) read
    st.push_back([=]() -> int {
      if (!ctx->group) return halo_exchange(ctx, cg1_u(ctx, b));
      const std::vector<pot3d_ctx *> &M = *ctx->group;
      const int q = ctx->rank;
      const size_t bytes = (size_t)G.plane * sizeof(double);
      if (q > 0)
        CK(cudaMemcpyAsync(cg1_u(M[q - 1], b) + sidx(M[q - 1]->G, M[q - 1]->G.nr_loc), cg1_u(ctx, b) + sidx(G, 0),
                           bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      if (q + 1 < (int)M.size())
        CK(cudaMemcpyAsync(cg1_u(M[q + 1], b) + sidx(M[q + 1]->G, -1), cg1_u(ctx, b) + sidx(G, G.nr_loc - 1),
                           bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      return 0;
    });
  }
  st.push_back([=]() -> int {
    Cg1Args a = cg1_args(ctx, init ? 1 : 0);
    CK(launch_k(ctx->pdl, k_cg1_dots, dim3(G.ntj * G.ntk, G.nchunks), dim3(NTHREADS), SMEM_C2, ctx->stream,
                ctx->cmaps, a, b));
    MARK("cg1_dots");
    ctx->n_enq++;
    return 0;
  });
  if (peer) {  // one reduction through the mailboxes, summed in rank order
    st.push_back([=]() -> int {
      CK(launch_k(ctx->pdl, k_finalize_cg1_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S,
                  (const PeerTab *)ctx->peers, ctx->hist));
      MARK("cg1_finalize");
      ctx->n_enq++;
      return 0;
    });
  } else if (ctx->nranks > 1) {  // one reduction: every rank's (gamma, delta, ||r||^2) in rank order
    st.push_back([=]() -> int {
      if (!ctx->group) {
        NK(ncclAllGather(ctx->local_sum, ctx->gathered, 4, ncclDouble, ctx->comm, ctx->stream));
      } else {
        const std::vector<pot3d_ctx *> &M = *ctx->group;
        for (size_t r = 0; r < M.size(); r++)
          CK(cudaMemcpyAsync(ctx->gathered + 4 * r, M[r]->local_sum, 3 * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
      }
      CK(launch_k(ctx->pdl, k_finalize_cg1, dim3(1), dim3(1), 0, ctx->stream, ctx->S, (const double *)ctx->gathered,
                  ctx->nranks, init ? (double *)nullptr : ctx->hist, init ? 1 : 0));
      MARK("cg1_finalize");
      ctx->n_enq++;
      return 0;
    });
  }
  return st;
}

std::vector<Step> poly_steps(pot3d_ctx *ctx, int finalize, bool iteration, int nz = 1,
                             const PeerTab *peers = nullptr);

std::vector<Step> iteration_steps(pot3d_ctx *ctx, int parity) {
  if (ctx->variant == 1) return cg1_steps(ctx, parity, false);
  std::vector<Step> st;
  const Grid &G = ctx->G;
  PassArgs a = make_args(ctx, parity);
  a.peers = ctx->peers;
  PassArgs ab = a;  // pass B: its own r-chunking
  ab.G.nchunks = ctx->nchunks_b;
  const dim3 grd(G.ntj * G.ntk, G.nchunks), grdb(G.ntj * G.ntk, ctx->nchunks_b);
  const bool pc2 = ctx->pc == 2;
  const bool zs = ctx->pc >= 2;  // PC2 / PC3: z stored apart from r
  const PeerTab *pt = ctx->peers;
  auto fin = [ctx, pt](int kind, int what, double *hist, const char *nm) -> Step {
    return [=]() -> int {
      CK(launch_k(ctx->pdl, k_finalize_mail, dim3(1), dim3(1), 0, ctx->stream, ctx->S, pt, kind, what, hist));
      MARK(nm);
      ctx->n_enq++;
      return 0;
    };
  };
  auto pass_b = [ctx, grdb, parity](PassArgs bx) -> Step {
    return [=]() -> int {
      CK(launch_pass(ctx->pdl, kern_b(ctx, parity), grdb, SMEM_B, ctx->stream, ctx->tmaps, bx, parity));
      MARK("passB");
      ctx->n_enq++;
      return 0;
    };
  };
  if (ctx->edge_in_a && !zs) {
    // pass A's first block row builds and sends the edge shells beside the interior
    // chunks; beta is finalised by its own kernel after pass B.  The halo waits of
    // the chunks next to a ghost shell (scheduled last in the grid) assume the
    // neighbour's edge blocks (blockIdx.y = 0, scheduled first) get dispatched --
    // linear block dispatch; POT3D_EDGE_IN_A=0 selects the separate edge kernel.
    PassArgs ax = a;
    ax.G.part = 3;
    ax.G.role_rows = 1;
    // at least 3 chunks, so an interior chunk runs while the halo travels (the two
    // chunks touching the ghost shells are scheduled last): 4 GPUs x 19 shells,
    // 84.9 us per iteration with 3 chunks vs 89.1 with the single-GPU choice of 1
    static const int min_a = getenv("POT3D_MIN_CHUNKS_A") ? std::max(1, atoi(getenv("POT3D_MIN_CHUNKS_A"))) : 3;
    if (ax.G.nchunks < min_a && G.nr_loc >= 2 * min_a) ax.G.nchunks = min_a;
    st.push_back([=]() -> int {
      CK(launch_pass(ctx->pdl, kern_a(ctx), dim3(0, ax.G.nchunks + 1), SMEM_A, ctx->stream, ctx->tmaps, ax,
                     parity));
      MARK("passA");
      ctx->n_enq++;
      return 0;
    });
    st.push_back(fin(MAIL_A, 0, nullptr, "finalize_alpha"));
    st.push_back(pass_b(ab));
    st.push_back(fin(MAIL_B, 1, ctx->hist, "finalize_beta"));
    return st;
  }
  // PC1: the previous iteration's beta finalisation lives in edge_p (fold)
  const int fold = zs ? 0 : 1;
  st.push_back([=]() -> int {
    CK(launch_k(ctx->pdl, k_edge_p, dim3(ctx->edge_blocks), dim3(256), 0, ctx->stream, G, ctx->M, ctx->S,
                (const double *)(zs ? ctx->z : ctx->r), (const double *)ctx->P[parity], ctx->P[parity ^ 1], 1,
                pt, parity ^ 1, ctx->hist, fold));
    MARK("edge_p");
    ctx->n_enq++;
    return 0;
  });
  PassArgs ax = a;
  ax.G.part = 3;
  st.push_back([=]() -> int {
    CK(launch_pass(ctx->pdl, kern_a(ctx), grd, SMEM_A, ctx->stream, ctx->tmaps, ax, parity));
    MARK("passA");
    ctx->n_enq++;
    return 0;
  });
  st.push_back(fin(MAIL_A, 0, nullptr, "finalize_alpha"));
  PassArgs bx = ab;
  bx.fold = fold;  // PC1: pass B only posts its sums and marks them pending
  st.push_back(pass_b(bx));
  if (pc2) {
    st.push_back(fin(MAIL_B, 2, ctx->hist, "finalize_rr"));
    st.push_back([=]() -> int {
      int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, 0, ctx->local_sum,
                         ctx->stream, true, pt);
      if (nk < 0) {
        ctx->err = pc2_last_error();
        return POT3D_ERR_CUDA;
      }
      ctx->n_enq += nk;
      MARK("pc2");
      return 0;
    });
    st.push_back(fin(MAIL_C, 3, nullptr, "finalize_rho"));
  }
  if (ctx->pc == 3) {  // the Chebyshev steps (halo of d between them), r.z to every mailbox
    st.push_back(fin(MAIL_B, 2, ctx->hist, "finalize_rr"));
    for (Step &f : poly_steps(ctx, 0, true, 1, pt)) st.push_back(f);
    st.push_back(fin(MAIL_C, 3, nullptr, "finalize_rho"));
  }
  return st;
}

// halo of a cell array between r-slabs: NCCL send/recv (rank processes) or device copies
// into the siblings' ghost shells (loopback slabs, which run it phase by phase)
int halo_slab(pot3d_ctx *ctx, double *(*arr)(pot3d_ctx *)) {
  if (!ctx->group) return halo_exchange(ctx, arr(ctx));
  const std::vector<pot3d_ctx *> &M = *ctx->group;
  const Grid &G = ctx->G;
  const int q = ctx->rank;
  const size_t bytes = (size_t)G.plane * sizeof(double);
  if (q > 0)
    CK(cudaMemcpyAsync(arr(M[q - 1]) + sidx(M[q - 1]->G, M[q - 1]->G.nr_loc), arr(ctx) + sidx(G, 0), bytes,
                       cudaMemcpyDeviceToDevice, ctx->stream));
  if (q + 1 < (int)M.size())
    CK(cudaMemcpyAsync(arr(M[q + 1]) + sidx(M[q + 1]->G, -1), arr(ctx) + sidx(G, G.nr_loc - 1), bytes,
                       cudaMemcpyDeviceToDevice, ctx->stream));
  return 0;
}

// PC3: z = M^-1 r (ctx->r -> ctx->z), the partial r.z to rho/beta (finalize), every
// mailbox (peers) or local_sum, as launch steps.  Across ranks the Chebyshev step k
// reads d_{k-1} with the neighbours' edge shells: a halo step precedes it.
// nz: problems covered (a batch leader's loop and profile: nrhs; the start of a solve: 1)
double *poly_d0(pot3d_ctx *c) { return c->p_d[0]; }
double *poly_d1(pot3d_ctx *c) { return c->p_d[1]; }

std::vector<Step> poly_steps(pot3d_ctx *ctx, int finalize, bool iteration, int nz, const PeerTab *peers) {
  std::vector<Step> st;
  const Grid &G = ctx->G;
  PolyArgs a{};
  a.G = G;
  a.M = ctx->M;
  a.S = ctx->S;
  a.r = ctx->r;
  a.res = ctx->p_res;
  a.d[0] = ctx->p_d[0];
  a.d[1] = ctx->p_d[1];
  a.x = ctx->p_x;
  a.z = ctx->z;
  a.theta = ctx->p_theta;
  for (int k = 0; k < POLY_MMAX; k++) {
    a.c1[k] = ctx->p_c1[k];
    a.c2[k] = ctx->p_c2[k];
  }
  a.partials = nz > 1 ? ctx->zpartials : ctx->partials;
  a.pstride = nz > 1 ? (long long)ctx->zpart_len : 0;
  a.local_sum = ctx->local_sum;
  a.finalize = finalize;
  a.predicated = iteration ? 1 : 0;
  a.peers = peers;
  // across ranks with peer memory the kernels exchange d's halo themselves (flags)
  const bool peer_halo = ctx->nranks > 1 && ctx->xfer && ctx->peers && ctx->pc == POT3D_PC3;
  a.hpeers = peer_halo ? ctx->peers : nullptr;
  const bool pdl = ctx->pdl && iteration && (ctx->nranks == 1 || peer_halo);
  auto count = [ctx, iteration]() {
    if (iteration)
      ctx->n_enq++;
    else
      ctx->n_launch++;
  };
  st.push_back([=]() -> int {
    CK(launch_k(pdl, k_poly_init, dim3(148 * 8, nz), dim3(256), 0, ctx->stream, a));
    count();
    return 0;
  });
  PolyArgs ak = a;
  ak.G.nchunks = ctx->nchunks_b;
  const dim3 grd(G.ntj * G.ntk, ctx->nchunks_b, nz);
  for (int k = 1; k < ctx->poly_m; k++) {
    if (ctx->nranks > 1 && !peer_halo) {
      const int src = (k - 1) & 1;  // d_{k-1}
      st.push_back([=]() -> int { return halo_slab(ctx, src ? poly_d1 : poly_d0); });
    }
    st.push_back([=]() -> int {
      CK(launch_k(pdl, k + 1 == ctx->poly_m ? k_poly_last : k_poly_step, grd, dim3(NTHREADS), SMEM_P, ctx->stream,
                  ctx->pmaps, ak, k));
      count();
      if (k + 1 == ctx->poly_m) MARK("pc3");
      return 0;
    });
  }
  return st;
}

int poly_apply(pot3d_ctx *ctx, int finalize, bool iteration, int nz = 1, const PeerTab *peers = nullptr) {
  for (auto &f : poly_steps(ctx, finalize, iteration, nz, peers)) TRY(f());
  return 0;
}

int enqueue_iteration(pot3d_ctx *ctx, int parity) {
  if (ctx->variant == 1) {
    for (auto &f : cg1_steps(ctx, parity, false)) TRY(f());
    return 0;
  }
  const Grid &G = ctx->G;
  PassArgs a = make_args(ctx, parity);
  dim3 grd(G.ntj * G.ntk, G.nchunks, ctx->nrhs);  // batch: blockIdx.z = right-hand side
  PassArgs ab = a;  // pass B: its own r-chunking
  ab.G.nchunks = ctx->nchunks_b;
  dim3 grdb(G.ntj * G.ntk, ctx->nchunks_b, ctx->nrhs);
  const bool pc2 = ctx->pc == 2;
  const bool zs = ctx->pc >= 2;  // PC2 / PC3: z stored apart from r
  const bool multi = ctx->nranks > 1;
  if (ctx->xfer) {
    // peer memory: edge shells of p_k stored into the neighbours' ghost shells
    // (flag per iteration); pass A waits for that flag only in the blocks whose
    // chunk touches a ghost shell (scheduled last); the rank sums go straight into
    // every rank's mailbox from the reductions' last blocks
    for (auto &f : iteration_steps(ctx, parity)) TRY(f());
    return 0;
  }
  if (multi && G.nr_loc >= 3) {
    // edge shells first; their halo travels on the comm stream while pass A
    // covers the interior shells, then pass A finishes the two edge shells
    k_edge_p<<<148 * 4, 256, 0, ctx->stream>>>(G, ctx->M, ctx->S, zs ? ctx->z : ctx->r,
                                                ctx->P[parity], ctx->P[parity ^ 1], 1,
                                                nullptr, 0, nullptr, 0);
    CK(cudaGetLastError());
    ctx->n_enq++;
    MARK("edge_p");
    CK(cudaEventRecord(ctx->ev_edge, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_edge, 0));
    TRY(halo_exchange(ctx, ctx->P[parity ^ 1], ctx->comm_stream));
    CK(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
    const int nci = std::max(1, std::min(G.nchunks, G.nr_loc - 2));
    const int ntl = pass_tiles(a.G);
    PassArgs ai = a, ae = a;
    ai.G.part = 1;
    ai.G.nchunks = nci;
    ai.G.blk_off = 0;
    ai.G.blk_total = ntl * (nci + 2);
    ae.G.part = 2;
    ae.G.blk_off = ntl * nci;
    ae.G.blk_total = ntl * (nci + 2);
    CK(launch_pass(false, kern_a(ctx), dim3(ntl, nci), SMEM_A, ctx->stream, ctx->tmaps, ai, parity));
    ctx->n_enq++;
    MARK("passA_interior");
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    MARK("halo_wait");
    CK(launch_pass(false, kern_a(ctx), dim3(ntl, 2), SMEM_A, ctx->stream, ctx->tmaps, ae, parity));
    ctx->n_enq++;
    MARK("passA_edge");
  } else {
    if (multi) {
      k_edge_p<<<148 * 4, 256, 0, ctx->stream>>>(G, ctx->M, ctx->S, zs ? ctx->z : ctx->r,
                                                  ctx->P[parity], ctx->P[parity ^ 1], 1,
                                                nullptr, 0, nullptr, 0);
      CK(cudaGetLastError());
      ctx->n_enq++;
      TRY(halo_exchange(ctx, ctx->P[parity ^ 1]));
    }
    CK(launch_pass(ctx->pdl && !multi, kern_a(ctx), grd, SMEM_A, ctx->stream, ctx->tmaps, a, parity));
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
  CK(launch_pass(ctx->pdl && !multi, kern_b(ctx, parity), grdb, SMEM_B, ctx->stream, ctx->tmaps, ab, parity));
    ctx->n_enq++;
  MARK("passB");
  if (multi) {
    TRY(gather_sums(ctx, 2));
    MARK("allgather_rz_rr");
    if (zs)
      k_finalize_rr<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks, ctx->hist);
    else
      k_finalize_beta<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks, ctx->hist);
    CK(cudaGetLastError());
    ctx->n_enq++;
  }
  if (ctx->pc == 3) {
    TRY(poly_apply(ctx, multi ? 0 : 1, true, ctx->nrhs));
    if (multi) {  // r.z across the ranks, then rho / beta
      TRY(gather_sums(ctx, 1));
      k_finalize_rho<<<1, 1, 0, ctx->stream>>>(ctx->S, ctx->gathered, ctx->nranks);
      CK(cudaGetLastError());
      ctx->n_enq++;
    }
  }
  if (pc2) {
    // a batch leader: the sweeps of all nrhs problems in one launch per sweep
    const long long vst = ctx->nrhs > 1 ? (long long)(G.nr_loc + 2) * G.plane : 0;
    int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->nrhs > 1 ? ctx->zpartials : ctx->partials,
                       multi ? 0 : 1, ctx->local_sum, ctx->stream, true, nullptr, ctx->nrhs, vst,
                       (long long)ctx->zpart_len);
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
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pass_b_pc1_odd, NTHREADS, SMEM_B));
  int occa = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occa, k_pass_a, NTHREADS, SMEM_A));
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

// ---------------------------------------------------------------------------
// Solve phases over the contexts of one process: {ctx} for a rank process, the k
// slab contexts of a loopback group (handle ctx).  The group runs every phase for
// all slabs on the one stream, so each collective point (gather_all, halo_all)
// sees all slabs' inputs already enqueued before it.
// ---------------------------------------------------------------------------
std::vector<pot3d_ctx *> members(pot3d_ctx *ctx) {
  if (!ctx->slabs.empty()) return ctx->slabs;
  return {ctx};
}

// every rank's / slab's 2-double local sums into every `gathered`, rank order
int gather_all(std::vector<pot3d_ctx *> &M) {
  pot3d_ctx *ctx = M[0];
  if (M.size() == 1) return gather_sums(ctx, 2);
  for (pot3d_ctx *m : M)
    for (size_t r = 0; r < M.size(); r++)
      CK(cudaMemcpyAsync(m->gathered + 2 * r, M[r]->local_sum, 2 * sizeof(double), cudaMemcpyDeviceToDevice,
                         m->stream));
  return 0;
}

// ghost shells of a cell array from the neighbours' edge shells
template <typename F>
int halo_all(std::vector<pot3d_ctx *> &M, F arr) {
  pot3d_ctx *ctx = M[0];
  if (M.size() == 1) return halo_exchange(ctx, arr(ctx));
  const size_t bytes = (size_t)ctx->G.plane * sizeof(double);
  for (size_t q = 0; q < M.size(); q++) {
    pot3d_ctx *m = M[q];
    if (q > 0)
      CK(cudaMemcpyAsync(arr(M[q - 1]) + sidx(M[q - 1]->G, M[q - 1]->G.nr_loc), arr(m) + sidx(m->G, 0), bytes,
                         cudaMemcpyDeviceToDevice, m->stream));
    if (q + 1 < M.size())
      CK(cudaMemcpyAsync(arr(M[q + 1]) + sidx(M[q + 1]->G, -1), arr(m) + sidx(m->G, m->G.nr_loc - 1), bytes,
                         cudaMemcpyDeviceToDevice, m->stream));
  }
  return 0;
}

// the cells of every member (F: device pointer of shell 0, device layout) into one
// r-fastest user array (host or device); a group assembles the whole grid
template <typename F>
int cells_out(pot3d_ctx *h, std::vector<pot3d_ctx *> &M, F src, double *user, int nj = 0,
              long long stride_i = 0, int coff = COFF, std::function<int(pot3d_ctx *)> ni_of = nullptr) {
  pot3d_ctx *ctx = h;
  if (nj <= 0) nj = h->nt;
  auto ni_f = [&](pot3d_ctx *m) { return ni_of ? ni_of(m) : m->G.nr_loc; };
  auto stride_f = [&](pot3d_ctx *m) { return stride_i > 0 ? stride_i : m->G.plane; };
  if (M.size() == 1) return from_device_cells(M[0], src(M[0]), user, ni_f(M[0]), nj, stride_f(M[0]), coff);
  int ld = 0;
  for (pot3d_ctx *m : M) ld += ni_f(m);
  const size_t n = (size_t)ld * nj * h->np;
  const bool dev = is_device_ptr(user);
  double *dst = user;
  if (!dev) {
    TRY(ensure_staging(h, n * sizeof(double)));
    dst = h->staging;
  }
  int off = 0;
  for (pot3d_ctx *m : M) {
    TRY(from_device_cells(m, src(m), dst + off, ni_f(m), nj, stride_f(m), coff, ld));
    off += ni_f(m);
  }
  if (!dev) {
    CK(cudaMemcpyAsync(user, dst, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return 0;
}

// an r-fastest user array (this process's cells: the whole grid for a group) into
// every member's device cells (F: device pointer of shell 0)
template <typename F>
int cells_in(pot3d_ctx *h, std::vector<pot3d_ctx *> &M, const double *user, F dst) {
  pot3d_ctx *ctx = h;
  if (M.size() == 1) return to_device_cells(M[0], user, dst(M[0]), M[0]->G.nr_loc, M[0]->G.plane);
  const size_t n = (size_t)h->nr * h->nt * h->np;
  const double *src = user;
  if (!is_device_ptr(user)) {
    TRY(ensure_staging(h, n * sizeof(double)));
    CK(cudaMemcpyAsync(h->staging, user, n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    src = h->staging;
  }
  for (pot3d_ctx *m : M) TRY(to_device_cells(m, src + m->G.i0, dst(m), m->G.nr_loc, m->G.plane, h->nr));
  return 0;
}

// hist buffer (maxit+1 doubles, capped at 2^24 entries); stale: the graph holds the old one
int ensure_hist(pot3d_ctx *ctx, int64_t maxit, bool &stale) {
  const int64_t hlen = std::min<int64_t>(maxit + 1, (int64_t)1 << 24);
  if (hlen > ctx->hist_len) {
    double *h = nullptr;
    TRY(dalloc(ctx, &h, (size_t)hlen));
    ctx->hist = h;
    ctx->hist_len = hlen;
    stale = true;
  }
  return 0;
}

// batch: one buffer of k histories (stride hist_len, the passes' hstride)
int ensure_hist_batch(pot3d_ctx *lead, std::vector<pot3d_ctx *> &M, int64_t maxit, bool &stale) {
  pot3d_ctx *ctx = lead;
  const int64_t hlen = std::min<int64_t>(maxit + 1, (int64_t)1 << 24);
  if (hlen > lead->hist_len) {
    double *h = nullptr;
    TRY(dalloc(lead, &h, (size_t)hlen * M.size()));
    for (size_t q = 0; q < M.size(); q++) {
      M[q]->hist = h + q * hlen;
      M[q]->hist_len = hlen;
    }
    stale = true;
  }
  return 0;
}

struct PinnedScalars {  // pinned host mirror of n device scalar blocks, freed on every path
  Scalars *p = nullptr;
  ~PinnedScalars() {
    if (p) cudaFreeHost(p);
  }
};

int build_graph_group(pot3d_ctx *h);

// x0 = 0, r = b, p = 0 (A9), the device scalars, PC2: z0 = M^-1 b, local init sums.
// Warm start (ctx->warm, pot3d_solve_from): x holds x0 (interior cells), r = b - A x0.
// phase 0: all of it; a warm start across ranks / slabs runs phase 1 (up to the local
// sums of ||b||), then -- after the global ||b|| and x0's halo (solve_run) -- phase 2.
int solve_begin(pot3d_ctx *ctx, double rtol, int64_t maxit, int phase = 0) {
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
  const size_t cells = (size_t)(G.nr_loc + 2) * G.plane;
  const bool warm = ctx->warm;
  if (phase != 2) {  // phase 2 starts at the residual of x0
    if (!warm) {
      CK(cudaMemsetAsync(ctx->x, 0, cells * sizeof(double), s));
    } else {  // the ghost shells of x0 are zero for the apply (the BCs are folded, A7)
      CK(cudaMemsetAsync(ctx->x + sidx(G, -1), 0, G.plane * sizeof(double), s));
      CK(cudaMemsetAsync(ctx->x + sidx(G, G.nr_loc), 0, G.plane * sizeof(double), s));
    }
    CK(cudaMemsetAsync(ctx->r, 0, cells * sizeof(double), s));
    CK(cudaMemsetAsync(ctx->P[0], 0, cells * sizeof(double), s));
    CK(cudaMemsetAsync(ctx->P[1], 0, cells * sizeof(double), s));
    if (ctx->s_cg) CK(cudaMemsetAsync(ctx->s_cg, 0, cells * sizeof(double), s));
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
    h0.maxit = (long long)maxit;  // the history keeps the first hist_len entries
    h0.hist_len = ctx->hist_len;
    CK(cudaMemcpyAsync(ctx->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
    if (warm) {
      // ||b|| from r = b (the stopping test stays relative to b, A9); across ranks only
      // this rank's sums here (phase 1)
      k_init_dots<<<148 * 4, 256, 0, s>>>(G, ctx->M, ctx->S, ctx->r, ctx->partials, phase == 1 ? 0 : 1,
                                          ctx->local_sum, 0, nullptr, 0, nullptr);
      CK(cudaGetLastError());
      ctx->n_launch++;
      if (phase == 1) return 0;
    }
  }  // phase != 2
  if (phase != 3) {  // phase 3 starts at the init dots (loopback PC3, after the z0 steps)
    if (warm) {
      // r = b - A x0 over every cell and its periodic ghost columns (a stencil operand
      // of pass A); x0's ghost shells hold the neighbours' edge shells (halo) or zero
      k_apply<<<148 * 4, 256, 0, s>>>(G, ctx->M, ctx->x, ctx->r, ctx->bshell, G.i0 == 0 ? 0 : -1000, nullptr,
                                      nullptr, nullptr);
      k_fix_ghost_cols<<<(G.nr_loc * ctx->nt + 255) / 256, 256, 0, s>>>(G, ctx->r, 0, G.nr_loc);
      CK(cudaGetLastError());
      ctx->n_launch += 2;
    }
    // z0 = M^-1 r0, rho0 = r0.z0, ||b|| (a10 init)
    if (ctx->pc == 2) {
      int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, ctx->partials, 0, ctx->local_sum,
                         s, false);
      TRY(nk);
      CK(cudaGetLastError());
      ctx->n_launch += nk;
    }
    if (ctx->pc == 3) {
      // loopback slabs exchange d between the Chebyshev steps phase by phase: solve_run
      // runs z0's steps for the whole group, then phase 3
      if (ctx->group) return 0;
      TRY(poly_apply(ctx, 0, false));  // z0 = M^-1 r0 (rank processes: NCCL halos)
    }
  }
  k_init_dots<<<148 * 4, 256, 0, s>>>(G, ctx->M, ctx->S, ctx->r, ctx->partials, ctx->nranks == 1,
                                      ctx->local_sum, ctx->pc >= 2, ctx->z, warm ? 1 : 0,
                                      warm ? ctx->hist : nullptr);
  CK(cudaGetLastError());
  ctx->n_launch++;
  if (ctx->pc == 1) {
    // PC1 keeps z = D^-1 r instead of r (A22): z_0 = D^-1 b in place (ghost columns included)
    k_edge_p<<<148 * 8, 256, 0, s>>>(G, ctx->M, ctx->S, ctx->r, nullptr, ctx->r, -1, nullptr, 0, nullptr, 0);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  // CG1 keeps u in P[0] / P[1] (the peer-mapped buffers) and p in r: u_0 = z_0
  if (ctx->variant == 1) CK(cudaMemcpyAsync(ctx->P[0], ctx->r, cells * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return 0;
}

// after gather_all: the global init scalars, hist[0] = 1 (||r_0|| = ||b||)
int solve_init_end(pot3d_ctx *ctx) {
  cudaStream_t s = ctx->stream;
  if (ctx->nranks > 1) {
    k_init_finalize<<<1, 1, 0, s>>>(ctx->S, ctx->gathered, ctx->nranks, ctx->warm ? 1 : 0,
                                    ctx->warm ? ctx->hist : nullptr);
    CK(cudaGetLastError());
    ctx->n_launch++;
  }
  if (ctx->warm) {  // hist[0] = ||r_0|| / ||b|| was written by k_init_dots
    ctx->warm = false;
  } else if (ctx->hist) {
    double one = 1.0;
    CK(cudaMemcpyAsync(ctx->hist, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  }
  return 0;
}

// the status of a finished loop (identical on every rank / slab)
int loop_status(pot3d_ctx *ctx, pot3d_ctx *rep) {
  const Scalars hs = *ctx->hS;
  if (hs.check) {  // POT3D_CHECK builds only (the bits are never set otherwise)
    rep->err = "POT3D_CHECK: invariant violated (bits " + std::to_string(hs.check) +
               ": 1 pass store, 2 sweep store, 4 sweep slot reuse, 8 peer store, 16 mailbox order, 32 CG1 store)";
    return POT3D_ERR_STATE;
  }
  const Grid &G = ctx->G;
  cudaStream_t s = ctx->stream;
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
    rep->err = "PC2 sweep handoff protocol error (bounded wait expired)";
    return POT3D_ERR_CUDA;
  }
  if (hs.xfer_error || hs.status == -5) {
    rep->err = "peer-memory exchange: bounded wait expired (a rank stalled or diverged)";
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
    rep->err = "p.Ap <= 0: operator or preconditioner not positive definite (S:341)";
    return POT3D_ERR_INDEFINITE;
  }
  if (!hs.stop) {
    rep->err = "loop ended without the stop flag";
    return POT3D_ERR_STATE;
  }
  return 0;
}

// setup of the iteration, the device-driven loop (graphs of `unroll` predicated
// iterations owned by h; the stop flag of graph g is read back while graph g+1 is
// already queued), the status checks.  M[0]->hS holds the final scalars.
int solve_run(pot3d_ctx *h, std::vector<pot3d_ctx *> &M, double rtol, int64_t maxit) {
  pot3d_ctx *ctx = h;
  cudaStream_t s = h->stream;
  const bool batch = h->nrhs > 1;  // h: the batch leader, M: its k problems
  bool stale = false;
  if (batch)
    TRY(ensure_hist_batch(h, M, maxit, stale));
  else
    for (pot3d_ctx *m : M) TRY(ensure_hist(m, maxit, stale));
  if (stale) TRY(M.size() > 1 && !batch ? build_graph_group(h) : build_graph(h));  // graph captured the old hist
  if (!batch && M[0]->warm && (M.size() > 1 || M[0]->nranks > 1)) {
    // a warm start across ranks / slabs: the global ||b|| first, then x0's halo and r_0
    for (pot3d_ctx *m : M) TRY(solve_begin(m, rtol, maxit, 1));
    TRY(gather_all(M));
    for (pot3d_ctx *m : M) {
      k_init_finalize<<<1, 1, 0, m->stream>>>(m->S, m->gathered, m->nranks, 0, nullptr);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    TRY(halo_all(M, [](pot3d_ctx *m) { return m->x; }));
    for (pot3d_ctx *m : M) TRY(solve_begin(m, rtol, maxit, 2));
  } else {
    for (pot3d_ctx *m : M) TRY(solve_begin(m, rtol, maxit));
  }
  if (!batch && M.size() > 1 && M[0]->pc == 3) {  // loopback PC3: z0's steps phase by phase
    std::vector<std::vector<Step>> st;
    for (pot3d_ctx *m : M) st.push_back(poly_steps(m, 0, false));
    for (size_t q = 0; q < st[0].size(); q++)
      for (size_t k = 0; k < st.size(); k++) {
        int rc = st[k][q]();
        if (rc) {
          h->err = M[k]->err;
          return rc;
        }
      }
    for (pot3d_ctx *m : M) TRY(solve_begin(m, rtol, maxit, 3));
  }
  if (!batch && (M.size() > 1 || M[0]->nranks > 1)) TRY(gather_all(M));
  for (pot3d_ctx *m : M) TRY(solve_init_end(m));
  if (M[0]->variant == 1) {  // CG1: w_0 = A u_0, delta_0 -> alpha_0 (the same steps, phase by phase)
    std::vector<std::vector<Step>> st;
    for (pot3d_ctx *m : M) st.push_back(cg1_steps(m, 0, true));
    for (size_t q = 0; q < st[0].size(); q++)
      for (size_t k = 0; k < st.size(); k++) {
        int rc = st[k][q]();
        if (rc) {
          h->err = M[k]->err;
          return rc;
        }
      }
  }
  pot3d_ctx *m0 = M[0];
  // the stop flags: one scalar block, or the leader's k stacked blocks of a batch (the
  // loop runs until every right-hand side has stopped; a stopped one's blocks return)
  const int nS = batch ? h->nrhs : 1;
  PinnedScalars hs2;
  CK(cudaMallocHost(&hs2.p, 3 * nS * sizeof(Scalars)));
  auto all_stop = [nS](const Scalars *v) {
    for (int q = 0; q < nS; q++)
      if (!v[q].stop) return false;
    return true;
  };
  CK(cudaMemcpyAsync(hs2.p + 2 * nS, m0->S, nS * sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int64_t launched = 0;
  if (!all_stop(hs2.p + 2 * nS)) {
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    CK(cudaGraphLaunch(h->gexec, s));
    h->n_launch += h->graph_nodes;
    CK(cudaMemcpyAsync(hs2.p, m0->S, nS * sizeof(Scalars), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ev[0], s));
    launched++;
    int cur = 0;
    while (true) {
      const bool more = (launched * h->graph_unroll) < maxit + h->graph_unroll;
      if (more) {
        CK(cudaGraphLaunch(h->gexec, s));
        h->n_launch += h->graph_nodes;
        CK(cudaMemcpyAsync(hs2.p + (cur ^ 1) * nS, m0->S, nS * sizeof(Scalars), cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(ev[cur ^ 1], s));
        launched++;
      }
      CK(cudaEventSynchronize(ev[cur]));
      if (all_stop(hs2.p + cur * nS) || !more) break;
      cur ^= 1;
    }
    CK(cudaStreamSynchronize(s));
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  for (pot3d_ctx *m : M) {
    CK(cudaMemcpyAsync(m->hS, m->S, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  for (pot3d_ctx *m : M) {
    m->last_iters = m->hS->iter;
    TRY(loop_status(m, h));
  }
  return 0;
}

// one graph for a loopback group: step q of every slab before step q+1 of any
int build_graph_group(pot3d_ctx *h) {
  pot3d_ctx *ctx = h;
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  for (pot3d_ctx *m : h->slabs) m->n_enq = 0;
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  for (int u = 0; u < h->unroll && rc == 0; u++) {
    std::vector<std::vector<Step>> st;
    for (pot3d_ctx *m : h->slabs) st.push_back(iteration_steps(m, u & 1));
    for (size_t q = 0; q < st[0].size() && rc == 0; q++)
      for (size_t k = 0; k < st.size() && rc == 0; k++) {
        rc = st[k][q]();
        if (rc) h->err = h->slabs[k]->err;
      }
  }
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  if (rc) return rc;
  CK(e);
  CK(cudaGraphInstantiate(&h->gexec, g, 0));
  cudaGraphDestroy(g);
  h->graph_unroll = h->unroll;
  h->graph_nodes = 0;
  for (pot3d_ctx *m : h->slabs) h->graph_nodes += m->n_enq;
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
  if (!ctx->rhs.empty()) {  // batch: the leader's geometry, the batch's bytes and launches
    pot3d_info(ctx->rhs[0], info);
    info->bytes_per_iter *= (int64_t)ctx->rhs.size();
    info->device_bytes = (int64_t)ctx->dev_bytes;
    info->kernel_launches = 0;
    pot3d_info_t mi{};
    for (const pot3d_ctx *m : ctx->rhs) {
      pot3d_info(m, &mi);
      info->device_bytes += mi.device_bytes;
      info->kernel_launches += mi.kernel_launches;
    }
    info->nrhs = (int32_t)ctx->rhs.size();
    return 0;
  }
  if (!ctx->slabs.empty()) {  // loopback group: the whole grid on one device
    pot3d_info_t mi{};
    *info = pot3d_info_t{};
    info->i0 = 0;
    info->i1 = info->nr_loc = ctx->nr;
    info->br_shells = ctx->nr + 1;
    info->pc = ctx->pc;
    info->pc2_blocks_total = ctx->pc2_blocks * (int32_t)ctx->slabs.size();
    info->kernel_launches = ctx->n_launch;
    for (const pot3d_ctx *m : ctx->slabs) {
      pot3d_info(m, &mi);
      info->graph_kernels_per_iter += mi.graph_kernels_per_iter;
      info->bytes_per_iter += mi.bytes_per_iter;
      info->device_bytes += mi.device_bytes;
      info->kernel_launches += mi.kernel_launches;
    }
    info->device_bytes += (int64_t)ctx->dev_bytes;
    info->exchange = 3;  // peer-memory exchange between the slabs of one device
    info->chunks_a = ctx->slabs[0]->G.nchunks;
    info->chunks_b = ctx->slabs[0]->nchunks_b;
    info->nrhs = 1;
    return 0;
  }
  info->i0 = ctx->G.i0;
  info->i1 = ctx->G.i0 + ctx->G.nr_loc;
  info->nr_loc = ctx->G.nr_loc;
  info->br_shells = ctx->G.nr_loc + (ctx->rank == ctx->nranks - 1 ? 1 : 0);
  info->pc = ctx->pc;
  info->pc2_blocks_total = ctx->pc2_blocks * ctx->nranks;
  int64_t k = 2;
  if (ctx->variant == 1)
    k += ctx->nranks > 1 ? 1 : 0;  // CG1: update, dots (+ the finalisation across ranks)
  else if (ctx->nranks > 1)
    k += (ctx->xfer && ctx->pc == 1) ? 2 : 3;
  if (ctx->pc == 2 && ctx->pc2) k += pc2_kernels_per_apply(ctx->pc2) + (ctx->nranks > 1 ? 1 : 0);
  if (ctx->pc == 3) k += ctx->poly_m;
  info->graph_kernels_per_iter = k;
  // algorithmic bytes
  const int64_t cells = (int64_t)ctx->G.nr_loc * ctx->nt * ctx->np;
  // PC1: pass A 24 + pass B 24 (even) / 40 (odd) = 56 B/cell on average (A23)
  // CG1: update 48 (even) / 64 (odd) + dots 8 = 64 B/cell on average
  // PC3: passes 64 + Chebyshev 32 (init) + 48 per middle step + 40 (last) = 48 m + 40
  info->bytes_per_iter = (ctx->pc == 2 ? 120 : ctx->pc == 3 ? 48 * ctx->poly_m + 40
                                                            : (ctx->variant == 1 ? 64 : 56)) * cells;
  info->device_bytes = (int64_t)ctx->dev_bytes;
  info->kernel_launches = ctx->n_launch;
  info->exchange = ctx->nranks == 1 ? 0 : (ctx->xfer ? 2 : 1);
  info->chunks_a = ctx->G.nchunks;
  info->chunks_b = ctx->nchunks_b;
  info->nrhs = 1;
  return 0;
}

int pot3d_set_br0(pot3d_ctx *ctx, const double *br0) {
  if (!ctx || !br0) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {  // batch: k consecutive maps
    for (size_t q = 0; q < ctx->rhs.size(); q++) {
      int rc = pot3d_set_br0(ctx->rhs[q], br0 + q * (size_t)ctx->nt * ctx->np);
      if (rc) {
        ctx->err = ctx->rhs[q]->err;
        return rc;
      }
    }
    ctx->solved = false;
    return 0;
  }
  if (!ctx->slabs.empty()) {
    for (pot3d_ctx *m : ctx->slabs) {
      int rc = pot3d_set_br0(m, br0);
      if (rc) {
        ctx->err = m->err;
        return rc;
      }
    }
    ctx->solved = false;
    return 0;
  }
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
    k_transpose<<<grd, blk, 0, ctx->stream>>>(ctx->nt, 1, ctx->np, G.PK, G.PK, COFF, src, ctx->br_dev, 1,
                                              ctx->nt);
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

// batch member (setup_batch): its slices of the handle's stacked vectors and scalars
struct BatchSlot {
  double *x, *r, *P0, *P1, *z;  // z: PC2 / PC3 (M^-1 r, pass A's staged vector)
  double *pres, *pd0, *pd1, *px;  // PC3: the Chebyshev steps' res, d_0, d_1, z_k
  Scalars *S;
  int q, k;                     // problem q of k (the leader q = 0 sets up the batched sweeps)
};

static int setup_one(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                     const pot3d_runtime *rt, pot3d_ctx **out, bool member,
                     const BatchSlot *slot = nullptr) {
  if (!out) return POT3D_ERR_INVALID;
  *out = nullptr;
  pot3d_ctx *ctx = new pot3d_ctx();
  ctx->member = member;
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
  if (pc != POT3D_PC1 && pc != POT3D_PC2 && pc != POT3D_PC3) {
    ctx->err = "pc must be 1, 2 or 3";
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
    const char *ec = getenv("POT3D_CLUSTER");  // "JxK": clusters of J x K tiles for the fused passes
    if (ec && sscanf(ec, "%dx%d", &ctx->pcj, &ctx->pck) != 2) ctx->pcj = ctx->pck = 1;
    ctx->pcj = std::max(1, std::min(ctx->pcj, 8));
    ctx->pck = std::max(1, std::min(ctx->pck, 8 / ctx->pcj));
    const char *ea = getenv("POT3D_EDGE_IN_A");
    // loopback slabs: the separate edge-shell kernel (no spin on a sibling's blocks
    // inside one launch)
    ctx->edge_in_a = !(ea && atoi(ea) == 0) && !member;
  }
  pot3d_runtime R{};
  R.nranks = 1;
  R.device = -1;
  if (rt) R = *rt;
  ctx->rank = R.rank;
  ctx->nranks = R.nranks < 1 ? 1 : R.nranks;
  ctx->pc2_blocks = R.pc2_blocks < 1 ? 1 : R.pc2_blocks;
  ctx->variant = R.variant;
  ctx->poly_m = R.poly_degree > 0 ? R.poly_degree : 4;
  ctx->poly_ratio = R.poly_ratio > 0.0 ? R.poly_ratio : 100.0;
  if (pc == POT3D_PC3 && (R.variant != 0 || ctx->poly_m < 2 || ctx->poly_m > POLY_MMAX || !(ctx->poly_ratio > 1.0))) {
    ctx->err = "PC3 runs the standard PCG with 2 <= poly_degree <= 8, poly_ratio > 1";
    return fail(POT3D_ERR_INVALID);
  }
  if (ctx->variant != 0 && (ctx->variant != 1 || pc != POT3D_PC1)) {
    ctx->err = "variant must be 0 (PCG) or 1 (CG1, PC1 only)";
    return fail(POT3D_ERR_INVALID);
  }
  ctx->unroll = R.unroll > 0 ? (R.unroll + 1) / 2 * 2 : 32;
  ctx->ualloc = R.alloc;
  ctx->ufree = R.free;
  ctx->actx = R.alloc_ctx;
  if (ctx->rank < 0 || ctx->rank >= ctx->nranks) { ctx->err = "bad rank"; return fail(POT3D_ERR_INVALID); }
  if (ctx->nranks > 1 && !R.nccl_unique_id && !member) { ctx->err = "nccl_unique_id required for nranks > 1"; return fail(POT3D_ERR_INVALID); }
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

  if (ctx->nranks > 1 && !member) {
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
  G.ntk = (np + 1 + TK - 1) / TK;  // tiles of columns 64t-1 .. 64t+62 cover -1 .. np-1
  {
    // peer memory, PC1: pass A's first block row builds the edge shells only where a
    // plane has fewer tiles than the resident pass blocks; on larger planes the separate
    // edge-shell kernel is faster (large on 2 / 4 GPUs: 817.2 vs 805.0 / 1520.2 vs 1467.6
    // iters/s; the 38-shell slab of 8 GPUs +4.8 %; medium on 4 GPUs: 7133 vs 7711,
    // profiles/r02_edge_dispatch_n4.log) and needs no dispatch-order assumption (§8.2)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    if (!getenv("POT3D_EDGE_IN_A") && (long long)G.ntj * G.ntk >= (long long)sms * PASS_MINB) ctx->edge_in_a = false;
  }
  {
    const void *fa[2] = {(const void *)k_pass_a, (const void *)k_pass_a_probe};
    const void *fb[3] = {(const void *)k_pass_b_pc1_even, (const void *)k_pass_b_pc1_odd,
                         (const void *)k_pass_b_pc2};
    for (int q = 0; q < 3; q++) {
      if ((q < 2 && cudaFuncSetAttribute(fa[q], cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_A)) ||
          cudaFuncSetAttribute(fb[q], cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_B)) {
        ctx->err = "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed";
        return fail(POT3D_ERR_CUDA);
      }
    }
  }
  if (cudaFuncSetAttribute(k_poly_step, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_P) ||
      cudaFuncSetAttribute(k_poly_last, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_P) ||
      cudaFuncSetAttribute(k_cg1_update_even, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_C1) ||
      cudaFuncSetAttribute(k_cg1_update_odd, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_C1) ||
      cudaFuncSetAttribute(k_cg1_dots, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_C2)) {
    ctx->err = "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed (CG1)";
    return fail(POT3D_ERR_CUDA);
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
  if (slot) {
    ctx->x = slot->x;
    ctx->r = slot->r;
  } else {
    DA(ctx->x, cells); DA(ctx->r, cells);
  }
  {
    const char *xe = getenv("POT3D_XFER");
    ctx->xfer_want = member || (ctx->nranks > 1 && ctx->nranks <= MAXR && !(xe && atoi(xe) == 0));
  }
  if (ctx->xfer_want) {
    if ((rc = ipc_alloc(ctx, &ctx->P[0], cells)) || (rc = ipc_alloc(ctx, &ctx->P[1], cells)) ||
        (rc = ipc_alloc(ctx, &ctx->mail, 1)))
      return fail(rc);
    if (cudaMemsetAsync(ctx->mail, 0, sizeof(Mailbox), ctx->stream)) { ctx->err = "memset"; return fail(POT3D_ERR_CUDA); }
  } else if (slot) {
    ctx->P[0] = slot->P0;
    ctx->P[1] = slot->P1;
  } else {
    DA(ctx->P[0], cells); DA(ctx->P[1], cells);
  }
  if (slot && slot->z)
    ctx->z = slot->z;
  else if (pc == POT3D_PC2 || pc == POT3D_PC3)
    DA(ctx->z, cells);
  if (pc == POT3D_PC3) {
    if (slot) {
      ctx->p_res = slot->pres;
      ctx->p_d[0] = slot->pd0;
      ctx->p_d[1] = slot->pd1;
      ctx->p_x = slot->px;
    } else {
      DA(ctx->p_res, cells); DA(ctx->p_x, cells);
      if (ctx->xfer_want) {  // peer memory: the neighbours store d's halo straight into these
        if ((rc = ipc_alloc(ctx, &ctx->p_d[0], cells)) || (rc = ipc_alloc(ctx, &ctx->p_d[1], cells))) return fail(rc);
      } else {
        DA(ctx->p_d[0], cells); DA(ctx->p_d[1], cells);
      }
    }
    for (double *p : {ctx->p_res, ctx->p_d[0], ctx->p_d[1], ctx->p_x})
      if (cudaMemsetAsync(p, 0, cells * sizeof(double), ctx->stream)) { ctx->err = "memset"; return fail(POT3D_ERR_CUDA); }
    // Saad Alg. 12.1 coefficients on [a, b] = [2 / ratio, 2] (the oracle's arithmetic)
    const double b = 2.0, a = 2.0 / ctx->poly_ratio;
    const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma1 = theta / delta;
    double rho = 1.0 / sigma1;
    ctx->p_theta = theta;
    for (int k = 1; k < ctx->poly_m; k++) {
      const double rho_new = 1.0 / (2.0 * sigma1 - rho);
      ctx->p_c1[k] = rho_new * rho;
      ctx->p_c2[k] = 2.0 * rho_new / delta;
      rho = rho_new;
    }
  }
  DA(ctx->bshell, G.plane + 16); DA(ctx->br_dev, G.plane + 16); DA(ctx->mean2, 2);
  if (slot)
    ctx->S = slot->S;
  else
    DA(ctx->S, 1);
  Grid Gc = G;  // the fused passes' tile count (clusters pad it)
  Gc.cj = ctx->pcj;
  Gc.ck = ctx->pck;
  ctx->partials_len = 4 * (size_t)std::max<long long>(
      (long long)pass_tiles(Gc) * (std::max(G.nchunks, ctx->nchunks_b) + 3), 65536);
  DA(ctx->partials, ctx->partials_len);
  DA(ctx->local_sum, 4);
  DA(ctx->gathered, 4 * (size_t)ctx->nranks + 4);  // 2 (PCG) or 4 (CG1) doubles per rank
  if (ctx->variant == 1) DA(ctx->s_cg, cells);
  DA(ctx->poles, 2 * (size_t)G.nr_loc);
#undef DA
  for (void *p : {(void *)ctx->x, (void *)ctx->r, (void *)ctx->P[0], (void *)ctx->P[1]})
    if (cudaMemsetAsync(p, 0, cells * sizeof(double), ctx->stream)) { ctx->err = "memset"; return fail(POT3D_ERR_CUDA); }
  if (ctx->z) cudaMemsetAsync(ctx->z, 0, cells * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->bshell, 0, (G.plane + 16) * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->br_dev, 0, (G.plane + 16) * sizeof(double), ctx->stream);
  cudaMemsetAsync(ctx->S, 0, sizeof(Scalars), ctx->stream);
  if (cudaMallocHost(&ctx->hS, sizeof(Scalars)) != cudaSuccess) { ctx->err = "pinned alloc"; return fail(POT3D_ERR_CUDA); }

  if (ctx->nranks > 1 && !member) {
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
    rc = pc2_create(&ctx->pc2, G, ctx->pc2_blocks, lb.data(), ctx->ualloc, ctx->actx, ctx->stream,
                    slot && slot->q == 0 ? slot->k : 1);
    if (rc) { ctx->err = "pc2_create failed"; return fail(POT3D_ERR_OOM); }
    double minpiv = 0;
    rc = pc2_factor(ctx->pc2, ctx->M, ctx->stream, &minpiv);
    if (rc) { ctx->err = "pc2_factor failed"; return fail(POT3D_ERR_CUDA); }
    // breakdown on any rank -> every rank falls back
    int bad = (minpiv < 1e-300) ? 1 : 0;
    if (ctx->nranks > 1 && !member) {  // loopback groups agree in setup_group
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
    if (!member && !slot) rc2 = build_graph(ctx);  // loopback / batch: the group's graph
    if (rc2) return fail(rc2);
  }
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    ctx->err = std::string("setup: ") + cudaGetErrorString(cudaGetLastError());
    return fail(POT3D_ERR_CUDA);
  }
  *out = ctx;
  return 0;
}

// Loopback group (pot3d_runtime.loopback_slabs = k > 1, one device): k slab contexts
// (ranks 0..k-1 of the r-slab partition) whose peer tables hold the siblings'
// P arrays and mailboxes directly; every kernel of the peer-memory exchange runs as
// in a k-process job, ordered on one stream (build_graph_group).
static int setup_group(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                       const pot3d_runtime *rt, pot3d_ctx **out) {
  *out = nullptr;
  const int k = rt->loopback_slabs;
  pot3d_ctx *h = new pot3d_ctx();
  auto fail = [&](int rc) {
    g_setup_error = h->err;
    for (pot3d_ctx *m : h->slabs) pot3d_destroy(m);
    h->slabs.clear();
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    dfree_all(h);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return rc;
  };
  if (!grid || !br0) {
    h->err = "null argument";
    return fail(POT3D_ERR_INVALID);
  }
  if (rt->nranks > 1 || k > MAXR) {
    h->err = "loopback_slabs needs nranks == 1 and at most 16 slabs";
    return fail(POT3D_ERR_INVALID);
  }
  h->nr = grid->nr; h->nt = grid->nt; h->np = grid->np;
  h->bc = outer_bc;
  h->pc_req = h->pc = pc;
  h->pc2_blocks = rt->pc2_blocks < 1 ? 1 : rt->pc2_blocks;
  h->unroll = rt->unroll > 0 ? (rt->unroll + 1) / 2 * 2 : 32;
  h->ualloc = rt->alloc;
  h->ufree = rt->free;
  h->actx = rt->alloc_ctx;
  if (rt->device >= 0) h->device = rt->device; else cudaGetDevice(&h->device);
  if (cudaSetDevice(h->device) != cudaSuccess) { h->err = "cudaSetDevice failed"; return fail(POT3D_ERR_CUDA); }
  if (rt->cuda_stream) {
    h->stream = (cudaStream_t)rt->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamDefault) != cudaSuccess) {
      h->err = "stream creation failed";
      return fail(POT3D_ERR_CUDA);
    }
    h->own_stream = true;
  }
  for (int q = 0; q < k; q++) {
    pot3d_runtime R = *rt;
    R.rank = q;
    R.nranks = k;
    R.loopback_slabs = 0;
    R.nccl_unique_id = nullptr;
    R.cuda_stream = h->stream;
    R.device = h->device;
    pot3d_ctx *m = nullptr;
    int rc = setup_one(grid, br0, outer_bc, pc, &R, &m, true);
    if (rc) {
      h->err = "loopback slab " + std::to_string(q) + ": " + g_setup_error;
      return fail(rc);
    }
    h->slabs.push_back(m);
  }
  for (pot3d_ctx *m : h->slabs) m->group = &h->slabs;
  // PC2 breakdown on any slab -> every slab falls back to PC1
  bool fell = false;
  for (pot3d_ctx *m : h->slabs) fell = fell || m->pc != pc;
  for (pot3d_ctx *m : h->slabs) {
    if (fell && m->pc != POT3D_PC1) {
      m->pc = POT3D_PC1;
      if (int rc = make_maps(m)) { h->err = m->err; return fail(rc); }
    }
    // the peer table from the siblings' plain device pointers
    const int q = m->rank;
    PeerTab T{};
    T.rank = q;
    T.nranks = k;
    T.nr_lo = q > 0 ? h->slabs[q - 1]->G.nr_loc : 0;
    for (int r = 0; r < k; r++) T.mail[r] = h->slabs[r]->mail;
    for (int b = 0; b < 2; b++) {
      if (q > 0) T.p_lo[b] = h->slabs[q - 1]->P[b];
      if (q < k - 1) T.p_hi[b] = h->slabs[q + 1]->P[b];
      if (pc == POT3D_PC3) {
        if (q > 0) T.d_lo[b] = h->slabs[q - 1]->p_d[b];
        if (q < k - 1) T.d_hi[b] = h->slabs[q + 1]->p_d[b];
      }
    }
    if (int rc = dalloc(m, &m->peers, 1)) { h->err = m->err; return fail(rc); }
    if (cudaMemcpyAsync(m->peers, &T, sizeof(PeerTab), cudaMemcpyHostToDevice, h->stream) != cudaSuccess) {
      h->err = "peer table upload failed";
      return fail(POT3D_ERR_CUDA);
    }
    m->xfer = true;
  }
  h->pc = h->slabs[0]->pc;
  h->G = h->slabs[0]->G;  // tiling constants (chunks reported by pot3d_info)
  h->G.i0 = 0;
  h->G.nr_loc = h->nr;
  if (int rc = build_graph_group(h)) return fail(rc);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
    h->err = std::string("loopback setup: ") + cudaGetErrorString(cudaGetLastError());
    return fail(POT3D_ERR_CUDA);
  }
  *out = h;
  return 0;
}

// Multi-RHS batch (pot3d_runtime.nrhs = k > 1): k single-problem contexts on the
// handle's stream over one stacked allocation of x, r, p_0, p_1 and the scalars; the
// leader rhs[0] launches each fused pass once for all k (grid z = k).
static int setup_batch(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                       const pot3d_runtime *rt, pot3d_ctx **out) {
  *out = nullptr;
  const int k = rt->nrhs;
  pot3d_ctx *h = new pot3d_ctx();
  pot3d_ctx *ctx = h;
  auto fail = [&](int rc) {
    g_setup_error = h->err;
    for (pot3d_ctx *m : h->rhs) pot3d_destroy(m);
    h->rhs.clear();
    dfree_all(h);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return rc;
  };
  if (!grid || !br0 || !grid->r_faces || !grid->t_faces || !grid->p_faces || grid->nr < 2 || grid->nt < 2 ||
      grid->np < 2) {
    h->err = "null argument or cell counts < 2 (S:45)";
    return fail(POT3D_ERR_INVALID);
  }
  if (rt->nranks > 1 || rt->loopback_slabs > 1 || rt->variant != 0 || k > 65535) {
    h->err = "nrhs > 1 runs on one rank (no loopback slabs) with standard PCG, nrhs <= 65535";
    return fail(POT3D_ERR_INVALID);
  }
  h->nr = grid->nr;
  h->nt = grid->nt;
  h->np = grid->np;
  h->bc = outer_bc;
  h->pc = h->pc_req = pc;
  h->ualloc = rt->alloc;
  h->ufree = rt->free;
  h->actx = rt->alloc_ctx;
  if (rt->device >= 0)
    h->device = rt->device;
  else
    cudaGetDevice(&h->device);
  if (cudaSetDevice(h->device) != cudaSuccess) {
    h->err = "cudaSetDevice failed";
    return fail(POT3D_ERR_CUDA);
  }
  if (rt->cuda_stream) {
    h->stream = (cudaStream_t)rt->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamDefault) != cudaSuccess) {
      h->err = "cudaStreamCreate failed";
      return fail(POT3D_ERR_CUDA);
    }
    h->own_stream = true;
  }
  // the single-problem layout (setup_one): PK physical columns, nr + 2 planes
  const long long PK = round_up(h->np + COFF + 1, 16);
  const size_t cells = (size_t)(h->nr + 2) * h->nt * PK;
  double *X = nullptr, *R = nullptr, *P0 = nullptr, *P1 = nullptr, *Z = nullptr;
  double *PR = nullptr, *PD0 = nullptr, *PD1 = nullptr, *PX = nullptr;
  Scalars *S = nullptr;
  int rc = 0;
  if ((rc = dalloc(h, &X, cells * k)) || (rc = dalloc(h, &R, cells * k)) || (rc = dalloc(h, &P0, cells * k)) ||
      (rc = dalloc(h, &P1, cells * k)) || (rc = dalloc(h, &S, (size_t)k)) ||
      (pc >= POT3D_PC2 && (rc = dalloc(h, &Z, cells * k))) ||
      (pc == POT3D_PC3 && ((rc = dalloc(h, &PR, cells * k)) || (rc = dalloc(h, &PD0, cells * k)) ||
                           (rc = dalloc(h, &PD1, cells * k)) || (rc = dalloc(h, &PX, cells * k)))))
    return fail(rc);
  auto at = [&](double *base, int q) { return base ? base + q * cells : nullptr; };
  const size_t nmap = (size_t)h->nt * h->np;
  for (int q = 0; q < k; q++) {
    BatchSlot sl{at(X, q),  at(R, q),   at(P0, q),  at(P1, q), at(Z, q), at(PR, q),
                 at(PD0, q), at(PD1, q), at(PX, q), S + q,    q,        k};
    pot3d_runtime Rq = *rt;
    Rq.nrhs = 1;
    Rq.device = h->device;
    Rq.cuda_stream = h->stream;
    pot3d_ctx *m = nullptr;
    rc = setup_one(grid, br0 + q * nmap, outer_bc, pc, &Rq, &m, false, &sl);
    if (rc) {
      h->err = "RHS " + std::to_string(q) + ": " + g_setup_error;
      return fail(rc);
    }
    h->rhs.push_back(m);
  }
  pot3d_ctx *lead = h->rhs[0];
  lead->nrhs = k;
  lead->zpart_len = lead->partials_len;
  if ((rc = dalloc(lead, &lead->zpartials, lead->partials_len * k))) {
    h->err = lead->err;
    return fail(rc);
  }
  if ((rc = make_maps(lead)) || (rc = build_graph(lead))) {
    h->err = lead->err;
    return fail(rc);
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) {
    h->err = std::string("batch setup: ") + cudaGetErrorString(cudaGetLastError());
    return fail(POT3D_ERR_CUDA);
  }
  *out = h;
  return 0;
}

int pot3d_setup(const pot3d_grid *grid, const double *br0, int32_t outer_bc, int32_t pc,
                const pot3d_runtime *rt, pot3d_ctx **out) {
  if (!out) return POT3D_ERR_INVALID;
  if (rt && rt->nrhs > 1) return setup_batch(grid, br0, outer_bc, pc, rt, out);
  if (rt && rt->loopback_slabs > 1) return setup_group(grid, br0, outer_bc, pc, rt, out);
  return setup_one(grid, br0, outer_bc, pc, rt, out, false);
}

// after the loop: the deferred x update, the closed-wall gauge, the true residual, Phi
// to the user and the status (one problem: one context, or the slabs of a group)
static int finish_solve(pot3d_ctx *ctx, std::vector<pot3d_ctx *> &M, double *phi, int64_t *iters,
                        double *rel_residual, double *true_rel_residual) {
  const Scalars hs = *M[0]->hS;
  cudaStream_t s = ctx->stream;
  if (!(hs.bnorm > 0))  // b = 0 -> Phi = 0, also from a warm start's x0
    for (pot3d_ctx *m : M) CK(cudaMemsetAsync(m->x, 0, (size_t)(m->G.nr_loc + 2) * m->G.plane * sizeof(double), s));
  const int nbi = 148 * 4;
  for (pot3d_ctx *m : M) {
    // PC1 defers the x update of even iterations to the next (odd) pass B (A23): when the
    // last iteration K = iters - 1 was even, x += alpha_K p_K (p_K in P[1]) now
    if (m->pc == 1 && (hs.iter & 1)) {
      k_x_finish<<<148 * 8, 256, 0, s>>>(m->G, m->S, m->x, m->variant == 1 ? m->r : m->P[1]);
      CK(cudaGetLastError());
      m->n_launch++;
    }
  }
  // closed wall: zero volume-weighted-mean gauge (A8)
  if (ctx->bc == POT3D_CLOSED_WALL && hs.bnorm > 0) {
    for (pot3d_ctx *m : M) {
      k_gauge_sums<<<nbi, 256, 0, s>>>(m->G, m->M, m->m_vr, m->x, m->S, m->partials, m->local_sum);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    TRY(gather_all(M));
    for (pot3d_ctx *m : M) {
      k_gauge_shift<<<148 * 8, 256, 0, s>>>(m->G, m->x, m->gathered, m->nranks);
      CK(cudaGetLastError());
      m->n_launch++;
    }
  }
  TRY(halo_all(M, [](pot3d_ctx *m) { return m->x; }));
  if (true_rel_residual) {
    for (pot3d_ctx *m : M) {
      k_apply<<<nbi, 256, 0, s>>>(m->G, m->M, m->x, nullptr, m->bshell, m->G.i0 == 0 ? 0 : -1000, m->S,
                                  m->partials, m->local_sum);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    TRY(gather_all(M));
    const int nr_ = M[0]->nranks;
    std::vector<double> g(2 * nr_);
    CK(cudaMemcpyAsync(g.data(), M[0]->gathered, sizeof(double) * 2 * nr_, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    double t = 0.0;
    for (int rr = 0; rr < nr_; rr++) t += g[2 * rr];
    *true_rel_residual = hs.bnorm > 0 ? std::sqrt(t) / hs.bnorm : 0.0;
  }
  if (phi) TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->x + m->G.plane; }, phi));
  CK(cudaStreamSynchronize(s));
  if (iters) *iters = hs.iter;
  if (rel_residual) *rel_residual = hs.bnorm > 0 ? std::sqrt(hs.rr) / hs.bnorm : 0.0;
  ctx->last_iters = hs.iter;
  for (pot3d_ctx *m : M) {
    m->last_iters = hs.iter;
    m->solved = m->has_x = true;
  }
  ctx->solved = ctx->has_x = true;
  // a fallen-back solve that did not converge reports NOT_CONVERGED; the fallback
  // itself stays visible through pot3d_info().pc != the requested pc
  if (hs.status == 1) return POT3D_NOT_CONVERGED;
  return ctx->pc != ctx->pc_req ? POT3D_PC2_FELL_BACK : POT3D_OK;
}

// a batch: one loop for all k problems, then each finished as a single problem with its
// slice of the outputs; the status is the first error, else NOT_CONVERGED if any hit maxit
static int solve_batch(pot3d_ctx *h, double rtol, int64_t maxit, double *phi, int64_t *iters,
                       double *rel_residual, double *true_rel_residual) {
  pot3d_ctx *ctx = h;
  CK(cudaSetDevice(h->device));
  std::vector<pot3d_ctx *> &M = h->rhs;
  for (pot3d_ctx *m : M) m->solved = m->has_x = false;
  int rc = solve_run(M[0], M, rtol, maxit);
  if (rc < 0) {
    h->err = M[0]->err;
    return rc;
  }
  const long long ncell = (long long)h->nr * h->nt * h->np;
  int worst = POT3D_OK;
  for (size_t q = 0; q < M.size(); q++) {
    std::vector<pot3d_ctx *> one{M[q]};
    rc = finish_solve(M[q], one, phi ? phi + q * ncell : nullptr, iters ? iters + q : nullptr,
                      rel_residual ? rel_residual + q : nullptr,
                      true_rel_residual ? true_rel_residual + q : nullptr);
    if (rc < 0) {
      h->err = M[q]->err;
      return rc;
    }
    if (rc == POT3D_NOT_CONVERGED) worst = rc;
  }
  h->last_iters = M[0]->last_iters;
  h->solved = true;
  return worst;
}

int pot3d_solve(pot3d_ctx *ctx, double rtol, int64_t maxit, double *phi, int64_t *iters,
                double *rel_residual, double *true_rel_residual) {
  if (!ctx) return POT3D_ERR_INVALID;
  if (!(rtol >= 0.0) || maxit < 1) {
    ctx->err = "rtol must be >= 0 and maxit >= 1";
    return POT3D_ERR_INVALID;
  }
  if (!ctx->rhs.empty()) return solve_batch(ctx, rtol, maxit, phi, iters, rel_residual, true_rel_residual);
  CK(cudaSetDevice(ctx->device));
  std::vector<pot3d_ctx *> M = members(ctx);
  for (pot3d_ctx *m : M) m->solved = m->has_x = false;
  ctx->solved = ctx->has_x = false;
  int rc = solve_run(ctx, M, rtol, maxit);
  if (rc < 0) return rc;
  return finish_solve(ctx, M, phi, iters, rel_residual, true_rel_residual);
}

int pot3d_solve_from(pot3d_ctx *ctx, const double *x0, double rtol, int64_t maxit, double *phi, int64_t *iters,
                     double *rel_residual, double *true_rel_residual) {
  if (!ctx) return POT3D_ERR_INVALID;
  if (!(rtol >= 0.0) || maxit < 1) {
    ctx->err = "rtol must be >= 0 and maxit >= 1";
    return POT3D_ERR_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  // a batch: one x0 per problem; a loopback group: x0 is the whole grid; a rank: its slab
  std::vector<pot3d_ctx *> M = ctx->rhs.empty() ? members(ctx) : ctx->rhs;
  for (pot3d_ctx *m : M)
    if (!x0 && !m->has_x) {
      ctx->err = "pot3d_solve_from(x0 = NULL): no solution in the context (a diagnostic call since the last solve)";
      return POT3D_ERR_STATE;
    }
  if (x0 && !ctx->rhs.empty()) {
    const size_t ncell = (size_t)ctx->nr * ctx->nt * ctx->np;
    for (size_t q = 0; q < M.size(); q++) {
      std::vector<pot3d_ctx *> one{M[q]};
      int rc = cells_in(M[q], one, x0 + q * ncell, [](pot3d_ctx *c) { return c->x + c->G.plane; });
      if (rc) {
        ctx->err = M[q]->err;
        return rc;
      }
    }
  } else if (x0) {
    TRY(cells_in(ctx, M, x0, [](pot3d_ctx *c) { return c->x + c->G.plane; }));
  }
  for (pot3d_ctx *m : M) m->warm = true;
  int rc = pot3d_solve(ctx, rtol, maxit, phi, iters, rel_residual, true_rel_residual);
  for (pot3d_ctx *m : M) m->warm = false;
  return rc;
}

int64_t pot3d_history(pot3d_ctx *ctx, double *hist, int64_t len) {
  if (!ctx || !hist) return POT3D_ERR_INVALID;
  if (!ctx->slabs.empty()) ctx = ctx->slabs[0];  // every slab holds the same history
  if (!ctx->rhs.empty()) ctx = ctx->rhs[0];      // batch: the first problem's
  if (!ctx->hist) return POT3D_ERR_STATE;
  int64_t n = std::min<int64_t>(std::min<int64_t>(len, ctx->last_iters + 1), ctx->hist_len);
  if (cudaMemcpy(hist, ctx->hist, sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess) {
    ctx->err = "history copy failed";
    return POT3D_ERR_CUDA;
  }
  return n;
}

int pot3d_field(pot3d_ctx *ctx, double *br, double *bt, double *bp) {
  if (!ctx) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {  // batch: k consecutive fields of the single-problem layout
    const size_t nc = (size_t)ctx->nr * ctx->nt * ctx->np;
    const size_t nbr = (size_t)(ctx->nr + 1) * ctx->nt * ctx->np, nbt = (size_t)ctx->nr * (ctx->nt + 1) * ctx->np;
    for (size_t q = 0; q < ctx->rhs.size(); q++) {
      int rc = pot3d_field(ctx->rhs[q], br ? br + q * nbr : nullptr, bt ? bt + q * nbt : nullptr,
                           bp ? bp + q * nc : nullptr);
      if (rc) {
        ctx->err = ctx->rhs[q]->err;
        return rc;
      }
    }
    return 0;
  }
  if (!ctx->solved) {
    ctx->err = "pot3d_field before a successful pot3d_solve";
    return POT3D_ERR_STATE;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  std::vector<pot3d_ctx *> M = members(ctx);
  const int ntf = ctx->nt + 1;
  auto nbr_of = [](pot3d_ctx *m) { return m->G.nr_loc + (m->rank == m->nranks - 1 ? 1 : 0); };
  for (pot3d_ctx *m : M) {
    const Grid &G = m->G;
    // temporaries: reuse the Krylov buffers (x keeps the solution); Bt needs
    // nr_loc * (nt+1) * PK <= (nr_loc+2) * nt * PK
    if ((long long)G.nr_loc * ntf > (long long)(G.nr_loc + 2) * m->nt) {
      ctx->err = "field buffer too small";
      return POT3D_ERR_STATE;
    }
    k_pole_avg<<<dim3(G.nr_loc, 2), 256, 0, s>>>(G, m->x, m->m_dp, m->pf[m->np] - m->pf[0], m->poles,
                                                  m->poles + G.nr_loc);
    CK(cudaGetLastError());
    m->n_launch++;
    FieldArgs F{};
    F.G = G;
    F.x = m->x;
    F.br = m->br_dev;
    F.mean2 = m->bc == POT3D_CLOSED_WALL ? m->mean2 : nullptr;
    F.rc = m->m_rc; F.dr = m->m_dr; F.drh = m->m_drh; F.tc = m->m_tc; F.tf = m->d_tf;
    F.dth = m->m_dth; F.st = m->m_st; F.dph = m->m_dph;
    F.poleN = m->poles; F.poleS = m->poles + G.nr_loc;
    F.bc = m->bc;
    F.nbr = nbr_of(m);
    F.Br = m->P[0]; F.Bt = m->P[1]; F.Bp = m->r;
    const long long nc = (long long)G.nr_loc * m->nt * m->np;
    if (br) {
      long long n = (long long)F.nbr * m->nt * m->np;
      k_field_r<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(F);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    if (bt) {
      long long n = (long long)G.nr_loc * ntf * m->np;
      k_field_t<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(F);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    if (bp) {
      k_field_p<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(F);
      CK(cudaGetLastError());
      m->n_launch++;
    }
  }
  if (br) TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->P[0]; }, br, ctx->nt, 0, 0, nbr_of));
  if (bt)
    TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->P[1]; }, bt, ntf,
                  (long long)ntf * M[0]->G.PK, 0));
  if (bp) TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->r; }, bp, ctx->nt, 0, 0));
  CK(cudaStreamSynchronize(s));
  // the Krylov buffers were reused: a later field call needs a new solve's x only
  return 0;
}

int pot3d_apply_fused(pot3d_ctx *ctx, const double *x, double *y, int32_t which) {
  if (!ctx || !x || !y || which < 0 || which > 2) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {
    ctx->err = "diagnostic applies run on single-problem contexts (not a batch)";
    return POT3D_ERR_INVALID;
  }
  if (which == 1 && ctx->pc != POT3D_PC1) {
    ctx->err = "pot3d_apply_fused(which=1) needs a PC1 context";
    return POT3D_ERR_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  std::vector<pot3d_ctx *> M = members(ctx);
  // the production passes with scalars that turn them into plain applies (parity 0:
  // pass A reads p_{k-1} from P[0] and writes p_k to P[1]; pass B reads p_k from P[1])
  auto src_of = [](pot3d_ctx *m) { return m->pc >= 2 ? m->z : m->r; };
  auto fix_cols = [&](pot3d_ctx *m, double *a) -> int {
    const Grid &G = m->G;
    k_fix_ghost_cols<<<(unsigned)((G.nr_loc * (long long)m->nt + 255) / 256), 256, 0, s>>>(G, a, 0, G.nr_loc);
    CK(cudaGetLastError());
    m->n_launch++;
    return 0;
  };
  Scalars h0{};
  h0.alpha = -1.0;  // pass B: r_out = r - alpha q = 0 + q (exact), x_out = 0 - p
  h0.beta = 0.0;    // pass A: p_k = src + 0 * p_{k-1} = x
  h0.rho = 1.0;
  h0.bnorm = 1.0;
  h0.maxit = 1;
  for (pot3d_ctx *m : M) {
    const size_t cells = (size_t)(m->G.nr_loc + 2) * m->G.plane;
    for (double *p : {m->x, m->r, m->P[0], m->P[1]}) CK(cudaMemsetAsync(p, 0, cells * sizeof(double), s));
    if (m->z) CK(cudaMemsetAsync(m->z, 0, cells * sizeof(double), s));
    CK(cudaMemcpyAsync(m->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
  }
  TRY(cells_in(ctx, M, x, [](pot3d_ctx *m) { return m->P[1] + m->G.plane; }));
  for (pot3d_ctx *m : M) TRY(fix_cols(m, m->P[1]));
  TRY(halo_all(M, [](pot3d_ctx *m) { return m->P[1]; }));  // ghost shells: the neighbours' edge shells
  if (which == 2) {
    TRY(cells_in(ctx, M, x, [&](pot3d_ctx *m) { return src_of(m) + m->G.plane; }));
    for (pot3d_ctx *m : M) TRY(fix_cols(m, src_of(m)));
  }
  for (pot3d_ctx *m : M) {
    const Grid &G = m->G;
    PassArgs a = make_args(m, 0);
    a.finalize = 0;  // the partials only reach local_sum; the scalars are not touched
    a.hist = nullptr;
    if (which == 2) {
      a.q_probe = m->x;
      CK(launch_pass(false, k_pass_a_probe, dim3(0, G.nchunks), SMEM_A, s, m->tmaps, a, 0));
    } else {
      a.G.nchunks = m->nchunks_b;
      CK(launch_pass(false, which == 0 ? k_pass_b_pc2 : k_pass_b_pc1_even, dim3(0, m->nchunks_b), SMEM_B, s,
                     m->tmaps, a, 0));
    }
    m->n_launch++;
    m->solved = m->has_x = false;
  }
  if (which == 2)
    TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->x + m->G.plane; }, y));
  else
    TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->r + m->G.plane; }, y));
  CK(cudaStreamSynchronize(s));
  ctx->solved = ctx->has_x = false;
  return 0;
}

int pot3d_apply(pot3d_ctx *ctx, const double *x, double *y) { return pot3d_apply_fused(ctx, x, y, 0); }

int pot3d_precond(pot3d_ctx *ctx, const double *rin, double *zout) {
  if (!ctx || !rin || !zout) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {
    ctx->err = "diagnostic applies run on single-problem contexts (not a batch)";
    return POT3D_ERR_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  std::vector<pot3d_ctx *> M = members(ctx);
  for (pot3d_ctx *m : M) {
    const size_t cells = (size_t)(m->G.nr_loc + 2) * m->G.plane;
    CK(cudaMemsetAsync(m->P[0], 0, cells * sizeof(double), s));
    CK(cudaMemsetAsync(m->P[1], 0, cells * sizeof(double), s));
  }
  TRY(cells_in(ctx, M, rin, [](pot3d_ctx *m) { return m->P[0] + m->G.plane; }));
  for (pot3d_ctx *m : M) {
    if (m->pc == 2) {
      int nk = pc2_apply(m->pc2, m->M, m->S, m->P[0], m->P[1], m->partials, 0, m->local_sum, s, false);
      TRY(nk);
      CK(cudaGetLastError());
      m->n_launch += nk;
    } else if (m->pc == 3) {  // the Chebyshev steps read r and write z (their TMA maps)
      const size_t bytes = (size_t)(m->G.nr_loc + 2) * m->G.plane * sizeof(double);
      Scalars h0{};
      CK(cudaMemcpyAsync(m->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(m->r, m->P[0], bytes, cudaMemcpyDeviceToDevice, s));
      TRY(poly_apply(m, 0, false));
      CK(cudaMemcpyAsync(m->P[1], m->z, bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      // PC1: the kernel that forms z_0 = D^-1 b at the start of a solve (mode -1)
      Scalars h0{};
      CK(cudaMemcpyAsync(m->S, &h0, sizeof(Scalars), cudaMemcpyHostToDevice, s));
      k_edge_p<<<148 * 8, 256, 0, s>>>(m->G, m->M, m->S, m->P[0], nullptr, m->P[1], -1, nullptr, 0, nullptr, 0);
      CK(cudaGetLastError());
      m->n_launch++;
    }
    m->solved = m->has_x = false;
  }
  TRY(cells_out(ctx, M, [](pot3d_ctx *m) { return (const double *)m->P[1] + m->G.plane; }, zout));
  CK(cudaStreamSynchronize(s));
  ctx->solved = ctx->has_x = false;
  return 0;
}

int pot3d_profile(pot3d_ctx *ctx, int32_t iters, double *ms_pass_a, double *ms_pass_b,
                  double *ms_precond) {
  if (!ctx || iters < 1) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {  // batch: the leader's launches over all k problems
    pot3d_ctx *lead = ctx->rhs[0];
    int rc = pot3d_profile(lead, iters, ms_pass_a, ms_pass_b, ms_precond);
    if (rc) ctx->err = lead->err;
    for (pot3d_ctx *m : ctx->rhs) m->solved = m->has_x = false;
    ctx->solved = ctx->has_x = false;
    return rc;
  }
  if (!ctx->slabs.empty() || ctx->variant != 0) {
    ctx->err = "profiling runs the standard PCG passes of one slab context (not a loopback group, not CG1)";
    return POT3D_ERR_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const Grid &G = ctx->G;
  // continue the recurrences of the current state without a stopping test (a batch
  // leader: all k scalar blocks, on the first problem's iteration parity)
  const int nS = ctx->nrhs;
  std::vector<Scalars> hv(nS);
  CK(cudaMemcpyAsync(hv.data(), ctx->S, nS * sizeof(Scalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long it0 = hv[0].iter;
  for (Scalars &v : hv) {
    v.stop = 0;
    v.status = 0;
    v.rtol = 0.0;
    v.iter = it0;
    v.maxit = it0 + iters + 1;
    if (!(v.rho != 0.0)) v.rho = 1.0;
    if (!(v.bnorm > 0.0)) v.bnorm = 1.0;
  }
  const Scalars h = hv[0];
  CK(cudaMemcpyAsync(ctx->S, hv.data(), nS * sizeof(Scalars), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t ev[4];
  for (auto &e : ev) CK(cudaEventCreate(&e));
  double ta = 0, tb = 0, tp = 0;
  const bool pc2 = ctx->pc == 2;
  dim3 grd(G.ntj * G.ntk, G.nchunks, nS);
  for (int it = 0; it < iters; it++) {
    const int par = (int)((h.iter + it) & 1);
    PassArgs a = make_args(ctx, par);
    a.hist = nullptr;
    a.finalize = 1;
    CK(cudaEventRecord(ev[0], s));
    CK(launch_pass(false, kern_a(ctx), grd, SMEM_A, s, ctx->tmaps, a, par));
    CK(cudaEventRecord(ev[1], s));
    PassArgs ab = a;
    ab.G.nchunks = ctx->nchunks_b;
    dim3 grdb(G.ntj * G.ntk, ctx->nchunks_b, nS);
    CK(launch_pass(false, kern_b(ctx, par), grdb, SMEM_B, s, ctx->tmaps, ab, par));
    CK(cudaEventRecord(ev[2], s));
    ctx->n_launch += 2;
    if (ctx->pc == 3) {
      TRY(poly_apply(ctx, 1, false, nS));
    }
    if (pc2) {
      const long long vst = nS > 1 ? (long long)(G.nr_loc + 2) * G.plane : 0;
      int nk = pc2_apply(ctx->pc2, ctx->M, ctx->S, ctx->r, ctx->z, nS > 1 ? ctx->zpartials : ctx->partials, 1,
                         ctx->local_sum, s, true, nullptr, nS, vst, (long long)ctx->zpart_len);
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
  ctx->solved = ctx->has_x = false;
  return 0;
}

int pot3d_profile_iteration(pot3d_ctx *ctx, int32_t iters, double *ms, char *names, int32_t nmax) {
  if (!ctx || iters < 1 || !ms || !names || nmax < 1) return POT3D_ERR_INVALID;
  if (!ctx->rhs.empty()) {
    ctx->err = "diagnostic applies run on single-problem contexts (not a batch)";
    return POT3D_ERR_INVALID;
  }
  if (!ctx->slabs.empty() || ctx->variant != 0) {
    ctx->err = "profiling runs the standard PCG passes of one slab context (not a loopback group, not CG1)";
    return POT3D_ERR_INVALID;
  }
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
  // the profiled iterations continue past the last solve's history buffer: record
  // no history (hist[iter+1 ..] would land beyond the allocation)
  struct HistOff {
    pot3d_ctx *c;
    double *h;
    ~HistOff() { c->hist = h; }
  } hist_off{ctx, ctx->hist};
  ctx->hist = nullptr;
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
  ctx->solved = ctx->has_x = false;
  return n;
}

int pot3d_trace_enable(pot3d_ctx *ctx, int32_t on) {
  if (!ctx) return POT3D_ERR_INVALID;
  for (pot3d_ctx *m : ctx->slabs) m->trace_on = on != 0;
  for (pot3d_ctx *m : ctx->rhs) m->trace_on = on != 0;
  ctx->trace_on = on != 0;
  return 0;
}

int pot3d_kernel_times(pot3d_ctx *ctx, double *us_pass_a, double *us_pass_b, int32_t *n) {
  if (!ctx || !us_pass_a || !us_pass_b || !n) return POT3D_ERR_INVALID;
  if (!ctx->slabs.empty()) ctx = ctx->slabs[0];
  if (!ctx->rhs.empty()) ctx = ctx->rhs[0];  // batch: the leader's launches
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

int pot3d_kernel_trace(pot3d_ctx *ctx, int64_t *iter, double *us_pass_a, double *us_pass_b, int32_t len) {
  if (!ctx || !iter || !us_pass_a || !us_pass_b || len < 1) return POT3D_ERR_INVALID;
  if (!ctx->slabs.empty()) ctx = ctx->slabs[0];
  if (!ctx->rhs.empty()) ctx = ctx->rhs[0];
  if (!ctx->trace) {
    ctx->err = "tracing not enabled (pot3d_trace_enable before pot3d_solve)";
    return POT3D_ERR_STATE;
  }
  CK(cudaSetDevice(ctx->device));
  std::vector<unsigned long long> t(64 * 16);
  CK(cudaMemcpy(t.data(), ctx->trace, t.size() * 8, cudaMemcpyDeviceToHost));
  // ring slot it holds iteration index it' with it' & 63 == it; recover it' from the
  // last iteration count (the ring keeps the last 64 iterations of the last solve)
  const int64_t last = ctx->last_iters;  // iterations 0 .. last-1 ran
  int n = 0;
  for (int64_t k = std::max<int64_t>(0, last - 64); k < last && n < len; k++) {
    const unsigned long long *r = &t[(k & 63) * 16];
    if (!r[TR_A0] || !r[TR_A1] || !r[TR_B0] || !r[TR_B1] || r[TR_A1] < r[TR_A0] || r[TR_B1] < r[TR_B0]) continue;
    iter[n] = k;
    us_pass_a[n] = (double)(r[TR_A1] - r[TR_A0]) / 1e3;
    us_pass_b[n] = (double)(r[TR_B1] - r[TR_B0]) / 1e3;
    n++;
  }
  return n;
}

int pot3d_destroy(pot3d_ctx *ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (pot3d_ctx *m : ctx->slabs) pot3d_destroy(m);
  ctx->slabs.clear();
  for (pot3d_ctx *m : ctx->rhs) pot3d_destroy(m);
  ctx->rhs.clear();
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
