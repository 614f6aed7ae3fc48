// pass_common.cuh -- tile geometry and per-cell helpers shared by the fused
// passes (passes.cu) and the single-reduction CG1 passes (cg1.cu): r-chunking,
// the lane -> column map of a theta-phi tile, the staged metric factors, the
// flux-form 7-point stencil (A1-A7) and the masked stores that keep the
// periodic ghost columns.
#pragma once
#include <type_traits>

#include "device_common.cuh"

namespace pot3d {

// The x update of the PC1 passes (reading A23).  XM_EVERY: x += alpha_k p_k.  PC1
// updates x every other iteration: XM_SKIP on even iterations k (x untouched); XM_PAIR
// on odd k: x += alpha_{k-1} p_{k-1} + alpha_k p_k with p_{k-1} = (p_k - z_k) / beta
// (beta the coefficient that built p_k from p_{k-1}) rebuilt from operands the pass
// holds anyway: x += (c + alpha_k) p_k - c z_k, c = alpha_{k-1} / beta.
enum XMode { XM_EVERY = 0, XM_SKIP = 1, XM_PAIR = 2 };

__device__ __forceinline__ void chunk_bounds(const Grid &G, int c, int &c0, int &c1) {
  if (G.part == 2) {  // the two edge shells
    c0 = (c == 0) ? 0 : G.nr_loc - 1;
    c1 = c0 + 1;
    return;
  }
  const int s0 = (G.part == 1) ? 1 : 0, n = (G.part == 1) ? G.nr_loc - 2 : G.nr_loc;
  int base = n / G.nchunks, rem = n % G.nchunks;
  c0 = s0 + c * base + (c < rem ? c : rem);
  c1 = c0 + base + (c < rem ? 1 : 0);
}

// Multi-RHS batches (pot3d_runtime.nrhs): blockIdx.z is the right-hand
// side.  Its vectors are stacked along the plane axis (each nr_loc + 2 planes, so one TMA
// descriptor covers the batch), its scalars are S[z], its partials and residual history
// PassArgs::pstride / hstride doubles further on.  Plane offset of this block's RHS:
__device__ __forceinline__ int rhs_planes(const Grid &G) { return (int)blockIdx.z * (G.nr_loc + 2); }

__device__ __forceinline__ int pass_bid(const Grid &G) {
  return G.blk_off + blockIdx.x + gridDim.x * blockIdx.y;
}
__device__ __forceinline__ int pass_nb(const Grid &G) {
  return G.blk_total > 0 ? G.blk_total : gridDim.x * gridDim.y;
}

// Column metric factors of the tile per smem index i (logical column k0-3+i,
// periodic): dp, app, apm.
struct TileConst {
  double dp[SROW], app[SROW], apm[SROW];
};

__device__ __forceinline__ void load_tile_const(TileConst &tc, const Grid &G, const Metrics &M,
                                                int k0) {
  for (int i = threadIdx.x; i < SROW; i += blockDim.x) {
    int k = k0 - 3 + i;
    k = (k < 0) ? k + G.np : k;
    k = (k >= G.np) ? (k - G.np) % G.np : k;
    tc.dp[i] = __ldg(M.dp + k);
    tc.app[i] = __ldg(M.app + k);
    tc.apm[i] = __ldg(M.apm + k);
  }
}

__device__ __forceinline__ int wrap_inc(int s, int n) { return (s + 1 == n) ? 0 : s + 1; }

// r-metric factors of the chunk's shells (c0-1 .. c1) staged in shared memory once
// per block, so the per-plane reads are shared-memory broadcasts instead of L2
// round trips on the plane loop's critical path (choose_chunks keeps every
// chunk within PLMAX-2 shells).
constexpr int PLMAX = POT3D_PLMAX;
struct PlaneSm {
  double arp[PLMAX], arm[PLMAX], dr[PLMAX], ss[PLMAX];
};
__device__ __forceinline__ void load_planes(PlaneSm &ps, const Metrics &M, int ig0, int n) {
  for (int q = threadIdx.x; q < n && q < PLMAX; q += blockDim.x) {
    ps.arp[q] = __ldg(M.arp + ig0 + q);
    ps.arm[q] = __ldg(M.arm + ig0 + q);
    ps.dr[q] = __ldg(M.dr + ig0 + q);
    ps.ss[q] = __ldg(M.ss + ig0 + q);
  }
}
// metrics of shell il = c0-1+q
__device__ __forceinline__ PlaneC plane_at(const PlaneSm &ps, int q) {
  PlaneC c;
  c.arp = ps.arp[q];
  c.arm = ps.arm[q];
  c.dr = ps.dr[q];
  c.ss = ps.ss[q];
  return c;
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

// stencil7 with the r flux shared between consecutive planes: Fu = arp (c - ip) is
// returned for the next plane, whose lower term arm (c - im) is exactly -Fu
// (arm_{i+1} == arp_i bitwise, a - b == -(b - a) exactly); Fd = arm (c - im).
__device__ __forceinline__ double stencil7f(double c, double ip, double Fd, double jp, double jm,
                                            double kp, double km, double dpk, double appk,
                                            double apmk, const PlaneC &P, const RowC &R, double &Fu) {
  Fu = P.arp * (c - ip);
  return dpk * (R.g * (Fu + Fd + P.ss * c) + P.dr * (R.atp * (c - jp) + R.atm * (c - jm))) +
         P.dr * R.q * (appk * (c - kp) + apmk * (c - km));
}

// The stencil with one theta face term tj and one phi face term tk already formed by
// the neighbouring cell of the same thread (FAST tiles, face_terms below): the other
// theta neighbour jo with coefficient ajo, the other phi neighbour ko with ako.
__device__ __forceinline__ double stencil7s(double c, double ip, double im, double tj, double ajo, double jo,
                                            double tk, double ako, double ko, double dpk, const PlaneC &P,
                                            const RowC &R) {
  return dpk * (R.g * (P.arp * (c - ip) + P.arm * (c - im) + P.ss * c) + P.dr * fma(ajo, c - jo, tj)) +
         P.dr * R.q * fma(ako, c - ko, tk);
}
// ... and with the r flux shared as in stencil7f
__device__ __forceinline__ double stencil7fs(double c, double ip, double Fd, double tj, double ajo, double jo,
                                             double tk, double ako, double ko, double dpk, const PlaneC &P,
                                             const RowC &R, double &Fu) {
  Fu = P.arp * (c - ip);
  return dpk * (R.g * (Fu + Fd + P.ss * c) + P.dr * fma(ajo, c - jo, tj)) + P.dr * R.q * fma(ako, c - ko, tk);
}

// A thread's 2 x 2 cells (rows e = 0, 1; columns x, y) share their inner faces: the theta
// face between the rows, atp_j (c_j - c_{j+1}), is -(atm_{j+1} (c_{j+1} - c_j)) exactly
// (atm_{j+1} == atp_j bitwise, k_metrics), and the phi face app_k (c_k - c_{k+1}) is
// -(apm_{k+1} (c_{k+1} - c_k)).  Valid on FAST tiles (every row and column an interior
// grid line away from the poles' halo rows and the periodic seam).
struct FaceTerms {
  double tx, ty;   // theta face between row 0 and row 1, columns x and y (row 0's view)
  double p0, p1;   // phi face between x and y, rows 0 and 1 (x's view)
};
__device__ __forceinline__ FaceTerms face_terms(double2 c0, double2 c1, const RowC &R0, double appx) {
  FaceTerms f;
  f.tx = R0.atp * (c0.x - c1.x);
  f.ty = R0.atp * (c0.y - c1.y);
  f.p0 = appx * (c0.x - c0.y);
  f.p1 = appx * (c1.x - c1.y);
  return f;
}

// Statically allocated shared state of a pass (declared once per kernel, so the
// FAST and general instantiations of a body share it).
struct PassShared {
  double sred[2 * NTHREADS / 32];
  TileConst tcs;
  PlaneSm pls;
};

// Per-thread geometry of a tile.
struct TileThread {
  int lane, w;
  int j0, k0, c0, c1;
  int row[RPW];          // haloed rows w*RPW + e (theta row j0-1+row)
  bool stencil[RPW];     // interior row inside the grid
  long long rowoff[RPW]; // j*PK + (k0-1+2*lane) + COFF, row clamped into the grid
  bool st0, st1;         // element 0/1 is an interior column of this tile inside the grid
  bool gr0, gr1, gl0, gl1;  // element 0/1 holds k = 0 (right-ghost dup) / k = np-1 (left ghost)
  bool valid;            // a tile of the grid (false: a cluster padding block, Grid::cj/ck)
};

__device__ __forceinline__ TileThread tile_thread(const Grid &G) {
  TileThread t;
  t.lane = threadIdx.x & 31;
  t.w = threadIdx.x >> 5;
  int tj, tk;
  tile_of(G, blockIdx.x, tj, tk);
  t.valid = (tj < G.ntj) && (tk < G.ntk);
  t.j0 = tj * TJ;
  t.k0 = tk * TK;
  // part 3: all shells, the two chunks touching a ghost shell scheduled last (their
  // blocks wait for the neighbours' halo, which meanwhile arrives in peer memory)
  int cy = blockIdx.y - G.role_rows;
  if (G.part == 3 && G.nchunks >= 3)
    cy = (cy < G.nchunks - 2) ? cy + 1 : (cy == G.nchunks - 2 ? 0 : G.nchunks - 1);
  chunk_bounds(G, cy, t.c0, t.c1);
  const int k = t.k0 - 1 + 2 * t.lane;  // logical column of element 0 (odd)
#pragma unroll
  for (int e = 0; e < RPW; e++) {
    const int r = RPW * t.w + e;
    const int j = t.j0 - 1 + r;
    const bool jv = (j >= 0) && (j < G.nt);
    t.row[e] = r;
    t.stencil[e] = (r >= 1) && (r <= TJ) && jv;
    t.rowoff[e] = (long long)(jv ? j : t.j0) * G.PK + k + COFF;
  }
  // every lane owns two cells of the tile's 64 columns k0-1 .. k0+62; only the first
  // tile (logical -1 = the ghost copy of np-1) and the last (columns >= np) mask some
  t.st0 = (k >= 0) && (k < G.np);
  t.st1 = (k + 1 < G.np);
  t.gr0 = t.st0 && (k == 0);
  t.gr1 = t.st1 && (k + 1 == 0);
  t.gl0 = t.st0 && (k == G.np - 1);
  t.gl1 = t.st1 && (k + 1 == G.np - 1);
  return t;
}

// A tile whose 64 columns k0-1 .. k0+62 are all interior cells away from the
// periodic seam (no masks, no ghost-column duplicates) and whose haloed rows are all
// grid rows: block-uniform, selects the FAST instantiation of the passes.
__device__ __forceinline__ bool tile_fast(const Grid &G) {
  int tj, tk;
  tile_of(G, blockIdx.x, tj, tk);
  const int k0 = tk * TK, j0 = tj * TJ;
  // every haloed row j0-1 .. j0+TJ a grid row too (the shared theta faces, face_terms)
  return tj < G.ntj && k0 >= TK && k0 + TK <= G.np && j0 >= 1 && j0 + TJ <= G.nt - 1;
}

// Store of a lane's column pair (interior elements only) with the periodic
// ghost-column duplicates; row_k points at the physical column of element 0.
template <bool FAST = false>
__device__ __forceinline__ void store_pair(double *row_k, const TileThread &t, int np, double2 v,
                                           bool streaming) {
  if (FAST || (t.st0 && t.st1)) {
    if (streaming)
      __stcs(reinterpret_cast<double2 *>(row_k), v);
    else
      *reinterpret_cast<double2 *>(row_k) = v;
  } else {
    if (t.st0) row_k[0] = v.x;
    if (t.st1) row_k[1] = v.y;
  }
  if (FAST) return;
  if (t.gr0) row_k[np] = v.x;        // k = 0 (element 0)    -> physical np+1
  if (t.gr1) row_k[np + 1] = v.y;    // k = 0 (element 1)    -> physical np+1
  if (t.gl0) row_k[-np] = v.x;       // k = np-1 (element 0) -> physical 0
  if (t.gl1) row_k[1 - np] = v.y;    // k = np-1 (element 1) -> physical 0
}

// A select the compiler cannot turn back into a branch (both operands are
// computed), so the transform of a plane stays in the step's basic block.
__device__ __forceinline__ double selp(double a, double b, bool p) {
  double r;
  asm("{.reg .pred q; setp.ne.s32 q, %3, 0; selp.f64 %0, %1, %2, q;}"
      : "=d"(r) : "d"(a), "d"(b), "r"((int)p));
  return r;
}
template <int V>
using IC = std::integral_constant<int, V>;

}  // namespace pot3d
