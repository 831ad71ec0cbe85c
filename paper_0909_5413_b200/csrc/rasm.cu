// rasm.cu -- restricted additive Schwarz preconditioner.
//
// M^-1 = sum_c R~_c^T A_c^-1 R_c  (Eq.(11)), one subdomain per non-empty
// cell c, Omega_c = the (2*rings+1)^2 block of cells around c (reading Q9),
// A_c = R_c A_rc R_c^T (reading Q10).
//
// Setup (PCSetUp; "only the small matrices A_i are formed"): one CTA
// per cell builds A_c in shared memory (packed lower triangle) in "factor order"
// (the block's other points first, own(c) last), factors it A_c = L L^T
// (P:310 uses a dense LU; Cholesky is the symmetric case of it, reading Q11) and
// forms only the rows of A_c^-1 that RASM keeps (R~_c, Eq.(9)):
//     A_c^-1[own, :] = S^-1 [-W, I],  W = L21 L11^-1,  S = L22 L22^T,
// which needs no storage beyond the factor itself.  The rows are written to HBM
// as X_c (n_own x n_ov, natural column order = the block's cells row-major).
//
// Apply (MatSolve, Eq.(10)): z[own(c)] = X_c u[Omega_c] -- a GEMV per
// cell that streams X once per GMRES iteration (HBM-bound).  Every output entry
// is written by exactly one cell (partition property): no atomics.
#include <cub/cub.cuh>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"

namespace rbf {

constexpr int kMaxRuns = 15;   // rings <= 7
constexpr int kRaThreads = 128;

struct Runs {
  int n;                 // number of runs (block rows inside the grid)
  int lo[kMaxRuns];      // global sorted start of each run
  int len[kMaxRuns];
  int n_ov, n_own, own_nat_lo;
  const int *list;       // box overlap: Omega_c's global indices (else null: the runs)
};

// The overlapping subdomain of cell (cx, cy): one contiguous run of the sorted
// arrays per block row (row-major keys).
__device__ __forceinline__ void block_runs(const Geom &g, const int *__restrict__ cell_start,
                                           int cx, int cy, Runs &R) {
  const int bx0 = max(cx - g.rings, 0), bx1 = min(cx + g.rings, g.ncx - 1);
  const int by0 = max(cy - g.rings, 0), by1 = min(cy + g.rings, g.ncy - 1);
  const int key = cy * g.ncx + cx;
  R.n = by1 - by0 + 1;
  R.n_ov = 0;
  R.own_nat_lo = 0;
  R.list = nullptr;
  for (int r = 0; r < R.n; ++r) {
    const int by = by0 + r;
    R.lo[r] = cell_start[by * g.ncx + bx0];
    R.len[r] = cell_start[by * g.ncx + bx1 + 1] - R.lo[r];
    if (by == cy) R.own_nat_lo = R.n_ov + (cell_start[key] - R.lo[r]);
    R.n_ov += R.len[r];
  }
  R.n_own = cell_start[key + 1] - cell_start[key];
}

// Omega_c of owned cell cl: the block's runs, or with box overlap its index list
__device__ __forceinline__ void sub_runs(const Geom &g, const int *__restrict__ cell_start,
                                         const OvList &ov, int cl, int cx, int cy, Runs &R) {
  block_runs(g, cell_start, cx, cy, R);
  if (ov.idx) {
    const long long o0 = ov.off[cl];
    R.list = ov.idx + o0;
    R.n_ov = (int)(ov.off[cl + 1] - o0);
    R.own_nat_lo = ov.own[cl];
  }
}

// Box-overlap membership (reading Q24): cell (cx, cy)'s box grown by g.ovw, closed;
// the edges are x0 + cx*c rounded twice (no contraction), exactly as in the oracle.
__device__ __forceinline__ bool in_grown_box(const Geom &g, double2 p, int cx, int cy) {
  return in_box(cell_box(g, cx, cy, g.ovw), p.x, p.y);
}

// MODE 0: |Omega_c| per owned cell (sizes[ncl] = 0 for the scan);  MODE 1: the lists.
template <int MODE>
__global__ void k_ov_lists(Geom g, Strip st, const double2 *__restrict__ xy,
                           const int *__restrict__ cell_start, int ncl, long long *__restrict__ sizes,
                           const long long *__restrict__ off, int *__restrict__ idx,
                           int *__restrict__ own) {
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl) {
    if (MODE == 0 && cl == ncl) sizes[cl] = 0;
    return;
  }
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  const int key = cy * g.ncx + cx;
  const int o0 = cell_start[key], o1 = cell_start[key + 1];
  if (o1 == o0) {  // no subdomain
    if (MODE == 0) sizes[cl] = 0;
    else own[cl] = 0;
    return;
  }
  Runs R;
  block_runs(g, cell_start, cx, cy, R);
  long long q = MODE == 1 ? off[cl] : 0;
  int cnt = 0, own_at = 0;
  for (int r = 0; r < R.n; ++r)
    for (int s = R.lo[r]; s < R.lo[r] + R.len[r]; ++s) {
      const bool mine = s >= o0 && s < o1;
      if (!mine && !in_grown_box(g, xy[s - st.ext_lo], cx, cy)) continue;
      if (s == o0) own_at = cnt;
      if (MODE == 1) idx[q + cnt] = s;
      ++cnt;
    }
  if (MODE == 0) sizes[cl] = cnt;
  else own[cl] = own_at;
}

__device__ __forceinline__ int nat_to_global(const Runs &R, int q) {
  if (R.list) return R.list[q];
  int r = 0;
  while (q >= R.len[r]) { q -= R.len[r]; ++r; }
  return R.lo[r] + q;
}

// ---------------------------------------------------------------------------
// Shared-memory tile layout of one subdomain matrix (tensor-core setup).
//
// Factor order: the block's other points [0, n0), padding to n0p = ceil8(n0), the
// cell's own points [n0p, n0p + n1), padding to N = n0p + n1p.  Padding unknowns
// are decoupled identity rows/columns, so they change nothing (their pivots are 1).
// The lower triangle is stored as 8x8 tiles, tile (it, jt) (jt <= it) at
// ((it (it+1))/2 + jt) * 64 doubles, row-major with an XOR swizzle of the column
// (c ^ 4*((r>>1)&1)) so that the DMMA fragment loads (8 rows x 4 columns) and the
// 16-byte accumulator stores are bank-conflict free.
// ---------------------------------------------------------------------------
constexpr int kTcThreads = 512;
constexpr int kTcWarps = kTcThreads / 32;
constexpr int kTcMaxTiles = 29;  // N <= 232: 435 tiles = 222,720 B of shared memory
constexpr size_t kTcMaxSmem = 227 * 1024 - 1024;  // dynamic shared memory (static part ~0.6 KB)

__device__ __forceinline__ int toff(int it, int jt) {  // it >= 0: the shift is the division
  return ((int)((unsigned)(it * (it + 1)) >> 1) + jt) * 64;
}
__device__ __forceinline__ int swz(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) << 2)); }

struct TileShape {
  int n, n0, n1, n0p, n1p, N, T, T0, T1;
  __host__ __device__ TileShape(int n_ov, int n_own) {
    n = n_ov;
    n1 = n_own;
    n0 = n_ov - n_own;
    n0p = (n0 + 7) & ~7;
    n1p = (n1 + 7) & ~7;
    N = n0p + n1p;
    T = N / 8;
    T0 = n0p / 8;
    T1 = n1p / 8;
  }
  // own(c) up to 64 points (8 tile rows): one W warp per own tile row (pairs up to 4 rows)
  __host__ __device__ bool fits_tc() const {
    return T <= kTcMaxTiles && n1p <= 64 && smem_bytes() <= kTcMaxSmem;
  }
  __host__ __device__ size_t smem_bytes() const {
    // tiles + rdiag + W partials + max(positions, the S^-1 phase's T1(T1-1)/2 M tiles + 1 scratch)
    const size_t mt = ((size_t)T1 * (T1 - 1) / 2 + 1) * 64 * 8;
    const size_t m = mt > 7 * 64 * 8 ? mt : 7 * 64 * 8;
    const size_t pos_or_m = (size_t)N * sizeof(double2) > m ? (size_t)N * sizeof(double2) : m;
    return ((size_t)T * (T + 1) / 2 * 64 + (size_t)T * 8 + 4 * 64) * 8 + pos_or_m;
  }
};

// D += A * B, one 8x8x4 fp64 tensor-core MMA (DMMA on sm_100a).
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Fragment offsets inside a swizzled tile (lane l): A[m][k] = X[m][k] and
// B[k][n] = X[n][k] use "rowk"; B[k][n] = X[k][n] and A[m][k] = X[k][m] use "colk".
__device__ __forceinline__ int frag_rowk(int lane, int h) { return swz(lane >> 2, 4 * h + (lane & 3)); }
__device__ __forceinline__ int frag_colk(int lane, int h) { return swz(4 * h + (lane & 3), lane >> 2); }
__device__ __forceinline__ int frag_acc(int lane) { return swz(lane >> 2, 2 * (lane & 3)); }

// factor index p -> global sorted index (or -1 for a padding unknown)
__device__ __forceinline__ int fac_to_global(const Runs &R, const TileShape &S, int p) {
  int q;
  if (p < S.n0) q = (p < R.own_nat_lo) ? p : p + S.n1;
  else if (p >= S.n0p && p < S.n0p + S.n1) q = R.own_nat_lo + (p - S.n0p);
  else return -1;
  return nat_to_global(R, q);
}

// natural column q -> factor index
__device__ __forceinline__ int nat_to_fac(const Runs &R, const TileShape &S, int q) {
  if (q < R.own_nat_lo) return q;
  if (q < R.own_nat_lo + S.n1) return S.n0p + (q - R.own_nat_lo);
  return q - S.n1;
}

// Per owned cell: X block size, maxima, and the list of cells that the tensor-core
// kernel cannot take (they go to the global-memory LU kernel).
// ASM (reading Q26): X holds all n_ov rows, every cell takes the LU path, and tsizes
// (non-null) receives n_ov per cell for the local-solution buffer.
__global__ void k_rasm_sizes(Geom g, Strip st, const int *__restrict__ cell_start, int ncl,
                             long long *__restrict__ sizes, int *__restrict__ maxes,
                             int *__restrict__ glist, OvList ov, long long *__restrict__ tsizes) {
  int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl) {
    if (cl == ncl) {
      sizes[cl] = 0;
      if (tsizes) tsizes[cl] = 0;
    }
    return;
  }
  int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  Runs R;
  sub_runs(g, cell_start, ov, cl, cx, cy, R);
  long long ld = (R.n_ov + 1) & ~1;
  const int rows = g.asm_full ? R.n_ov : R.n_own;
  sizes[cl] = R.n_own ? (long long)rows * ld : 0;
  if (tsizes) tsizes[cl] = R.n_own ? R.n_ov : 0;
  if (R.n_own) {
    atomicMax(&maxes[0], R.n_ov);
    atomicMax(&maxes[1], rows);
    atomicAdd(&maxes[2], 1);
    TileShape S(R.n_ov, R.n_own);
    if (g.asm_full || !S.fits_tc()) glist[atomicAdd(&maxes[3], 1)] = cl;
    else atomicMax(&maxes[4], (int)S.smem_bytes());
  }
}

// One CTA per cell.  Left-looking blocked Cholesky A_c = L L^T on 8x8 tiles with the
// products on the fp64 tensor cores (DMMA 8x8x4), software-pipelined so that the
// serial 8x8 diagonal factorization of column j (one warp) overlaps the
// accumulation of column j+1 (the other warps); then
//   W = L21 L11^-1 (backward tile sweep, one warp per own tile row),
//   S^-1 = (L22 L22^T)^-1 (the Schur complement's inverse, concurrently on the other warps),
//   X_c = S^-1 [-W, I]  (the rows of A_c^-1 for own(c), Eq.(9)-(11)),
// written to HBM in natural column order.
constexpr int kAccWarps = kTcWarps - 2;  // warps 14, 15 alternate as diagonal warps
constexpr int kWWarps = 12;              // W phase warps (the other four form S^-1)
constexpr int kWSlots = 9;               // W tiles per warp and row group: ceil(T0 / Q) <= 25 / 3

#ifdef RBF_PROBE
__device__ long long g_probe[64][8];
__device__ long long g_trace[65536][3];  // per CTA: smid, globaltimer at entry, at exit
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
__device__ long long g_col[2][64][4];  // per tile column of one interior CTA (see PCOL)
__device__ long long g_wcol[32][4];    // W phase of the same CTA: warp 0 per jt; [31] = warp 15
#define PW(jt, k) \
  if (lane == 0 && blockIdx.x == kColCta && (jt) < 32) g_wcol[jt][k] = clock64();
constexpr int kColCta = 20660;
#define PCOL(a, j, k) \
  if ((threadIdx.x & 31) == 0 && blockIdx.x == kColCta && (j) < 64) g_col[a][j][k] = clock64();
#define TRACE(i) \
  if (threadIdx.x == 0 && blockIdx.x < 65536) { g_trace[blockIdx.x][0] = smid(); g_trace[blockIdx.x][i] = gtimer(); }
// LU path phase clocks per CTA (persistent grid <= 296 CTAs): 0 assembly, 1 panel copy +
// factor, 2 panel write-back + L11, 3 U12 solve, 4 trailing update, 5 back substitution,
// 6 X copy-out; [7] cells, [8] sum of n
__device__ long long g_lu_acc[512][10];
__device__ long long g_lu_t[512];
// k_rasm_setup_tc2 phase clocks per CTA (warp 0 lane 0): 0 cells, 1 runs + positions,
// 2 Cholesky, 3 W + S^-1, 4 X
__device__ long long g_t2_acc[512][8];
__device__ long long g_t2_col[32][8];  // one interior cell of CTA 7: per column j (see T2C)
__device__ long long g_t2_w[32][8];    // the same cell's W phase: warp 0 per step jt
#define T2W(k)                                                                   \
  if (blockIdx.x == 7 && t2_cellno == 40 && (threadIdx.x & 31) == 0 && jt < 32) \
    g_t2_w[jt][k] = clock64();
#define T2C(k)                                                                  \
  if (blockIdx.x == 7 && t2_cellno == 40 && (threadIdx.x & 31) == 0 && j < 32) \
    g_t2_col[j][k] = clock64();
#define T2P(p)                                             \
  if (threadIdx.x == 0) {                                  \
    const long long t_ = clock64();                        \
    if ((p) > 0) g_t2_acc[blockIdx.x][p] += t_ - t2_last;  \
    t2_last = t_;                                          \
  }
#define LUP0() \
  if (threadIdx.x == 0) g_lu_t[blockIdx.x] = clock64();
#define LUP(p) \
  if (threadIdx.x == 0) { \
    const long long t_ = clock64(); \
    g_lu_acc[blockIdx.x][p] += t_ - g_lu_t[blockIdx.x]; \
    g_lu_t[blockIdx.x] = t_; \
  }
#define PROBE(i) /* 64 sampled CTAs spread over the grid (mostly interior cells) */ \
  if (threadIdx.x == 0 && blockIdx.x % 509 == 300 && blockIdx.x / 509 < 64) g_probe[blockIdx.x / 509][i] = clock64();
#else
#define LUP0()
#define LUP(p)
#define T2P(p) {}
#define T2C(k) {}
#define T2W(k) {}
#define PROBE(i)
#define TRACE(i)
#define PCOL(a, j, k) {}
#define PW(jt, k) {}
#endif

struct AccSet {
  double a0, a1, b0, b1;  // two independent DMMA chains (even / odd kt)
  double v0, v1;          // the tile's A_c entries at this lane's accumulator positions
  __device__ __forceinline__ void zero() { a0 = a1 = b0 = b1 = 0.0; }
};

// acc += sum_{kt in [k0, k1)} L(it, kt) L(jt, kt)^T
__device__ __forceinline__ void acc_range(AccSet &A, const double *sm, int it, int jt, int k0,
                                          int k1, int lane) {
  const double *Li = sm + toff(it, 0), *Lj = sm + toff(jt, 0);
  const int f0 = frag_rowk(lane, 0), f1 = frag_rowk(lane, 1);
  int kt = k0;
  for (; kt + 1 < k1; kt += 2) {
    dmma(A.a0, A.a1, Li[kt * 64 + f0], Lj[kt * 64 + f0]);
    dmma(A.b0, A.b1, Li[(kt + 1) * 64 + f0], Lj[(kt + 1) * 64 + f0]);
    dmma(A.a0, A.a1, Li[kt * 64 + f1], Lj[kt * 64 + f1]);
    dmma(A.b0, A.b1, Li[(kt + 1) * 64 + f1], Lj[(kt + 1) * 64 + f1]);
  }
  if (kt < k1) {
    dmma(A.a0, A.a1, Li[kt * 64 + f0], Lj[kt * 64 + f0]);
    dmma(A.a0, A.a1, Li[kt * 64 + f1], Lj[kt * 64 + f1]);
  }
}

// tile(it, jt) -= acc, in place (accumulator layout)
__device__ __forceinline__ void acc_finish_rmw(const AccSet &A, double *sm, int it, int jt, int lane) {
  double2 *cp = reinterpret_cast<double2 *>(sm + toff(it, jt) + frag_acc(lane));
  double2 cv = *cp;
  cv.x -= A.a0 + A.b0;
  cv.y -= A.a1 + A.b1;
  *cp = cv;
}

// C(it, jt) = A(it, jt) - acc, stored (accumulator layout)
__device__ __forceinline__ void acc_finish(const AccSet &A, double *sm, int it, int jt, int lane) {
  double2 *cp = reinterpret_cast<double2 *>(sm + toff(it, jt) + frag_acc(lane));
  *cp = make_double2(A.v0 - (A.a0 + A.b0), A.v1 - (A.a1 + A.b1));
}

// 8x8 Cholesky of the diagonal tile j in place (lanes 0..7 = rows) plus its inverse:
// lower part = L_d, upper part (r < c) = Linv[c][r], rdiag = 1 / diag(L_d).
__device__ __forceinline__ bool diag_factor_t(double *D, double *rdiag, int j, int lane) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = (lane < 8) ? D[swz(lane, c)] : 1.0;
  bool bad = false;
  double rinv = 1.0;  // 1 / L[lane][lane]
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    bad |= !(akk > 0.0);
    const double il = rsqrt(akk);  // 1 / l_kk
    const double lik = (lane == k) ? akk * il : a[k] * il;
    if (lane == k) rinv = il;
    a[k] = (lane >= k) ? lik : 0.0;
#pragma unroll
    for (int jj = k + 1; jj < 8; ++jj) {
      const double ljk = __shfl_sync(0xffffffffu, lik, jj);
      if (lane >= jj) a[jj] = fma(-lik, ljk, a[jj]);
    }
  }
  // Linv column `lane`: x = L^-1 e_lane by forward substitution
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double sacc = (lane == i) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) sacc = fma(-__shfl_sync(0xffffffffu, a[k], i), x[k], sacc);
    x[i] = sacc * __shfl_sync(0xffffffffu, rinv, i);
  }
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) D[swz(lane, c)] = (c <= lane) ? a[c] : x[c];
    rdiag[j * 8 + lane] = rinv;
  }
  return bad;
}
__device__ __forceinline__ bool diag_factor(double *sm, double *rdiag, int j, int lane) {
  return diag_factor_t(sm + toff(j, j), rdiag, j, lane);
}

// A_c = R_c A_rc R_c^T (reading Q10) entries of tile (it, jt) at this lane's
// accumulator positions (row lane>>2, columns 2(lane&3), +1), in factor order;
// padding unknowns are decoupled identity rows/columns.  Evaluated just in time
// (when the tile is finished), so the FP64 work of the assembly overlaps the
// latency-bound factorization instead of running as a separate phase.
__device__ __forceinline__ void a_entries(const double2 *pos, const TileShape &S, const Geom &g,
                                          int it, int jt, int lane, double &v0, double &v1) {
  const int r = lane >> 2, c0 = 2 * (lane & 3);
  const int pi = it * 8 + r;
  const bool padi = (pi >= S.n0 && pi < S.n0p) || pi >= S.n0p + S.n1;
  const double2 xi = pos[pi];
  double v[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int pj = jt * 8 + c0 + u;
    const bool padj = (pj >= S.n0 && pj < S.n0p) || pj >= S.n0p + S.n1;
    if (padi || padj) {
      v[u] = (pi == pj) ? 1.0 : 0.0;
    } else {
      const double2 xj = pos[pj];
      const double dx = xi.x - xj.x, dy = xi.y - xj.y;
      const double r2 = fma(dx, dx, dy * dy);
      v[u] = (r2 < g.rc2) ? exp_neg(r2 * g.neg_inv_2s2) * g.norm : 0.0;
    }
  }
  v0 = v[0];
  v1 = v[1];
}

// The phases after the factorisation: W = L21 L11^-1,
// S^-1 = L22^-T L22^-1, and X_c = S^-1 [-W, I] written to HBM.
__device__ __forceinline__ void setup_post(double *sm, double *rdiag, double2 *pos, const TileShape &S,
                                           const Runs &R, const Geom &g, double *__restrict__ X,
                                           const long long *__restrict__ x_off, int cl, int tid,
                                           int lane, int warp, int *s_fail) {
  const int T = S.T, T0 = S.T0, T1 = S.T1;
  (void)T;
  PROBE(2)
  // ---- W = L21 L11^-1 (warps 0..11) and S^-1 = L22^-T L22^-1 (warps 12..15), concurrently.
  //
  // W solves W L11 = L21 backwards over the tile columns of L11.  Right-looking: once
  // column kt of W is final, every own tile row r subtracts W(r,kt) L(kt,jt) from its
  // columns jt < kt (in place in the L21 tiles), so the work of a step is spread over
  // twelve warps and the chain from one column to the next is only the jt = kt-1 update
  // and that column's finish W(r,kt-1) = C(r,kt-1) L_d(kt-1)^-1, done first by the
  // owners of (r, kt-1), then one named barrier.  Tile (r, jt) belongs to warp
  // (r + T1 jt) mod 12: the T1 <= 8 rows of a column are on distinct warps.
  if (warp < kWWarps) {
    const int f0 = frag_rowk(lane, 0), f1 = frag_rowk(lane, 1);
    const int g0 = frag_colk(lane, 0), g1 = frag_colk(lane, 1);
    // W(r, jt) = C(r, jt) L_d(jt)^-1   (B[k][n] = Linv[k][n])
    auto finish = [&](int r, int jt) {
      double *Ct = sm + toff(T0 + r, jt);
      const double *D = sm + toff(jt, jt);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 4 * h + (lane & 3), n = lane >> 2;
        const double bv = (k > n) ? D[swz(n, k)] : (k == n ? rdiag[jt * 8 + k] : 0.0);
        dmma(d0, d1, Ct[frag_rowk(lane, h)], bv);
      }
      __syncwarp();
      *reinterpret_cast<double2 *>(Ct + frag_acc(lane)) = make_double2(d0, d1);
    };
    // Own tile rows in groups of up to four (rows are independent).  In a group of Tg
    // rows, Q = 12 / Tg column classes: warp w < Q Tg owns row rg + w % Tg and the
    // columns jt = q + Q s (q = w / Tg, slot s).  The contributions sum_{kt > jt}
    // W(r,kt) L(kt,jt) of its tiles accumulate in registers, one column kt per step
    // (the W(r,kt) fragments are loaded once per step for all slots), and a tile is
    // finished in the step after its last contribution: (C(r,jt) - acc) L_d(jt)^-1.
    for (int rg = 0; rg < T1; rg += 4) {
      const int Tg = T1 - rg < 4 ? T1 - rg : 4, Q = kWWarps / Tg;
      const bool active = warp < Q * Tg;
      const int r = rg + warp % Tg, q = warp / Tg;
      double acc0[kWSlots], acc1[kWSlots];
#pragma unroll
      for (int s = 0; s < kWSlots; ++s) acc0[s] = acc1[s] = 0.0;
      // the last column has no contributions
      if (active && T0 - 1 - q >= 0 && (T0 - 1 - q) % Q == 0) finish(r, T0 - 1);
      // d = kt - 1 - q (column kt-1 is slot d / Q when d % Q == 0), dm = d mod Q, s_lim =
      // slots with jt < kt - 1 = ceil(d / Q): kept incrementally (no division per step)
      int d = T0 - 2 - q, dm = d >= 0 ? d % Q : 0, s_lim = d > 0 ? (d + Q - 1) / Q : 0;
      for (int kt = T0 - 1; kt >= 1; --kt, --d) {
        if (warp == 0) PW(kt, 0)
        asm volatile("bar.sync 1, %0;" ::"n"(kWWarps * 32) : "memory");  // W(:, kt) final
        if (warp == 0) PW(kt, 1)
        if (active && d >= 0) {
          const double *Wt = sm + toff(T0 + r, kt), *Lrow = sm + toff(kt, 0);
          const double wa = Wt[f0], wb = Wt[f1];
          // the chain first: column kt-1's last contribution and its finish
          if (dm == 0) {
#pragma unroll
            for (int s = 0; s < kWSlots; ++s)
              if (s == s_lim) {
                const double *Lk = Lrow + (kt - 1) * 64;
                dmma(acc0[s], acc1[s], wa, Lk[g0]);
                dmma(acc0[s], acc1[s], wb, Lk[g1]);
                double2 *cp = reinterpret_cast<double2 *>(sm + toff(T0 + r, kt - 1) + frag_acc(lane));
                double2 cv = *cp;
                cv.x -= acc0[s];
                cv.y -= acc1[s];
                *cp = cv;
              }
            __syncwarp();
            finish(r, kt - 1);
          }
          if (warp == 0) PW(kt, 2)
          // the other tiles' contributions from column kt (jt < kt - 1)
#pragma unroll
          for (int s = 0; s < kWSlots; ++s)
            if (s < s_lim) {
              const double *Lk = Lrow + (q + Q * s) * 64;
              dmma(acc0[s], acc1[s], wa, Lk[g0]);
              dmma(acc0[s], acc1[s], wb, Lk[g1]);
            }
          if (warp == 0) PW(kt, 3)
          if (dm == 1 || (Q == 1 && d > 0)) --s_lim;  // ceil((d-1)/Q)
          dm = dm == 0 ? Q - 1 : dm - 1;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kWWarps * 32) : "memory");  // the group's W final
    }
  } else {
    if (warp == kWWarps) PW(31, 0)
    // S^-1 = L22^-T L22^-1 on tiles with the tensor cores, warps 12..15:
    //   M = L22^-1:  M(a,a) = L_a^-1 (already formed by the diagonal factorization),
    //                M(a,b) = -L_a^-1 sum_{k=b}^{a-1} L22(a,k) M(k,b),   a > b:
    //                the columns b of M are independent -- one warp per column;
    //   S^-1(a,b) = sum_{k>=a} M(k,a)^T M(k,b),   a >= b: tiles spread over the four
    //                warps, held in registers and written over L22 after a barrier (they
    //                read the L_a^-1 scratch of the diagonal tiles they overwrite).
    // M (strictly lower tiles) lives in the positions buffer (dead after the factorisation),
    // each warp's product scratch tile in the (former) W partials area.
    const int sw = warp - kWWarps;
    // L22: Cholesky of the Schur complement S (formed in place by all warps), right-looking
    // over the T1 own tile columns, while warps 0..11 run the W phase (which reads L11 and
    // L21 only)
    for (int a = 0; a < T1; ++a) {
      if (sw == 0 && diag_factor(sm, rdiag, T0 + a, lane) && lane == 0) *s_fail = 1;
      asm volatile("bar.sync 2, %0;" ::"n"((kTcWarps - kWWarps) * 32) : "memory");
      // panel L(T0+b, T0+a) = C L_d^-T, b > a
      const double *D = sm + toff(T0 + a, T0 + a);
      double bv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 4 * h + (lane & 3), n = lane >> 2;
        bv[h] = (n > k) ? D[swz(k, n)] : (n == k ? rdiag[(T0 + a) * 8 + k] : 0.0);
      }
      for (int b = a + 1 + sw; b < T1; b += kTcWarps - kWWarps) {
        double *Ct = sm + toff(T0 + b, T0 + a);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) dmma(d0, d1, Ct[frag_rowk(lane, h)], bv[h]);
        __syncwarp();
        *reinterpret_cast<double2 *>(Ct + frag_acc(lane)) = make_double2(d0, d1);
      }
      asm volatile("bar.sync 2, %0;" ::"n"((kTcWarps - kWWarps) * 32) : "memory");
      // trailing update C(T0+b, T0+c) -= L(T0+b, T0+a) L(T0+c, T0+a)^T, a < c <= b
      const int nr = T1 - 1 - a, nt = nr * (nr + 1) / 2;
      for (int t = sw; t < nt; t += kTcWarps - kWWarps) {
        int bb = 0;
        while ((bb + 1) * (bb + 2) / 2 <= t) ++bb;
        const int cc = t - bb * (bb + 1) / 2;
        AccSet A;
        A.zero();
        acc_range(A, sm, T0 + a + 1 + bb, T0 + a + 1 + cc, T0 + a, T0 + a + 1, lane);
        acc_finish_rmw(A, sm, T0 + a + 1 + bb, T0 + a + 1 + cc, lane);
      }
      asm volatile("bar.sync 2, %0;" ::"n"((kTcWarps - kWWarps) * 32) : "memory");
    }
    double *Mt = reinterpret_cast<double *>(pos);
    double *scr = rdiag + T * 8 + sw * 64;
    auto mt = [&](int a, int b) { return Mt + ((a * (a - 1)) / 2 + b) * 64; };  // a > b only
    const int m_ = lane >> 2, q_ = lane & 3;
    // Linv_a fragments: as A (A[m][k] = Linv[m][k]) or B (B[k][n] = Linv[k][n]); Linv[r][c]
    // (r > c) is stored at (c, r) of the diagonal tile, 1 / L_rr in rdiag.
    auto linvA = [&](int a, int h) -> double {
      const double *D = sm + toff(T0 + a, T0 + a);
      const int kk = 4 * h + q_;
      return (m_ > kk) ? D[swz(kk, m_)] : (m_ == kk ? rdiag[(T0 + a) * 8 + m_] : 0.0);
    };
    auto linvB = [&](int a, int h) -> double {
      const double *D = sm + toff(T0 + a, T0 + a);
      const int kk = 4 * h + q_;
      return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiag[(T0 + a) * 8 + kk] : 0.0);
    };
    auto linvT = [&](int a, int h) -> double {  // A[m][k] = Linv[k][m] (transposed)
      const double *D = sm + toff(T0 + a, T0 + a);
      const int kk = 4 * h + q_;
      return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiag[(T0 + a) * 8 + m_] : 0.0);
    };
    for (int b = sw; b < T1 - 1; b += kTcWarps - kWWarps) {
      for (int a = b + 1; a < T1; ++a) {
        double d0 = 0.0, d1 = 0.0;
        for (int k = b; k < a; ++k) {
          const double *La = sm + toff(T0 + a, T0 + k);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            dmma(d0, d1, La[frag_rowk(lane, h)], k == b ? linvB(b, h) : mt(k, b)[frag_colk(lane, h)]);
        }
        *reinterpret_cast<double2 *>(scr + frag_acc(lane)) = make_double2(d0, d1);
        __syncwarp();
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) dmma(e0, e1, linvA(a, h), scr[frag_colk(lane, h)]);
        __syncwarp();
        *reinterpret_cast<double2 *>(mt(a, b) + frag_acc(lane)) = make_double2(-e0, -e1);
        __syncwarp();
      }
    }
    asm volatile("bar.sync 2, %0;" ::"n"((kTcWarps - kWWarps) * 32) : "memory");  // M complete
    constexpr int kSlots = (8 * 9 / 2 + kTcWarps - kWWarps - 1) / (kTcWarps - kWWarps);
    double res[kSlots][2];
    const int ntl = T1 * (T1 + 1) / 2;
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int t = sw + sl * (kTcWarps - kWWarps);
      res[sl][0] = res[sl][1] = 0.0;
      if (t < ntl) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        const int bb = t - a * (a + 1) / 2;
        for (int k = a; k < T1; ++k) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double av = (k == a) ? linvT(a, h) : mt(k, a)[frag_colk(lane, h)];
            const double bv = (k == bb) ? linvB(bb, h) : mt(k, bb)[frag_colk(lane, h)];
            dmma(res[sl][0], res[sl][1], av, bv);
          }
        }
      }
    }
    asm volatile("bar.sync 2, %0;" ::"n"((kTcWarps - kWWarps) * 32) : "memory");  // L^-1 scratch read
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl) {
      const int t = sw + sl * (kTcWarps - kWWarps);
      if (t < ntl) {
        int a = 0;
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        const int bb = t - a * (a + 1) / 2;
        *reinterpret_cast<double2 *>(sm + toff(T0 + a, T0 + bb) + frag_acc(lane)) =
            make_double2(res[sl][0], res[sl][1]);
      }
    }
    if (warp == kWWarps) PW(31, 1)
  }
  __syncthreads();
}

__device__ __forceinline__ void setup_x(double *sm, double *rdiag, double2 *pos, const TileShape &S,
                                        const Runs &R, const Geom &g, double *__restrict__ X,
                                        const long long *__restrict__ x_off, int cl, int tid, int lane,
                                        int warp) {
  const int T0 = S.T0, T1 = S.T1;
  (void)rdiag;
  (void)pos;
  (void)g;
  PROBE(3)
  // ---- X_c = S^-1 [-W, I] in natural column order, ld = n rounded up to even, staged
  // in shared memory (the L11 tiles are dead) as the contiguous n_own x ld block and
  // written to HBM by one bulk copy (TMA), which drains while the next CTA starts (one
  // copy per row was measured no faster).
  // X_other = -S^-1 W straight from the DMMA accumulators; X_own = S^-1 (full tiles).
  const int n = S.n;
  const int ld = (n + 1) & ~1;
  // the staging block must lie inside the dead L11 tiles (the X loop still reads the W
  // and S^-1 tiles beyond them); else (small T0) the rows go straight to HBM
  const bool stage = (long long)S.n1 * ld <= (long long)toff(T0, 0);
  double *Xs = stage ? sm : X + x_off[cl];
  // the X_other tile (ot, jt) = -sum_kt S^-1(ot, kt) W(kt, jt)
  auto x_store = [&](int ot, int jt, double d0, double d1) {
    const int o = ot * 8 + (lane >> 2);
    const int p0 = jt * 8 + 2 * (lane & 3);
    // the X rows overlap tiles of L11 only (rows of factor order < T0): other warps
    // may still read W / S^-1 tiles, which lie beyond toff(T0, 0)
    if (o < S.n1) {
      if (p0 < S.n0) Xs[o * ld + (p0 < R.own_nat_lo ? p0 : p0 + S.n1)] = -d0;
      if (p0 + 1 < S.n0) Xs[o * ld + (p0 + 1 < R.own_nat_lo ? p0 + 1 : p0 + 1 + S.n1)] = -d1;
    }
  };
  // A = S^-1 tile (ot, kt): the lower tiles are stored, (ot, kt) above the diagonal is
  // the transpose of (kt, ot); diagonal tiles are full (symmetric)
  auto sinv_frag = [&](int ot, int kt, int h) -> double {
    const bool lower = kt <= ot;
    const double *At = lower ? sm + toff(T0 + ot, T0 + kt) : sm + toff(T0 + kt, T0 + ot);
    const int m = lane >> 2, k = 4 * h + (lane & 3);
    return lower ? At[swz(m, k)] : At[swz(k, m)];
  };
  if (T1 == 4) {
    // four warps per own tile row ot: the row's S^-1 fragments (4 tiles x 2 halves) are
    // loaded once and reused for the warp's columns jt = q, q + 4, ...; two DMMA chains
    const int ot = warp & 3, q = warp >> 2;
    double a[4][2];
#pragma unroll
    for (int kt = 0; kt < 4; ++kt)
#pragma unroll
      for (int h = 0; h < 2; ++h) a[kt][h] = sinv_frag(ot, kt, h);
    for (int jt = q; jt < T0; jt += 4) {
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int kt = 0; kt < 4; ++kt) {
        const double *Bt = sm + toff(T0 + kt, jt);
        if (kt & 1) {
          dmma(e0, e1, a[kt][0], Bt[frag_colk(lane, 0)]);
          dmma(e0, e1, a[kt][1], Bt[frag_colk(lane, 1)]);
        } else {
          dmma(d0, d1, a[kt][0], Bt[frag_colk(lane, 0)]);
          dmma(d0, d1, a[kt][1], Bt[frag_colk(lane, 1)]);
        }
      }
      x_store(ot, jt, d0 + e0, d1 + e1);
    }
  } else {
    for (int task = warp; task < T1 * T0; task += kTcWarps) {
      const int ot = task / T0, jt = task - ot * T0;
      double d0 = 0.0, d1 = 0.0;
      for (int kt = 0; kt < T1; ++kt) {
        const double *Bt = sm + toff(T0 + kt, jt);
#pragma unroll
        for (int h = 0; h < 2; ++h) dmma(d0, d1, sinv_frag(ot, kt, h), Bt[frag_colk(lane, h)]);
      }
      x_store(ot, jt, d0, d1);
    }
  }
  PROBE(5)
  for (int t = tid; t < S.n1 * S.n1; t += kTcThreads) {
    const int o = t / S.n1, j = t - o * S.n1;
    const int i1 = o >= j ? o : j, j1 = o >= j ? j : o;
    Xs[o * ld + R.own_nat_lo + j] = sm[toff(T0 + (i1 >> 3), T0 + (j1 >> 3)) + swz(i1 & 7, j1 & 7)];
  }
  if (ld != n)
    for (int o = tid; o < S.n1; o += kTcThreads) Xs[o * ld + n] = 0.0;
  if (!stage) {  // written straight to HBM
    PROBE(4)
    TRACE(2)
    return;
  }
  // generic-proxy shared-memory writes -> visible to the async (bulk copy) proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  PROBE(6)
  if (tid == 0) {
    const unsigned bytes = (unsigned)(S.n1 * ld * sizeof(double));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(X + x_off[cl]),
                 "r"((unsigned)__cvta_generic_to_shared(Xs)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read out: may exit
  }
  PROBE(4)
  TRACE(2)
}

__global__ __launch_bounds__(kTcThreads, 1) void k_rasm_setup_tc(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, int *__restrict__ counts,
    int *__restrict__ glist, OvList ov, const int *__restrict__ list) {
  TRACE(1)
  extern __shared__ __align__(16) double sm[];
  __shared__ Runs R;
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = list ? list[blockIdx.x] : blockIdx.x;  // list: the cells k_rasm_setup_tc2 left
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  if (tid == 0) {
    sub_runs(g, cell_start, ov, cl, cx, cy, R);
    s_fail = 0;
  }
  __syncthreads();
  if (R.n_own == 0) return;
  const TileShape S(R.n_ov, R.n_own);
  if (!S.fits_tc()) return;  // handled by k_rasm_setup_lu
  const int T = S.T, N = S.N;
  PROBE(0)
  double *rdiag = sm + T * (T + 1) / 2 * 64;
  double2 *pos = reinterpret_cast<double2 *>(rdiag + T * 8 + 4 * 64);  // after rdiag and wpart

  // ---- positions in factor order, then A_c = R_c A_rc R_c^T (reading Q10)
  for (int p = tid; p < N; p += kTcThreads) {
    const int gi = fac_to_global(R, S, p);
    pos[p] = (gi >= 0) ? xy[gi - st.ext_lo] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  __syncthreads();

  PROBE(1)
  // ---- software-pipelined left-looking Cholesky over tile columns
  AccSet acc[2];
  acc[0].zero();
  acc[1].zero();
  // A entries of the tiles finished in the first step (column 0)
  if (warp < kAccWarps) {
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int it = 1 + warp + kAccWarps * m;
      if (it < T) a_entries(pos, S, g, it, 0, lane, acc[m].v0, acc[m].v1);
    }
  } else if (warp == kAccWarps) {
    a_entries(pos, S, g, 0, 0, lane, acc[0].v0, acc[0].v1);
  }
  // the loop factors the columns of L11 (and L21); the Schur complement block L22 is
  // formed and factored after it (see below), concurrently with the W phase
  const int T0 = S.T0;
  for (int j = 0; j < T0; ++j) {
    const int dw = kAccWarps + (j & 1);  // diagonal warp of column j
    if (warp == 0) PCOL(0, j, 0)
    if (warp == dw) PCOL(1, j, 0)
    if (warp < kAccWarps) {
      // step 1: finish column j (tiles it > j) with the kt = j-1 term
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int it = j + 1 + warp + kAccWarps * m;
        if (it < T) {
          if (j >= 1) acc_range(acc[m], sm, it, j, j - 1, j, lane);
          acc_finish(acc[m], sm, it, j, lane);
        }
      }
      // step 2: accumulate column j+1 (tiles it > j+1) over kt < j
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int it = j + 2 + warp + kAccWarps * m;
        acc[m].zero();
        if (it < T && j + 1 < T0) {
          a_entries(pos, S, g, it, j + 1, lane, acc[m].v0, acc[m].v1);
          acc_range(acc[m], sm, it, j + 1, 0, j, lane);
        }
      }
    } else if (warp == dw) {
      // finish the diagonal tile (its sum over kt < j-1 was accumulated last step)
      if (j >= 1) acc_range(acc[0], sm, j, j, j - 1, j, lane);
      acc_finish(acc[0], sm, j, j, lane);
      __syncwarp();
      PCOL(1, j, 1)
      if (diag_factor(sm, rdiag, j, lane) && lane == 0) s_fail = 1;
      PCOL(1, j, 2)
    } else if (j + 1 < T0) {
      // the other diagonal warp accumulates the next diagonal tile over kt < j
      acc[0].zero();
      a_entries(pos, S, g, j + 1, j + 1, lane, acc[0].v0, acc[0].v1);
      acc_range(acc[0], sm, j + 1, j + 1, 0, j, lane);
    }
    if (warp == 0) PCOL(0, j, 1)
    __syncthreads();
    if (warp == 0) PCOL(0, j, 2)
    if (s_fail) break;  // uniform
    // step 4: panel L(it, j) = C(it, j) L_d^-T  (B[k][n] = Linv[n][k]; the B fragments
    // are loaded once per column)
    if (warp < kAccWarps && j + 1 + warp < T) {
      const double *D = sm + toff(j, j);
      double bv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 4 * h + (lane & 3), n = lane >> 2;
        bv[h] = (n > k) ? D[swz(k, n)] : (n == k ? rdiag[j * 8 + k] : 0.0);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int it = j + 1 + warp + kAccWarps * m;
        if (it < T) {
          double *Ct = sm + toff(it, j);
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) dmma(d0, d1, Ct[frag_rowk(lane, h)], bv[h]);
          __syncwarp();
          *reinterpret_cast<double2 *>(Ct + frag_acc(lane)) = make_double2(d0, d1);
        }
      }
    }
    __syncthreads();
    if (warp == 0) PCOL(0, j, 3)
  }
  if (s_fail) {  // Cholesky broke down: redo this cell with LU (reading Q11)
    if (tid == 0) glist[atomicAdd(&counts[3], 1)] = cl;
    return;
  }
  // ---- the Schur complement S = A22 - L21 L21^T on the own tile rows, all warps: tile
  // (T0 + a, T0 + b), b <= a, summed over the T0 columns of L21 (two DMMA chains)
  {
    const int T1 = S.T1;
    const int ntl = T1 * (T1 + 1) / 2;
    for (int t = warp; t < ntl; t += kTcWarps) {
      int a = 0;
      while ((a + 1) * (a + 2) / 2 <= t) ++a;
      const int b = t - a * (a + 1) / 2;
      AccSet A;
      A.zero();
      a_entries(pos, S, g, T0 + a, T0 + b, lane, A.v0, A.v1);
      acc_range(A, sm, T0 + a, T0 + b, 0, T0, lane);
      acc_finish(A, sm, T0 + a, T0 + b, lane);
    }
  }
  __syncthreads();

  setup_post(sm, rdiag, pos, S, R, g, X, x_off, cl, tid, lane, warp, &s_fail);
  if (s_fail) {  // the Schur complement's Cholesky broke down (LU, reading Q11)
    if (tid == 0) glist[atomicAdd(&counts[3], 1)] = cl;
    return;
  }
  setup_x(sm, rdiag, pos, S, R, g, X, x_off, cl, tid, lane, warp);
}

// ---------------------------------------------------------------------------
// Two factorisations per SM: k_rasm_setup_tc2 (same arithmetic as k_rasm_setup_tc).
//
// The one-CTA-per-SM kernel above holds the whole tile-packed factor (223 KB for
// n = 225) although the left-looking column loop only ever reads the rows at or
// below the current column: a row of L11 is final, and no longer read by the
// factorisation, once its own column has been formed.  Here each such row is
// copied to a per-CTA global workspace (L2-resident, column-major so that a
// column of L11 is contiguous) as soon as the loop is done with it, and its
// tiles' shared-memory slots are reused by the next columns.  The live set is
// then at most (T-1-j)(j+1) + 2 tiles at column j (212 tiles = 106 KB for T = 29
// instead of 435), so two CTAs of 8 warps fit on an SM and two subdomains are
// factored concurrently: one CTA's per-column barriers and serial 8x8 diagonal
// chain overlap the other CTA's tensor-core accumulations.
//
// Tile (it, jt) lives in slot slot[it(it+1)/2 + jt]; the slot plan (lowest free
// slot first, in the order the loop forms and retires tiles) is computed on the
// host per tile shape (T, T1) -- see t2_plan in rasm_setup -- together with the
// slots that are free after the factorisation (the W phase streams the columns
// of L11 back through them).  After the factorisation:
//   W = L21 L11^-1 by a backward sweep over the columns jt of L11 (one warp per own
//       tile row; column jt of L11 arrives by cp.async three columns ahead),
//   S^-1 = L22^-T L22^-1 concurrently on the other four warps (as above),
//   X_c = S^-1 [-W, I] written straight to HBM.
// Persistent: 2 CTAs per SM take the cells from an atomic counter.  Cells with
// more than 4 own tile rows (n_own > 32) are left to k_rasm_setup_tc (list).
// ---------------------------------------------------------------------------
constexpr int kT2Threads = 256;
constexpr int kT2Warps = kT2Threads / 32;
constexpr int kT2Acc = kT2Warps - 2;  // accumulate warps; the last two alternate as diagonal warps
constexpr int kT2M = (kTcMaxTiles - 1 + kT2Acc - 1) / kT2Acc;  // tiles per accumulate warp and column
constexpr int kT2MaxT1 = 4;           // own tile rows (n_own <= 32)
constexpr int kT2Cap = 212;           // tile slots: max_j (T-1-j)(j+1) + 2 at T = 29
constexpr int kT2Rec = 1024;          // bytes per (T, T1) plan record (see rbf::t2_plan)
constexpr int kT2RecFree = 512;       // record offset of the free-slot list
constexpr int kT2RecPeak = 1016;      // int: slots used; int at 1020: free slots after the factorisation
constexpr int kT2WsTiles = kTcMaxTiles * (kTcMaxTiles + 1) / 2;  // workspace tiles per CTA
constexpr size_t kT2Smem = (size_t)kT2Cap * 512 + kTcMaxTiles * 8 * sizeof(double) +
                           kTcMaxTiles * 8 * sizeof(double2) + 440;

__device__ __forceinline__ int t2_gcol(int kt, int T0) { return kt * T0 - ((kt * (kt - 1)) >> 1); }

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// Plan record of tile shape (T, T1): slot table, free list, peak (host-written).
__host__ __device__ inline int t2_rec_index(int T, int T1) { return T * (kT2MaxT1 + 1) + T1; }
constexpr int kT2Recs = (kTcMaxTiles + 1) * (kT2MaxT1 + 1);

// acc[m] += sum_{kt < j} L(it0 + kT2Acc m, kt) L(j+1, kt)^T for m < NM (one chain per row;
// the B fragments of row j+1 are shared by the NM rows)
template <int NM, int ACC = kT2Acc, int MM = kT2M>
__device__ __forceinline__ void t2_acc_rows(double (&acc)[MM][2], const double *sm, const unsigned char *slot,
                                            int j, int it0, int f0, int f1) {
  const unsigned char *sj = slot + (((j + 1) * (j + 2)) >> 1);
  const unsigned char *si[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int it = it0 + ACC * m;
    si[m] = slot + ((it * (it + 1)) >> 1);
  }
#pragma unroll 2
  for (int kt = 0; kt < j; ++kt) {
    const double *Bt = sm + (int)sj[kt] * 64;
    const double *At[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) At[m] = sm + (int)si[m][kt] * 64;
    const double b0 = Bt[f0], b1 = Bt[f1];
    double a0[NM], a1[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      a0[m] = At[m][f0];
      a1[m] = At[m][f1];
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) dmma(acc[m][0], acc[m][1], a0[m], b0);
#pragma unroll
    for (int m = 0; m < NM; ++m) dmma(acc[m][0], acc[m][1], a1[m], b1);
  }
}

__global__ __launch_bounds__(kT2Threads, 2) void k_rasm_setup_tc2(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, int *__restrict__ counts,
    int *__restrict__ glist, OvList ov, const unsigned char *__restrict__ plans, double *__restrict__ ws,
    int *__restrict__ work, int *__restrict__ deferred, int ncl) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Runs R;
  __shared__ int s_cl, s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *rdiag = sm + kT2Cap * 64;
  double2 *pos = reinterpret_cast<double2 *>(rdiag + kTcMaxTiles * 8);
  unsigned char *slot = reinterpret_cast<unsigned char *>(pos + kTcMaxTiles * 8);
  double *wsl = ws + (size_t)blockIdx.x * kT2WsTiles * 64;
  const int f0 = frag_rowk(lane, 0), f1 = frag_rowk(lane, 1);
#ifdef RBF_PROBE
  long long t2_last = 0;
  int t2_cellno = 0;
#endif
  for (;;) {
    __syncthreads();  // the previous cell is done with R and the shared tiles
    T2P(0)
    if (tid == 0) {
      const int cl = atomicAdd(work, 1);
      s_cl = cl;
      s_fail = 0;
      if (cl < ncl) sub_runs(g, cell_start, ov, cl, cl % g.ncx, st.row_lo + cl / g.ncx, R);
    }
    __syncthreads();
    const int cl = s_cl;
    if (cl >= ncl) return;
    if (R.n_own == 0) continue;
    const TileShape S(R.n_ov, R.n_own);
    if (!S.fits_tc()) continue;  // handled by k_rasm_setup_lu
    const unsigned char *plan = plans + (size_t)t2_rec_index(S.T, S.T1 <= kT2MaxT1 ? S.T1 : 0) * kT2Rec;
    const int *pint = reinterpret_cast<const int *>(plan + kT2RecPeak);
    if (S.T1 > kT2MaxT1 || pint[0] > kT2Cap || pint[1] < 3 * S.T0 + 4) {
      if (tid == 0) deferred[atomicAdd(work + 1, 1)] = cl;  // left to k_rasm_setup_tc
      continue;
    }
    const int T = S.T, N = S.N, T0 = S.T0, T1 = S.T1;
    const int ntix = T * (T + 1) / 2;
    for (int i = tid; i < (ntix + 3) / 4; i += kT2Threads)
      reinterpret_cast<unsigned *>(slot)[i] = __ldg(reinterpret_cast<const unsigned *>(plan) + i);
    for (int p = tid; p < N; p += kT2Threads) {
      const int gi = fac_to_global(R, S, p);
      pos[p] = (gi >= 0) ? xy[gi - st.ext_lo] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    T2P(1)
#ifdef RBF_PROBE
    if (tid == 0) g_t2_acc[blockIdx.x][0] += 1;
    ++t2_cellno;
#endif
    auto tile = [&](int it, int jt) -> double * { return sm + (int)slot[((it * (it + 1)) >> 1) + jt] * 64; };

    // ---- left-looking Cholesky over tile columns (as k_rasm_setup_tc), rows retired
    // to the workspace.  Accumulate warp w handles the rows j+1+w+kT2Acc m of column j;
    // with one row only, it runs two DMMA chains (even / odd kt) for it.
    double acc[kT2M][2], accb[2];
#pragma unroll
    for (int m = 0; m < kT2M; ++m) acc[m][0] = acc[m][1] = 0.0;
    accb[0] = accb[1] = 0.0;
    // the A entries of column 0's tiles (accumulators start at -A: C = -acc at the end)
    if (warp < kT2Acc) {
#pragma unroll
      for (int m = 0; m < kT2M; ++m) {
        const int it = 1 + warp + kT2Acc * m;
        if (it < T) {
          double v0, v1;
          a_entries(pos, S, g, it, 0, lane, v0, v1);
          acc[m][0] = -v0;
          acc[m][1] = -v1;
        }
      }
    } else if (warp == kT2Acc) {
      double v0, v1;
      a_entries(pos, S, g, 0, 0, lane, v0, v1);
      acc[0][0] = -v0;
      acc[0][1] = -v1;
    }
    for (int j = 0; j < T; ++j) {
      const int dw = kT2Acc + (j & 1);
      if (warp == 0) T2C(0)
      if (warp < kT2Acc) {
        // rows of column j (step 1) = rows of column j+1's accumulation (step 2) shifted
        const int nm1 = (T - (j + 1) - warp + kT2Acc - 1) / kT2Acc;  // it = j+1+warp+kT2Acc m < T
        const int nm2 = (T - (j + 2) - warp + kT2Acc - 1) / kT2Acc;
        // step 1: finish column j with the kt = j-1 term, store C = A - sum
        if (nm1 > 0) {
          const double *Bt = j >= 1 ? tile(j, j - 1) : sm;
          const double b0 = Bt[f0], b1 = Bt[f1];
#pragma unroll
          for (int m = 0; m < kT2M; ++m)
            if (m < nm1) {
              const int it = j + 1 + warp + kT2Acc * m;
              if (j >= 1) {
                const double *At = tile(it, j - 1);
                dmma(acc[m][0], acc[m][1], At[f0], b0);
                dmma(acc[m][0], acc[m][1], At[f1], b1);
              }
              double c0 = acc[m][0], c1 = acc[m][1];
              if (m == 0 && nm1 == 1) {
                c0 += accb[0];
                c1 += accb[1];
              }
              *reinterpret_cast<double2 *>(tile(it, j) + frag_acc(lane)) = make_double2(-c0, -c1);
            }
        }
        if (warp == 0) T2C(1)
        // step 2: accumulate column j+1 (rows it > j+1) over kt < j
        accb[0] = accb[1] = 0.0;
        if (nm2 > 0) {
#pragma unroll
          for (int m = 0; m < kT2M; ++m)
            if (m < nm2) {
              double v0, v1;
              a_entries(pos, S, g, j + 2 + warp + kT2Acc * m, j + 1, lane, v0, v1);
              acc[m][0] = -v0;
              acc[m][1] = -v1;
            }
          const unsigned char *sj = slot + (((j + 1) * (j + 2)) >> 1);
          if (nm2 == 1) {
            const int it = j + 2 + warp;
            const unsigned char *si = slot + ((it * (it + 1)) >> 1);
            int kt = 0;
            for (; kt + 1 < j; kt += 2) {
              const double *B0 = sm + (int)sj[kt] * 64, *B1 = sm + (int)sj[kt + 1] * 64;
              const double *A0 = sm + (int)si[kt] * 64, *A1 = sm + (int)si[kt + 1] * 64;
              dmma(acc[0][0], acc[0][1], A0[f0], B0[f0]);
              dmma(accb[0], accb[1], A1[f0], B1[f0]);
              dmma(acc[0][0], acc[0][1], A0[f1], B0[f1]);
              dmma(accb[0], accb[1], A1[f1], B1[f1]);
            }
            if (kt < j) {
              const double *B0 = sm + (int)sj[kt] * 64, *A0 = sm + (int)si[kt] * 64;
              dmma(acc[0][0], acc[0][1], A0[f0], B0[f0]);
              dmma(acc[0][0], acc[0][1], A0[f1], B0[f1]);
            }
          } else {
            switch (nm2) {  // straight-line code per tile count (no per-tile branches)
              case 2: t2_acc_rows<2>(acc, sm, slot, j, j + 2 + warp, f0, f1); break;
              case 3: t2_acc_rows<3>(acc, sm, slot, j, j + 2 + warp, f0, f1); break;
              case 4: t2_acc_rows<4>(acc, sm, slot, j, j + 2 + warp, f0, f1); break;
              default: t2_acc_rows<kT2M>(acc, sm, slot, j, j + 2 + warp, f0, f1); break;
            }
          }
        }
      } else if (warp == dw) {
        // finish the diagonal tile (its sum over kt < j-1 was accumulated last column)
        double *D = tile(j, j);
        if (j >= 1) {
          const double *Lt = tile(j, j - 1);
          const double l0 = Lt[f0], l1 = Lt[f1];
          dmma(acc[0][0], acc[0][1], l0, l0);
          dmma(accb[0], accb[1], l1, l1);
        }
        *reinterpret_cast<double2 *>(D + frag_acc(lane)) =
            make_double2(-(acc[0][0] + accb[0]), -(acc[0][1] + accb[1]));
        __syncwarp();
        T2C(5)
        if (diag_factor_t(D, rdiag, j, lane) && lane == 0) s_fail = 1;
        T2C(6)
      } else if (j + 1 < T) {
        // the other diagonal warp accumulates the next diagonal tile over kt < j
        double v0, v1;
        a_entries(pos, S, g, j + 1, j + 1, lane, v0, v1);
        acc[0][0] = -v0;
        acc[0][1] = -v1;
        accb[0] = accb[1] = 0.0;
        const unsigned char *sj = slot + (((j + 1) * (j + 2)) >> 1);
        int kt = 0;
        for (; kt + 1 < j; kt += 2) {
          const double *L0 = sm + (int)sj[kt] * 64, *L1 = sm + (int)sj[kt + 1] * 64;
          const double x0 = L0[f0], x1 = L0[f1], y0 = L1[f0], y1 = L1[f1];
          dmma(acc[0][0], acc[0][1], x0, x0);
          dmma(accb[0], accb[1], y0, y0);
          dmma(acc[0][0], acc[0][1], x1, x1);
          dmma(accb[0], accb[1], y1, y1);
        }
        if (kt < j) {
          const double *L0 = sm + (int)sj[kt] * 64;
          const double x0 = L0[f0], x1 = L0[f1];
          dmma(acc[0][0], acc[0][1], x0, x0);
          dmma(acc[0][0], acc[0][1], x1, x1);
        }
      }
      if (warp == 0) T2C(2)
      __syncthreads();
      if (warp == 0) T2C(3)
      if (s_fail) break;  // uniform
      if (warp < kT2Acc) {
        // panel L(it, j) = C(it, j) L_d^-T
        const int nm1 = (T - (j + 1) - warp + kT2Acc - 1) / kT2Acc;
        if (nm1 > 0) {
          const double *D = tile(j, j);
          double bv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 4 * h + (lane & 3), n = lane >> 2;
            bv[h] = (n > k) ? D[swz(k, n)] : (n == k ? rdiag[j * 8 + k] : 0.0);
          }
#pragma unroll
          for (int m = 0; m < kT2M; ++m)
            if (m < nm1) {
              double *Ct = tile(j + 1 + warp + kT2Acc * m, j);
              double d0 = 0.0, d1 = 0.0;
#pragma unroll
              for (int h = 0; h < 2; ++h) dmma(d0, d1, Ct[frag_rowk(lane, h)], bv[h]);
              __syncwarp();
              *reinterpret_cast<double2 *>(Ct + frag_acc(lane)) = make_double2(d0, d1);
            }
        }
      } else {
        // retire the rows the loop is done with (rows of L11 only): row j+1's tiles
        // (j+1, kt < j) and row j's last two, (j, j-1) and (j, j); their slots are
        // reused from the next column on (the plan frees them here)
        const int t = tid - kT2Acc * 32;
        const int na = (j + 1 < T0) ? j : 0;
        const int nb = (j < T0) ? (j >= 1 ? 2 : 1) : 0;
        for (int q = t; q < (na + nb) * 32; q += 64) {
          const int e = q >> 5, p = q & 31;
          int it, kt;
          if (e < na) {
            it = j + 1;
            kt = e;
          } else {
            it = j;
            kt = (e - na == nb - 1) ? j : j - 1;
          }
          const double2 v = *reinterpret_cast<const double2 *>(tile(it, kt) + 2 * p);
          __stcg(reinterpret_cast<double2 *>(wsl + (size_t)(t2_gcol(kt, T0) + it - kt) * 64 + 2 * p), v);
        }
      }
      if (warp == 0) T2C(4)
      __syncthreads();
    }
    if (s_fail) {  // Cholesky broke down: redo this cell with LU (reading Q11)
      if (tid == 0) glist[atomicAdd(&counts[3], 1)] = cl;
      continue;
    }

    T2P(2)
#ifdef RBF_PROBE
    const long long t2_post0 = clock64();
#endif
    // ---- W = L21 L11^-1 (warps 0..3, one own tile row each) and S^-1 (warps 4..7)
    const unsigned char *fl = plan + kT2RecFree;  // slots free after the factorisation
    if (warp < 4) {
      // W(r, jt) = (C(r, jt) - sum_{kt > jt} W(r, kt) L(kt, jt)) L_d(jt)^-1, jt = T0-1 .. 0;
      // column jt of L11 (tiles (jt..T0-1, jt), contiguous in the workspace) in ring buffer jt % 3
      // lane e holds the slot of tile e of each ring buffer (column jt of L11 is buffer
      // jt % 3, its tile e = row jt + e) and the slot of this warp's W(r, e)
      const int r = warp;
      int flr[3] = {0, 0, 0};
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (lane < T0) flr[b] = __ldg(fl + b * T0 + lane);
      const int wslot = (r < T1 && lane < T0) ? (int)slot[(((T0 + r) * (T0 + r + 1)) >> 1) + lane] : 0;
      auto fetch = [&](int jt) {
        const int nt = T0 - jt, b = jt % 3;
        const int fb = b == 0 ? flr[0] : (b == 1 ? flr[1] : flr[2]);
        const double *src = wsl + (size_t)t2_gcol(jt, T0) * 64;
        for (int e = warp; e < nt; e += 4) {  // one tile per warp and pass
          const int sl = __shfl_sync(0xffffffffu, fb, e);
          cp_async16(sm + sl * 64 + 2 * lane, src + e * 64 + 2 * lane);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      if (T0 >= 1) fetch(T0 - 1);
      if (T0 >= 2) fetch(T0 - 2);
      for (int jt = T0 - 1; jt >= 0; --jt) {
        if (warp == 0) T2W(0)
        if (jt >= 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        if (warp == 0) T2W(1)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 0) T2W(2)
        if (jt >= 2) fetch(jt - 2);
        if (warp == 0) T2W(3)
        if (r < T1) {
          const int b = jt % 3;
          const int fb = b == 0 ? flr[0] : (b == 1 ? flr[1] : flr[2]);
          double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
          int kt = jt + 1;
#pragma unroll 2
          for (; kt + 1 < T0; kt += 2) {
            const double *W0 = sm + __shfl_sync(0xffffffffu, wslot, kt) * 64;
            const double *W1 = sm + __shfl_sync(0xffffffffu, wslot, kt + 1) * 64;
            const double *L0 = sm + __shfl_sync(0xffffffffu, fb, kt - jt) * 64;
            const double *L1 = sm + __shfl_sync(0xffffffffu, fb, kt + 1 - jt) * 64;
            dmma(a0, a1, W0[f0], L0[frag_colk(lane, 0)]);
            dmma(c0, c1, W1[f0], L1[frag_colk(lane, 0)]);
            dmma(a0, a1, W0[f1], L0[frag_colk(lane, 1)]);
            dmma(c0, c1, W1[f1], L1[frag_colk(lane, 1)]);
          }
          if (kt < T0) {
            const double *W0 = sm + __shfl_sync(0xffffffffu, wslot, kt) * 64;
            const double *L0 = sm + __shfl_sync(0xffffffffu, fb, kt - jt) * 64;
            dmma(a0, a1, W0[f0], L0[frag_colk(lane, 0)]);
            dmma(a0, a1, W0[f1], L0[frag_colk(lane, 1)]);
          }
          if (warp == 0) T2W(4)
          double *Ct = sm + __shfl_sync(0xffffffffu, wslot, jt) * 64;
          double2 *cp = reinterpret_cast<double2 *>(Ct + frag_acc(lane));
          double2 cv = *cp;
          cv.x -= a0 + c0;
          cv.y -= a1 + c1;
          *cp = cv;
          __syncwarp();
          const double *D = sm + __shfl_sync(0xffffffffu, fb, 0) * 64;  // diagonal tile (jt, jt)
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 4 * h + (lane & 3), n = lane >> 2;
            const double bv = (k > n) ? D[swz(n, k)] : (k == n ? rdiag[jt * 8 + k] : 0.0);
            dmma(d0, d1, Ct[frag_rowk(lane, h)], bv);
          }
          __syncwarp();
          *cp = make_double2(d0, d1);
          __syncwarp();
          if (warp == 0) T2W(5)
        }
      }
#ifdef RBF_PROBE
      if (tid == 0) g_t2_acc[blockIdx.x][5] += clock64() - t2_post0;
#endif
    } else {
      // S^-1 = L22^-T L22^-1 (as setup_post): M = L22^-1 by columns, one warp per column
      const int sw = warp - 4;
      double *Mt = reinterpret_cast<double *>(pos);
      double *scr = sm + (int)__ldg(fl + 3 * T0 + sw) * 64;
      auto mt = [&](int a, int b) { return Mt + ((a * (a - 1)) / 2 + b) * 64; };  // a > b only
      const int m_ = lane >> 2, q_ = lane & 3;
      auto linvA = [&](int a, int h) -> double {
        const double *D = tile(T0 + a, T0 + a);
        const int kk = 4 * h + q_;
        return (m_ > kk) ? D[swz(kk, m_)] : (m_ == kk ? rdiag[(T0 + a) * 8 + m_] : 0.0);
      };
      auto linvB = [&](int a, int h) -> double {
        const double *D = tile(T0 + a, T0 + a);
        const int kk = 4 * h + q_;
        return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiag[(T0 + a) * 8 + kk] : 0.0);
      };
      auto linvT = [&](int a, int h) -> double {
        const double *D = tile(T0 + a, T0 + a);
        const int kk = 4 * h + q_;
        return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiag[(T0 + a) * 8 + m_] : 0.0);
      };
      for (int b = sw; b < T1 - 1; b += 4) {
        for (int a = b + 1; a < T1; ++a) {
          double d0 = 0.0, d1 = 0.0;
          for (int k = b; k < a; ++k) {
            const double *La = tile(T0 + a, T0 + k);
#pragma unroll
            for (int h = 0; h < 2; ++h)
              dmma(d0, d1, La[frag_rowk(lane, h)], k == b ? linvB(b, h) : mt(k, b)[frag_colk(lane, h)]);
          }
          *reinterpret_cast<double2 *>(scr + frag_acc(lane)) = make_double2(d0, d1);
          __syncwarp();
          double e0 = 0.0, e1 = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) dmma(e0, e1, linvA(a, h), scr[frag_colk(lane, h)]);
          __syncwarp();
          *reinterpret_cast<double2 *>(mt(a, b) + frag_acc(lane)) = make_double2(-e0, -e1);
          __syncwarp();
        }
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");  // M complete
      constexpr int kSlots = (kT2MaxT1 * (kT2MaxT1 + 1) / 2 + 3) / 4;
      double res[kSlots][2];
      const int ntl = T1 * (T1 + 1) / 2;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int t = sw + sl * 4;
        res[sl][0] = res[sl][1] = 0.0;
        if (t < ntl) {
          int a = 0;
          while ((a + 1) * (a + 2) / 2 <= t) ++a;
          const int bb = t - a * (a + 1) / 2;
          for (int k = a; k < T1; ++k) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double av = (k == a) ? linvT(a, h) : mt(k, a)[frag_colk(lane, h)];
              const double bv = (k == bb) ? linvB(bb, h) : mt(k, bb)[frag_colk(lane, h)];
              dmma(res[sl][0], res[sl][1], av, bv);
            }
          }
        }
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");  // L^-1 scratch read
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int t = sw + sl * 4;
        if (t < ntl) {
          int a = 0;
          while ((a + 1) * (a + 2) / 2 <= t) ++a;
          const int bb = t - a * (a + 1) / 2;
          *reinterpret_cast<double2 *>(tile(T0 + a, T0 + bb) + frag_acc(lane)) =
              make_double2(res[sl][0], res[sl][1]);
        }
      }
#ifdef RBF_PROBE
      if (tid == 128) g_t2_acc[blockIdx.x][6] += clock64() - t2_post0;
#endif
    }
    __syncthreads();
    T2P(3)

    // ---- X_c = S^-1 [-W, I] in natural column order (ld = n rounded up to even), to HBM
    const int n = S.n;
    const int ld = (n + 1) & ~1;
    double *Xc = X + x_off[cl];
    auto x_store = [&](int ot, int jt, double d0, double d1) {
      const int o = ot * 8 + (lane >> 2);
      const int p0 = jt * 8 + 2 * (lane & 3);
      if (o < S.n1) {
        if (p0 < S.n0) Xc[(size_t)o * ld + (p0 < R.own_nat_lo ? p0 : p0 + S.n1)] = -d0;
        if (p0 + 1 < S.n0) Xc[(size_t)o * ld + (p0 + 1 < R.own_nat_lo ? p0 + 1 : p0 + 1 + S.n1)] = -d1;
      }
    };
    auto sinv_frag = [&](int ot, int kt, int h) -> double {
      const bool lower = kt <= ot;
      const double *At = lower ? tile(T0 + ot, T0 + kt) : tile(T0 + kt, T0 + ot);
      const int m = lane >> 2, k = 4 * h + (lane & 3);
      return lower ? At[swz(m, k)] : At[swz(k, m)];
    };
    for (int task = warp; task < T1 * T0; task += kT2Warps) {
      const int ot = task / T0, jt = task - ot * T0;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
      for (int kt = 0; kt < T1; ++kt) {
        const double *Bt = tile(T0 + kt, jt);
        if (kt & 1) {
          dmma(e0, e1, sinv_frag(ot, kt, 0), Bt[frag_colk(lane, 0)]);
          dmma(e0, e1, sinv_frag(ot, kt, 1), Bt[frag_colk(lane, 1)]);
        } else {
          dmma(d0, d1, sinv_frag(ot, kt, 0), Bt[frag_colk(lane, 0)]);
          dmma(d0, d1, sinv_frag(ot, kt, 1), Bt[frag_colk(lane, 1)]);
        }
      }
      x_store(ot, jt, d0 + e0, d1 + e1);
    }
    for (int t = tid; t < S.n1 * S.n1; t += kT2Threads) {
      const int o = t / S.n1, jj = t - o * S.n1;
      const int i1 = o >= jj ? o : jj, j1 = o >= jj ? jj : o;
      Xc[(size_t)o * ld + R.own_nat_lo + jj] = tile(T0 + (i1 >> 3), T0 + (j1 >> 3))[swz(i1 & 7, j1 & 7)];
    }
    if (ld != n)
      for (int o = tid; o < S.n1; o += kT2Threads) Xc[(size_t)o * ld + n] = 0.0;
    T2P(4)
  }
}

// ---------------------------------------------------------------------------
// Factorisation and post phase pipelined on one SM: k_rasm_setup_tc3 (option setup_tc = 3).
//
// One persistent CTA of 20 warps per SM (96 registers).  Warps 0..15 factor cell i (14
// accumulate warps, two alternating diagonal warps; the row-retiring column loop of
// k_rasm_setup_tc2 in its 212-slot region C), while warps 16..19 run the post phase of cell i-1 -- W = L21 L11^-1
// from the retired L11 columns (cp.async ring), S^-1 = L22^-T L22^-1 and X_c = S^-1 [-W, I]
// -- from a region P that holds that cell's own tile rows.  At the end of cell i's
// factorisation the two groups meet (named barrier 3): the post warps are done with cell
// i-1, the factor warps copy cell i's own rows and diagonal reciprocals into P and hand
// over.  The retired rows alternate between two workspace slices per CTA, so that cell
// i+1 can retire rows while the post warps read cell i's.  Measured: the
// post phase is hidden (75k of the 155k cycles per cell), but the factorisation next to it
// takes 155k cycles instead of the one-per-SM kernel's 125k, so the setup is at parity.
// ---------------------------------------------------------------------------
constexpr int kT3FacWarps = 16;              // factor warps 0..15
constexpr int kT3Threads = (kT3FacWarps + 4) * 32;
constexpr int kT3Acc = kT3FacWarps - 2;      // accumulate warps; the last two alternate as diagonal warps
constexpr int kT3M = (kTcMaxTiles - 1 + kT3Acc - 1) / kT3Acc;  // rows per accumulate warp and column
constexpr int kT3PostWarps = 4;              // the last four warps
constexpr int kT3OwnTiles = kT2MaxT1 * kTcMaxTiles;   // P: own tile rows, row-major (r, jt)
constexpr int kT3Ring = 3 * kTcMaxTiles;             // P: three L11 column buffers
constexpr int kT3Scr = 4;                            // P: S^-1 product scratch, one per warp
constexpr int kT3MTiles = kT2MaxT1 * (kT2MaxT1 - 1) / 2;  // P: M = L22^-1 strictly lower tiles
constexpr size_t kT3SmemTiles = (size_t)kT2Cap + kT3OwnTiles + kT3Ring + kT3Scr + kT3MTiles;
constexpr size_t kT3Smem = kT3SmemTiles * 512 + 2 * kTcMaxTiles * 8 * sizeof(double) +
                           kTcMaxTiles * 8 * sizeof(double2) + 440;

struct T3Post {  // the cell handed to the post warps
  int cl, n, n0, n1, own_nat_lo, T0, T1, slice;
};

__global__ __launch_bounds__(kT3Threads, 1) void k_rasm_setup_tc3(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, int *__restrict__ counts,
    int *__restrict__ glist, OvList ov, const unsigned char *__restrict__ plans, double *__restrict__ ws,
    int *__restrict__ work, int *__restrict__ deferred, int ncl) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Runs R;
  __shared__ int s_cl, s_fail;
  __shared__ T3Post s_post;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *Pown = sm + (size_t)kT2Cap * 64;            // own tile (T0 + r, jt) at Pown + (r * 29 + jt) * 64
  double *Pring = Pown + (size_t)kT3OwnTiles * 64;    // ring tile e of buffer b at Pring + (b * 29 + e) * 64
  double *Pscr = Pring + (size_t)kT3Ring * 64;        // scratch of post warp w at Pscr + w * 64
  double *Pm = Pscr + (size_t)kT3Scr * 64;            // M tiles
  double *rdiag = Pm + (size_t)kT3MTiles * 64;        // factor side
  double *rdiagP = rdiag + kTcMaxTiles * 8;           // post side
  double2 *pos = reinterpret_cast<double2 *>(rdiagP + kTcMaxTiles * 8);
  unsigned char *slot = reinterpret_cast<unsigned char *>(pos + kTcMaxTiles * 8);
  const int f0 = frag_rowk(lane, 0), f1 = frag_rowk(lane, 1);
#ifdef RBF_PROBE
#define T3P(k, who)                                                   \
  if (tid == (who)) {                                                 \
    const long long t_ = clock64();                                   \
    if ((k) > 0) g_t2_acc[blockIdx.x][k] += t_ - t3_last;             \
    t3_last = t_;                                                     \
  }
  long long t3_last = 0;
#else
#define T3P(k, who) {}
#endif

  if (warp >= kT3FacWarps) {
    // =================== post warps: W, S^-1, X of the handed-over cell ===================
    const int pw = warp - kT3FacWarps, ptid = tid - kT3FacWarps * 32;
    for (;;) {
      asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");  // done with the previous cell
      asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");  // the next cell is in P
      const T3Post q = s_post;
      if (q.cl < 0) return;
      T3P(0, kT3FacWarps * 32)
#ifdef RBF_T3_NOPOST
      continue;  // timing diagnostic only: the factorisation without the post phase
#endif
      const int T0 = q.T0, T1 = q.T1;
      const double *wsl = ws + ((size_t)blockIdx.x * 2 + q.slice) * kT2WsTiles * 64;
      auto ptile = [&](int it, int jt) -> double * { return Pown + ((it - T0) * kTcMaxTiles + jt) * 64; };
      // ---- W(r, jt) = (C(r, jt) - sum_{kt > jt} W(r, kt) L(kt, jt)) L_d(jt)^-1, jt = T0-1..0
      auto fetch = [&](int jt) {
        const int nt = T0 - jt, b = jt % 3;
        const double2 *src = reinterpret_cast<const double2 *>(wsl + (size_t)t2_gcol(jt, T0) * 64);
        double2 *dst = reinterpret_cast<double2 *>(Pring + (size_t)b * kTcMaxTiles * 64);
        for (int q2 = ptid; q2 < nt * 32; q2 += kT3PostWarps * 32) cp_async16(dst + q2, src + q2);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      if (T0 >= 1) fetch(T0 - 1);
      if (T0 >= 2) fetch(T0 - 2);
      const int r = pw;
      for (int jt = T0 - 1; jt >= 0; --jt) {
        if (jt >= 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"n"(kT3PostWarps * 32) : "memory");
        if (jt >= 2) fetch(jt - 2);
        if (r < T1) {
          const double *col = Pring + (size_t)(jt % 3) * kTcMaxTiles * 64;  // tile e = L(jt + e, jt)
          const int g0 = frag_colk(lane, 0), g1 = frag_colk(lane, 1);
          double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
          const double *Wr = ptile(T0 + r, 0);
          int kt = jt + 1;
#pragma unroll 2
          for (; kt + 1 < T0; kt += 2) {
            const double *W0 = Wr + kt * 64, *W1 = W0 + 64;
            const double *L0 = col + (kt - jt) * 64, *L1 = L0 + 64;
            dmma(a0, a1, W0[f0], L0[g0]);
            dmma(c0, c1, W1[f0], L1[g0]);
            dmma(a0, a1, W0[f1], L0[g1]);
            dmma(c0, c1, W1[f1], L1[g1]);
          }
          if (kt < T0) {
            const double *W0 = Wr + kt * 64, *L0 = col + (kt - jt) * 64;
            dmma(a0, a1, W0[f0], L0[g0]);
            dmma(a0, a1, W0[f1], L0[g1]);
          }
          double *Ct = ptile(T0 + r, jt);
          double2 *cp = reinterpret_cast<double2 *>(Ct + frag_acc(lane));
          double2 cv = *cp;
          cv.x -= a0 + c0;
          cv.y -= a1 + c1;
          *cp = cv;
          __syncwarp();
          const double *D = col;  // diagonal tile (jt, jt)
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 4 * h + (lane & 3), n = lane >> 2;
            const double bv = (k > n) ? D[swz(n, k)] : (k == n ? rdiagP[jt * 8 + k] : 0.0);
            dmma(d0, d1, Ct[frag_rowk(lane, h)], bv);
          }
          __syncwarp();
          *cp = make_double2(d0, d1);
          __syncwarp();
        }
      }
      T3P(5, kT3FacWarps * 32)
      // ---- S^-1 = L22^-T L22^-1 (M = L22^-1 by columns, one warp per column)
      {
        const int sw = pw;
        double *scr = Pscr + sw * 64;
        auto mt = [&](int a, int b) { return Pm + ((a * (a - 1)) / 2 + b) * 64; };  // a > b only
        const int m_ = lane >> 2, q_ = lane & 3;
        auto linvA = [&](int a, int h) -> double {
          const double *D = ptile(T0 + a, T0 + a);
          const int kk = 4 * h + q_;
          return (m_ > kk) ? D[swz(kk, m_)] : (m_ == kk ? rdiagP[(T0 + a) * 8 + m_] : 0.0);
        };
        auto linvB = [&](int a, int h) -> double {
          const double *D = ptile(T0 + a, T0 + a);
          const int kk = 4 * h + q_;
          return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiagP[(T0 + a) * 8 + kk] : 0.0);
        };
        auto linvT = [&](int a, int h) -> double {
          const double *D = ptile(T0 + a, T0 + a);
          const int kk = 4 * h + q_;
          return (kk > m_) ? D[swz(m_, kk)] : (kk == m_ ? rdiagP[(T0 + a) * 8 + m_] : 0.0);
        };
        for (int b = sw; b < T1 - 1; b += kT3PostWarps) {
          for (int a = b + 1; a < T1; ++a) {
            double d0 = 0.0, d1 = 0.0;
            for (int k = b; k < a; ++k) {
              const double *La = ptile(T0 + a, T0 + k);
#pragma unroll
              for (int h = 0; h < 2; ++h)
                dmma(d0, d1, La[frag_rowk(lane, h)], k == b ? linvB(b, h) : mt(k, b)[frag_colk(lane, h)]);
            }
            *reinterpret_cast<double2 *>(scr + frag_acc(lane)) = make_double2(d0, d1);
            __syncwarp();
            double e0 = 0.0, e1 = 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) dmma(e0, e1, linvA(a, h), scr[frag_colk(lane, h)]);
            __syncwarp();
            *reinterpret_cast<double2 *>(mt(a, b) + frag_acc(lane)) = make_double2(-e0, -e1);
            __syncwarp();
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kT3PostWarps * 32) : "memory");  // M complete
        constexpr int kSlots = (kT2MaxT1 * (kT2MaxT1 + 1) / 2 + kT3PostWarps - 1) / kT3PostWarps;
        double res[kSlots][2];
        const int ntl = T1 * (T1 + 1) / 2;
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const int t = sw + sl * kT3PostWarps;
          res[sl][0] = res[sl][1] = 0.0;
          if (t < ntl) {
            int a = 0;
            while ((a + 1) * (a + 2) / 2 <= t) ++a;
            const int bb = t - a * (a + 1) / 2;
            for (int k = a; k < T1; ++k) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const double av = (k == a) ? linvT(a, h) : mt(k, a)[frag_colk(lane, h)];
                const double bv = (k == bb) ? linvB(bb, h) : mt(k, bb)[frag_colk(lane, h)];
                dmma(res[sl][0], res[sl][1], av, bv);
              }
            }
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kT3PostWarps * 32) : "memory");  // L^-1 scratch read
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const int t = sw + sl * kT3PostWarps;
          if (t < ntl) {
            int a = 0;
            while ((a + 1) * (a + 2) / 2 <= t) ++a;
            const int bb = t - a * (a + 1) / 2;
            *reinterpret_cast<double2 *>(ptile(T0 + a, T0 + bb) + frag_acc(lane)) =
                make_double2(res[sl][0], res[sl][1]);
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kT3PostWarps * 32) : "memory");  // S^-1 final
      }
      T3P(6, kT3FacWarps * 32)
      // ---- X_c = S^-1 [-W, I] in natural column order (ld = n rounded up to even), to HBM
      {
        const int n = q.n, n0 = q.n0, n1 = q.n1, onl = q.own_nat_lo;
        const int ld = (n + 1) & ~1;
        double *Xc = X + x_off[q.cl];
        auto sinv_frag = [&](int ot, int kt, int h) -> double {
          const bool lower = kt <= ot;
          const double *At = lower ? ptile(T0 + ot, T0 + kt) : ptile(T0 + kt, T0 + ot);
          const int m = lane >> 2, k = 4 * h + (lane & 3);
          return lower ? At[swz(m, k)] : At[swz(k, m)];
        };
        for (int task = pw; task < T1 * T0; task += kT3PostWarps) {
          const int ot = task / T0, jt = task - ot * T0;
          double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
          for (int kt = 0; kt < T1; ++kt) {
            const double *Bt = ptile(T0 + kt, jt);
            if (kt & 1) {
              dmma(e0, e1, sinv_frag(ot, kt, 0), Bt[frag_colk(lane, 0)]);
              dmma(e0, e1, sinv_frag(ot, kt, 1), Bt[frag_colk(lane, 1)]);
            } else {
              dmma(d0, d1, sinv_frag(ot, kt, 0), Bt[frag_colk(lane, 0)]);
              dmma(d0, d1, sinv_frag(ot, kt, 1), Bt[frag_colk(lane, 1)]);
            }
          }
          const int o = ot * 8 + (lane >> 2);
          const int p0 = jt * 8 + 2 * (lane & 3);
          if (o < n1) {
            if (p0 < n0) Xc[(size_t)o * ld + (p0 < onl ? p0 : p0 + n1)] = -(d0 + e0);
            if (p0 + 1 < n0) Xc[(size_t)o * ld + (p0 + 1 < onl ? p0 + 1 : p0 + 1 + n1)] = -(d1 + e1);
          }
        }
        for (int t = ptid; t < n1 * n1; t += kT3PostWarps * 32) {
          const int o = t / n1, jj = t - o * n1;
          const int i1 = o >= jj ? o : jj, j1 = o >= jj ? jj : o;
          Xc[(size_t)o * ld + onl + jj] = ptile(T0 + (i1 >> 3), T0 + (j1 >> 3))[swz(i1 & 7, j1 & 7)];
        }
        if (ld != n)
          for (int o = ptid; o < n1; o += kT3PostWarps * 32) Xc[(size_t)o * ld + n] = 0.0;
      }
      T3P(7, kT3FacWarps * 32)
    }
  }

  // =================== factor warps 0..11 ===================
  int ncell = 0;
  for (;;) {
    asm volatile("bar.sync 1, %0;" ::"n"(kT3FacWarps * 32) : "memory");  // done with R and region C
    T3P(0, 0)
    if (tid == 0) {
      const int cl = atomicAdd(work, 1);
      s_cl = cl;
      s_fail = 0;
      if (cl < ncl) sub_runs(g, cell_start, ov, cl, cl % g.ncx, st.row_lo + cl / g.ncx, R);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kT3FacWarps * 32) : "memory");
    const int cl = s_cl;
    if (cl >= ncl) break;
    if (R.n_own == 0) continue;
    const TileShape S(R.n_ov, R.n_own);
    if (!S.fits_tc()) continue;  // handled by k_rasm_setup_lu
    const unsigned char *plan = plans + (size_t)t2_rec_index(S.T, S.T1 <= kT2MaxT1 ? S.T1 : 0) * kT2Rec;
    const int *pint = reinterpret_cast<const int *>(plan + kT2RecPeak);
    if (S.T1 > kT2MaxT1 || pint[0] > kT2Cap) {
      if (tid == 0) deferred[atomicAdd(work + 1, 1)] = cl;  // left to k_rasm_setup_tc
      continue;
    }
    const int T = S.T, N = S.N, T0 = S.T0, T1 = S.T1;
    const int slice = ncell & 1;
    double *wsl = ws + ((size_t)blockIdx.x * 2 + slice) * kT2WsTiles * 64;
    const int ntix = T * (T + 1) / 2;
    for (int i = tid; i < (ntix + 3) / 4; i += kT3FacWarps * 32)
      reinterpret_cast<unsigned *>(slot)[i] = __ldg(reinterpret_cast<const unsigned *>(plan) + i);
    for (int p = tid; p < N; p += kT3FacWarps * 32) {
      const int gi = fac_to_global(R, S, p);
      pos[p] = (gi >= 0) ? xy[gi - st.ext_lo] : make_double2(0.0, 0.0);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kT3FacWarps * 32) : "memory");
    auto tile = [&](int it, int jt) -> double * { return sm + (int)slot[((it * (it + 1)) >> 1) + jt] * 64; };
    T3P(1, 0)
#ifdef RBF_PROBE
    if (tid == 0) g_t2_acc[blockIdx.x][0] += 1;
#endif

    double acc[kT3M][2], accb[2];
#pragma unroll
    for (int m = 0; m < kT3M; ++m) acc[m][0] = acc[m][1] = 0.0;
    accb[0] = accb[1] = 0.0;
    if (warp < kT3Acc) {
#pragma unroll
      for (int m = 0; m < kT3M; ++m) {
        const int it = 1 + warp + kT3Acc * m;
        if (it < T) {
          double v0, v1;
          a_entries(pos, S, g, it, 0, lane, v0, v1);
          acc[m][0] = -v0;
          acc[m][1] = -v1;
        }
      }
    } else if (warp == kT3Acc) {
      double v0, v1;
      a_entries(pos, S, g, 0, 0, lane, v0, v1);
      acc[0][0] = -v0;
      acc[0][1] = -v1;
    }
    for (int j = 0; j < T; ++j) {
      const int dw = kT3Acc + (j & 1);
      if (warp < kT3Acc) {
        const int nm1 = (T - (j + 1) - warp + kT3Acc - 1) / kT3Acc;
        const int nm2 = (T - (j + 2) - warp + kT3Acc - 1) / kT3Acc;
        if (nm1 > 0) {
          const double *Bt = j >= 1 ? tile(j, j - 1) : sm;
          const double b0 = Bt[f0], b1 = Bt[f1];
#pragma unroll
          for (int m = 0; m < kT3M; ++m)
            if (m < nm1) {
              const int it = j + 1 + warp + kT3Acc * m;
              if (j >= 1) {
                const double *At = tile(it, j - 1);
                dmma(acc[m][0], acc[m][1], At[f0], b0);
                dmma(acc[m][0], acc[m][1], At[f1], b1);
              }
              double c0 = acc[m][0], c1 = acc[m][1];
              if (m == 0 && nm1 == 1) {
                c0 += accb[0];
                c1 += accb[1];
              }
              *reinterpret_cast<double2 *>(tile(it, j) + frag_acc(lane)) = make_double2(-c0, -c1);
            }
        }
        accb[0] = accb[1] = 0.0;
        if (nm2 > 0) {
#pragma unroll
          for (int m = 0; m < kT3M; ++m)
            if (m < nm2) {
              double v0, v1;
              a_entries(pos, S, g, j + 2 + warp + kT3Acc * m, j + 1, lane, v0, v1);
              acc[m][0] = -v0;
              acc[m][1] = -v1;
            }
          if (nm2 == 1) {
            const unsigned char *sj = slot + (((j + 1) * (j + 2)) >> 1);
            const int it = j + 2 + warp;
            const unsigned char *si = slot + ((it * (it + 1)) >> 1);
            int kt = 0;
            for (; kt + 1 < j; kt += 2) {
              const double *B0 = sm + (int)sj[kt] * 64, *B1 = sm + (int)sj[kt + 1] * 64;
              const double *A0 = sm + (int)si[kt] * 64, *A1 = sm + (int)si[kt + 1] * 64;
              dmma(acc[0][0], acc[0][1], A0[f0], B0[f0]);
              dmma(accb[0], accb[1], A1[f0], B1[f0]);
              dmma(acc[0][0], acc[0][1], A0[f1], B0[f1]);
              dmma(accb[0], accb[1], A1[f1], B1[f1]);
            }
            if (kt < j) {
              const double *B0 = sm + (int)sj[kt] * 64, *A0 = sm + (int)si[kt] * 64;
              dmma(acc[0][0], acc[0][1], A0[f0], B0[f0]);
              dmma(acc[0][0], acc[0][1], A0[f1], B0[f1]);
            }
          } else if (nm2 == 2) {
            t2_acc_rows<2, kT3Acc, kT3M>(acc, sm, slot, j, j + 2 + warp, f0, f1);
          } else {
            t2_acc_rows<kT3M, kT3Acc, kT3M>(acc, sm, slot, j, j + 2 + warp, f0, f1);
          }
        }
      } else if (warp == dw) {
        double *D = tile(j, j);
        if (j >= 1) {
          const double *Lt = tile(j, j - 1);
          const double l0 = Lt[f0], l1 = Lt[f1];
          dmma(acc[0][0], acc[0][1], l0, l0);
          dmma(accb[0], accb[1], l1, l1);
        }
        *reinterpret_cast<double2 *>(D + frag_acc(lane)) =
            make_double2(-(acc[0][0] + accb[0]), -(acc[0][1] + accb[1]));
        __syncwarp();
        if (diag_factor_t(D, rdiag, j, lane) && lane == 0) s_fail = 1;
      } else if (j + 1 < T) {
        double v0, v1;
        a_entries(pos, S, g, j + 1, j + 1, lane, v0, v1);
        acc[0][0] = -v0;
        acc[0][1] = -v1;
        accb[0] = accb[1] = 0.0;
        const unsigned char *sj = slot + (((j + 1) * (j + 2)) >> 1);
        int kt = 0;
        for (; kt + 1 < j; kt += 2) {
          const double *L0 = sm + (int)sj[kt] * 64, *L1 = sm + (int)sj[kt + 1] * 64;
          const double x0 = L0[f0], x1 = L0[f1], y0 = L1[f0], y1 = L1[f1];
          dmma(acc[0][0], acc[0][1], x0, x0);
          dmma(accb[0], accb[1], y0, y0);
          dmma(acc[0][0], acc[0][1], x1, x1);
          dmma(accb[0], accb[1], y1, y1);
        }
        if (kt < j) {
          const double *L0 = sm + (int)sj[kt] * 64;
          const double x0 = L0[f0], x1 = L0[f1];
          dmma(acc[0][0], acc[0][1], x0, x0);
          dmma(acc[0][0], acc[0][1], x1, x1);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kT3FacWarps * 32) : "memory");
      if (s_fail) break;  // uniform
      if (warp < kT3Acc) {
        const int nm1 = (T - (j + 1) - warp + kT3Acc - 1) / kT3Acc;
        if (nm1 > 0) {
          const double *D = tile(j, j);
          double bv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 4 * h + (lane & 3), n = lane >> 2;
            bv[h] = (n > k) ? D[swz(k, n)] : (n == k ? rdiag[j * 8 + k] : 0.0);
          }
#pragma unroll
          for (int m = 0; m < kT3M; ++m)
            if (m < nm1) {
              double *Ct = tile(j + 1 + warp + kT3Acc * m, j);
              double d0 = 0.0, d1 = 0.0;
#pragma unroll
              for (int h = 0; h < 2; ++h) dmma(d0, d1, Ct[frag_rowk(lane, h)], bv[h]);
              __syncwarp();
              *reinterpret_cast<double2 *>(Ct + frag_acc(lane)) = make_double2(d0, d1);
            }
        }
      } else {
        // retire row j+1's tiles (j+1, kt < j) and row j's (j, j-1), (j, j) (rows of L11)
        const int t = tid - kT3Acc * 32;
        const int na = (j + 1 < T0) ? j : 0;
        const int nb = (j < T0) ? (j >= 1 ? 2 : 1) : 0;
        for (int q2 = t; q2 < (na + nb) * 32; q2 += 64) {
          const int e = q2 >> 5, p = q2 & 31;
          int it, kt;
          if (e < na) {
            it = j + 1;
            kt = e;
          } else {
            it = j;
            kt = (e - na == nb - 1) ? j : j - 1;
          }
          const double2 v = *reinterpret_cast<const double2 *>(tile(it, kt) + 2 * p);
          __stcg(reinterpret_cast<double2 *>(wsl + (size_t)(t2_gcol(kt, T0) + it - kt) * 64 + 2 * p), v);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kT3FacWarps * 32) : "memory");
    }
    if (s_fail) {  // Cholesky broke down: redo this cell with LU (reading Q11)
      if (tid == 0) glist[atomicAdd(&counts[3], 1)] = cl;
      continue;
    }
    T3P(2, 0)
    // ---- hand the cell over: wait for the post warps, copy the own rows into P
    asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");
    T3P(3, 0)
    for (int q2 = tid; q2 < T1 * T * 32; q2 += kT3FacWarps * 32) {
      const int e = q2 >> 5, p = q2 & 31;
      const int r = e / T, jt = e - r * T;
      if (jt <= T0 + r) {
        const double2 v = *reinterpret_cast<const double2 *>(tile(T0 + r, jt) + 2 * p);
        *reinterpret_cast<double2 *>(Pown + ((size_t)r * kTcMaxTiles + jt) * 64 + 2 * p) = v;
      }
    }
    for (int i = tid; i < T * 8; i += kT3FacWarps * 32) rdiagP[i] = rdiag[i];
    if (tid == 0) s_post = T3Post{cl, S.n, S.n0, S.n1, R.own_nat_lo, T0, T1, slice};
    asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");
    T3P(4, 0)
    ++ncell;
  }
  // no cells left: release the post warps
  asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");
  if (tid == 0) s_post.cl = -1;
  asm volatile("bar.sync 3, %0;" ::"n"(kT3Threads) : "memory");
}

// Global-memory local solve for subdomains whose factor does not fit in shared
// memory, and for cells whose Cholesky broke down (reading Q11): LU with partial
// pivoting (largest |a|, lowest row on ties) of the augmented matrix [A_c | E_own]
// in factor order, then back substitution U Z = L^-1 P E_own; X_c = Z^T.
//
// Right-looking and blocked by kLuNb columns so that the trailing matrix is read
// and written once per panel instead of once per column: (1) the panel is factored
// in a transposed copy PT (kLuNb x n, coalesced column access), whole rows are
// swapped eagerly in A; (2) the unit-lower solve U12 = L11^-1 A12 over all remaining
// columns, then the rank-kLuNb update A22 -= L21 U12 on the fp64 tensor cores
// (lu_trailing_update: DMMA.8x8x4, L21 fragments in registers).  The back substitution
// is blocked the same way.  One CTA per cell; A (n x lda, lda = n +
// n_own) and PT live in a per-CTA slice of a global workspace (L2).
// threads per LU CTA: 512 (one cell per SM) for subdomains beyond kLuBigN points, else
// 256 (two cells in flight per SM: the panel's barrier and L2 latency hide better)
constexpr int kLuBigN = 330;
constexpr int kLuNb = 32;     // panel width
constexpr int kBsCols = 64;   // right-hand-side columns per back-substitution sweep

__device__ __forceinline__ void lu_argmax(double v, int i, double *red_v, int *red_i, int *out) {
  // CTA reduction: largest value, lowest index on ties; result in *out (shared)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
  if (lane == 0) { red_v[warp] = v; red_i[warp] = i; }
  __syncthreads();
  if (warp == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? red_v[lane] : -1.0;
    i = (lane < (int)(blockDim.x >> 5)) ? red_i[lane] : 0x7fffffff;
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
      if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
    }
    if (lane == 0) *out = (v > 0.0) ? i : -1;
  }
  __syncthreads();
}

// Trailing update of one panel step:
// (1) U12 = L11^-1 A12 for every column right of the panel, one column per thread over
//     all threads (the unit-lower L11 in shared memory), written back in place;
// (2) A22 -= L21 U12 on DMMA.8x8x4: work items of 8 RT rows x 64 columns spread over
//     the warps; a warp holds its item's L21 fragments (RT row tiles x k = 32) in
//     registers and walks the 8 column tiles with the next tile's U12 fragments and C
//     values loaded before the current tile's RT independent DMMA chains run.  (Round 1
//     solved U12 in 64-column blocks on 64 threads, staged each block in shared memory
//     behind a barrier and ran one 8-DMMA chain per load round trip: 9-16% slower.)
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

template <int RT, bool SYM>
__device__ __forceinline__ void lu_trailing_update(double *__restrict__ A, const double *__restrict__ PT,
                                                   const double (*L11)[kLuNb + 1], const double *dpiv, int n,
                                                   long long lda, int k0, int kb) {
  const int tid = threadIdx.x, T = blockDim.x;
  const int j0 = k0 + kb;
  const unsigned l11 = (unsigned)__cvta_generic_to_shared(&L11[0][0]);
  // SYM: U12 is solved for the right-hand-side columns only (left of n, U = D L^T)
  for (long long j = (SYM ? n : j0) + tid; j < lda; j += T) {
    double u[kLuNb];
#pragma unroll
    for (int t = 0; t < kLuNb; ++t) u[t] = t < kb ? A[(long long)(k0 + t) * lda + j] : 0.0;
    // L11 read with volatile shared loads: the compiler would otherwise hoist all 496
    // entries out of the column loop and spill them to local memory
#pragma unroll
    for (int r = 1; r < kLuNb; ++r)
#pragma unroll
      for (int t = 0; t < r; ++t) u[r] = fma(-lds_f64(l11 + 8u * (unsigned)(r * (kLuNb + 1) + t)), u[t], u[r]);
#pragma unroll
    for (int t = 0; t < kLuNb; ++t)
      if (t < kb) A[(long long)(k0 + t) * lda + j] = u[t];
  }
  __syncthreads();
  LUP(3)
  const int lane = tid & 31, warp = tid >> 5, nwarps = T >> 5, q = lane & 3, r8 = lane >> 2;
  const int m = n - j0;
  const long long w = lda - j0;
  if (m <= 0 || w <= 0) return;
  constexpr int RH = 8 * RT;  // rows per work item
  // 32-bit element offsets (n * lda < 2^31 on this path)
  const int ldi = (int)lda;
  // column chunks of 64: SYM splits them at n (left: the lower triangle plus the strip up
  // to the end of the row group's own 32-row panel block, so that every later diagonal
  // block is complete; right: the right-hand sides), else one run over [j0, lda)
  const int nchL = SYM ? (m + 63) >> 6 : (int)((w + 63) >> 6);
  const int nchR = SYM ? (int)((lda - n + 63) >> 6) : 0;
  const int nch = nchL + nchR;
  const int ngr = (m + RH - 1) / RH;
  for (int it = warp; it < ngr * nch; it += nwarps) {
    const int gr = it / nch, ch = it - gr * nch;
    const int ib = j0 + RH * gr;
    const bool left = !SYM || ch < nchL;
    const int jbi = left ? j0 + 64 * ch : n + 64 * (ch - nchL);
    const int jend = !SYM ? ldi : (left ? n : ldi);
    if (SYM && left && jbi >= (((ib - k0) >> 5) << 5) + k0 + kLuNb) continue;  // strictly upper: never read
    const int ncol = jend - jbi < 64 ? jend - jbi : 64;
    double af[RT][kLuNb / 4];
    int coff[RT];
    unsigned rowok = 0;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int ia = ib + 8 * t + r8;
      const bool ok = ia < n;
#pragma unroll
      for (int s4 = 0; s4 < kLuNb / 4; ++s4) {
        const int k = 4 * s4 + q;
        // SYM, left of n: C -= (L21 D) L^T, the pivots folded into the L21 fragments
        const double v = (k < kb && ok) ? PT[(long long)k * n + ia] : 0.0;
        af[t][s4] = (SYM && left) ? v * dpiv[k] : v;
      }
      coff[t] = (ok ? ia : 0) * ldi + jbi + 2 * q;
      rowok |= (ok ? 1u : 0u) << t;
    }
    // B fragment (k = 4 s4 + q, column jbi + cj + r8): U12 from A, or (SYM, left of n)
    // L^T from the transposed panel
    const double *Bp = (SYM && left) ? PT + q * n + jbi + r8 : A + (k0 + q) * ldi + jbi + r8;
    const int bst = (SYM && left) ? 4 * n : 4 * ldi;
    const int kq = kb - q;  // fragment k = 4 s4 + q is valid while 4 s4 < kq
    double bf[kLuNb / 4], c[RT][2];
    auto load = [&](int cj, double *b, double (*cc)[2]) {
      const bool okb = jbi + cj + r8 < jend, ok0 = jbi + cj + 2 * q < jend, ok1 = jbi + cj + 2 * q + 1 < jend;
#pragma unroll
      for (int s4 = 0; s4 < kLuNb / 4; ++s4) b[s4] = (okb && 4 * s4 < kq) ? Bp[s4 * bst + cj] : 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const bool rk = (rowok >> t) & 1u;
        cc[t][0] = (rk && ok0) ? A[coff[t] + cj] : 0.0;
        cc[t][1] = (rk && ok1) ? A[coff[t] + cj + 1] : 0.0;
      }
    };
    load(0, bf, c);
#pragma unroll 1
    for (int cj = 0; cj < ncol; cj += 8) {
      double bn[kLuNb / 4], cn[RT][2];
      if (cj + 8 < ncol) load(cj + 8, bn, cn);
      double d[RT][2];
#pragma unroll
      for (int t = 0; t < RT; ++t) d[t][0] = d[t][1] = 0.0;
#pragma unroll
      for (int s4 = 0; s4 < kLuNb / 4; ++s4)
#pragma unroll
        for (int t = 0; t < RT; ++t) dmma(d[t][0], d[t][1], af[t][s4], bf[s4]);
      const bool ok0 = jbi + cj + 2 * q < jend, ok1 = jbi + cj + 2 * q + 1 < jend;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const bool rk = (rowok >> t) & 1u;
        if (rk && ok0) A[coff[t] + cj] = c[t][0] - d[t][0];
        if (rk && ok1) A[coff[t] + cj + 1] = c[t][1] - d[t][1];
      }
#pragma unroll
      for (int s4 = 0; s4 < kLuNb / 4; ++s4) bf[s4] = bn[s4];
#pragma unroll
      for (int t = 0; t < RT; ++t) { c[t][0] = cn[t][0]; c[t][1] = cn[t][1]; }
    }
  }
  __syncthreads();
  LUP(4)
}

// Block-strided copy dst[d(t)] = src[s(t)] for t = threadIdx.x + k blockDim.x < count,
// 8 loads issued before their 8 stores (source and destination share the workspace, so
// the compiler would not move a load above an earlier store); idx(t) -> {s(t), d(t)}.
template <class Idx>
__device__ __forceinline__ void lu_copy_batched(long long count, const double *src, double *dst, Idx idx) {
  const int T = blockDim.x;
  for (long long t0 = threadIdx.x; t0 < count; t0 += 8LL * T) {
    double v[8];
    long long d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long t = t0 + (long long)u * T;
      const longlong2 sd = idx(t < count ? t : 0);
      d[u] = sd.y;
      v[u] = t < count ? src[sd.x] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t0 + (long long)u * T < count) dst[d[u]] = v[u];
  }
}

// One cell of the LU path (the body of the persistent kernel below); A and PT live in
// this CTA's workspace slice ws.
// PIV = false: no row exchanges -- LU of an SPD matrix needs none (it is Cholesky with
// the diagonal kept in U); a pivot that is not positive sends the cell to the retry list
// for the pivoting pass (reading Q11's fallback, unchanged).
template <int kLuThreads, bool PIV>
__device__ __forceinline__ void lu_cell(Geom g, Strip st, const double2 *__restrict__ xy,
                                        const int *__restrict__ cell_start,
                                        const long long *__restrict__ x_off, double *__restrict__ X,
                                        const int cl, double *__restrict__ ws,
                                        int *__restrict__ fail_key, OvList ov,
                                        int *__restrict__ retry, int *__restrict__ nretry,
                                        double *pt_sm) {
  __shared__ Runs R;
  __shared__ double red_v[kLuThreads / 32];
  __shared__ int red_i[kLuThreads / 32];
  __shared__ int s_piv;
  __shared__ double Zs[kLuNb][kBsCols + 1];  // back substitution: the solved block Z_b
  __shared__ double L11[kLuNb][kLuNb + 1];
  __shared__ double prow[kLuNb];
  __shared__ double dpiv[kLuNb];  // the panel's pivots U(kk, kk) (no-pivot pass: U = D L^T)
  const int tid = threadIdx.x, T = blockDim.x;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  LUP0()
  if (tid == 0) sub_runs(g, cell_start, ov, cl, cx, cy, R);
  __syncthreads();
  const int n = R.n_ov, n_own = R.n_own, n0 = n - n_own, own_nat = R.own_nat_lo;
#ifdef RBF_PROBE
  if (tid == 0) {
    g_lu_acc[blockIdx.x][7] += 1;
    g_lu_acc[blockIdx.x][8] += n;
  }
#endif
  // right-hand sides: E_own (RASM), or the identity in natural order (ASM, reading Q26)
  const int nrhs = g.asm_full ? n : n_own;
  const long long lda = n + nrhs;
  double *A = ws;  // n x lda row-major: [A_c | E]
  // kLuNb x n: transposed panel, in dynamic shared memory when the launch gave it room
  double *PT = pt_sm ? pt_sm : A + (long long)n * lda;
  double2 *pos = reinterpret_cast<double2 *>(A + (((long long)n * lda + (long long)kLuNb * n + 1) & ~1LL));
  for (int p = tid; p < n; p += T) {
    const int q = (p < n0) ? (p < own_nat ? p : p + n_own) : own_nat + (p - n0);
    pos[p] = xy[nat_to_global(R, q) - st.ext_lo];
  }
  __syncthreads();
  // row by row (no 64-bit index division); the no-pivot pass assembles only what its
  // symmetric factorisation reads: the lower triangle and each row's diagonal block
  for (int i = 0; i < n; ++i) {
    const double2 pi = pos[i];
    double *Ai = A + (long long)i * lda;
    const int jn = PIV ? n : min(n, ((i >> 5) << 5) + kLuNb);
    for (int j = tid; j < jn; j += T) {
      const double dx = pi.x - pos[j].x, dy = pi.y - pos[j].y;
      const double r2 = fma(dx, dx, dy * dy);
      Ai[j] = (r2 < g.rc2) ? exp(r2 * g.neg_inv_2s2) * g.norm : 0.0;
    }
    for (int j = n + tid; j < lda; j += T) {  // column j - n = e_{natural index}, in factor order
      const int q = g.asm_full ? j - n : own_nat + (j - n);
      const int fq = q < own_nat ? q : (q < own_nat + n_own ? n0 + (q - own_nat) : q - n_own);
      Ai[j] = (i == fq) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  LUP(0)
  bool singular = false;
  for (int k0 = 0; k0 < n && !singular; k0 += kLuNb) {
    const int kb = n - k0 < kLuNb ? n - k0 : kLuNb;
    // ---- panel: PT[c][i] = A[i][k0 + c], rows i >= k0 (batched: A and PT share the
    //      workspace, so loads are not moved above earlier stores by the compiler)
    lu_copy_batched((long long)kb * (n - k0), A, PT, [&](long long t) {
      const int c = (int)t / (n - k0), i = k0 + (int)t - c * (n - k0);  // kb (n - k0) < 2^31
      return make_longlong2((long long)i * lda + k0 + c, (long long)c * n + i);
    });
    __syncthreads();
    for (int c = 0; c < kb; ++c) {
      const int kk = k0 + c;
      int p = kk;
      if (PIV) {
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = kk + tid; i < n; i += T) {
        const double v = fabs(PT[(long long)c * n + i]);
        if (v > best) { best = v; bi = i; }
      }
      lu_argmax(best, bi, red_v, red_i, &s_piv);
      p = s_piv;
      if (p < 0) { singular = true; break; }
      }
      if (PIV && p != kk) {  // swap rows kk and p: the panel copy and the rest of the augmented row
        for (int cc = tid; cc < kb; cc += T) {
          const double t0 = PT[(long long)cc * n + kk];
          PT[(long long)cc * n + kk] = PT[(long long)cc * n + p];
          PT[(long long)cc * n + p] = t0;
        }
        // right of the panel only (the L columns of earlier panels are never read
        // again: the right-hand sides are carried in A); four column pairs per pass
        for (long long j0s = k0 + kb + tid; j0s < lda; j0s += 4LL * T) {
          double x0[4], x1[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const long long j = j0s + (long long)u * T;
            x0[u] = j < lda ? A[(long long)kk * lda + j] : 0.0;
            x1[u] = j < lda ? A[(long long)p * lda + j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const long long j = j0s + (long long)u * T;
            if (j < lda) {
              A[(long long)kk * lda + j] = x1[u];
              A[(long long)p * lda + j] = x0[u];
            }
          }
        }
      }
      __syncthreads();
      if (tid < kb) prow[tid] = PT[(long long)tid * n + kk];  // pivot row, panel part
      __syncthreads();
      if (!PIV && !(prow[c] > 0.0)) { singular = true; break; }  // uniform: not SPD here
      const double inv = 1.0 / prow[c];
      for (int i = kk + 1 + tid; i < n; i += T) {
        // the row's panel values in groups of 8 loaded together: PT shares the workspace
        // with A, so the compiler would not move a load above the previous store (one L2
        // round trip per group instead of one per element)
        const double l = PT[(long long)c * n + i] * inv;
        PT[(long long)c * n + i] = l;
        for (int c8 = c + 1; c8 < kb; c8 += 8) {
          double rv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) rv[u] = c8 + u < kb ? PT[(long long)(c8 + u) * n + i] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c8 + u < kb) PT[(long long)(c8 + u) * n + i] = fma(-l, prow[c8 + u], rv[u]);
        }
      }
      __syncthreads();
    }
    LUP(1)
    if (singular) break;
    // write the factored panel back (L below the diagonal, U on and above it)
    lu_copy_batched((long long)kb * (n - k0), PT, A, [&](long long t) {
      const int c = (int)t / (n - k0), i = k0 + (int)t - c * (n - k0);
      return make_longlong2((long long)c * n + i, (long long)i * lda + k0 + c);
    });
    // L11 (unit lower) to shared memory, zero beyond kb: the unrolled solves below run
    // over all kLuNb rows and columns, and 0 * (stale shared memory) can be NaN
    for (int t = tid; t < kLuNb * kLuNb; t += T) {
      const int r = t / kLuNb, c = t - r * kLuNb;
      L11[r][c] = (c < r && r < kb) ? PT[(long long)c * n + k0 + r] : 0.0;
    }
    if (tid < kLuNb) dpiv[tid] = tid < kb ? PT[(long long)tid * n + k0 + tid] : 0.0;
    __syncthreads();
    LUP(2)
    // ---- U12 = L11^-1 A12, then A22 -= L21 U12 on the fp64 tensor cores
    lu_trailing_update<2, !PIV>(A, PT, L11, dpiv, n, lda, k0, kb);
  }
  LUP(4)
  if (singular) {
    if (tid == 0) {
      if (PIV) atomicMin(fail_key, cy * g.ncx + cx);
      else retry[atomicAdd(nretry, 1)] = cl;  // to the pivoting pass
    }
    return;
  }
  __syncthreads();
  // ---- back substitution U Z = Y on the nrhs right-hand-side columns (A[:, n:]), in
  //      chunks of kBsCols columns, blocks of kLuNb rows from the bottom: the diagonal
  //      block solved one column per thread (U block in shared memory), Z_b staged in
  //      shared memory, then every row above updated at once, Y[0:r0] -= U[0:r0, b] Z_b,
  //      on DMMA.8x8x4 (warps over 8-row tiles, U fragments in registers, the next
  //      column tile's Y values loaded before the current one's chain): three barriers
  //      per block instead of two per 64 rows above it
  for (int cb = 0; cb < nrhs; cb += kBsCols) {
    const int nc = nrhs - cb < kBsCols ? nrhs - cb : kBsCols;
    for (int r0 = ((n - 1) / kLuNb) * kLuNb; r0 >= 0; r0 -= kLuNb) {
      const int kb = n - r0 < kLuNb ? n - r0 : kLuNb;
      __syncthreads();
      for (int t = tid; t < kLuNb * kLuNb; t += T) {  // U block (upper incl. diagonal), zero beyond kb
        const int r = t / kLuNb, c = t - r * kLuNb;
        L11[r][c] = (c >= r && c < kb) ? A[(long long)(r0 + r) * lda + r0 + c] : 0.0;
      }
      __syncthreads();
      if (tid < kBsCols) {  // solve the diagonal block for this column; Z_b to shared memory
        const long long j = n + cb + tid;
        const bool act = tid < nc;
        double z[kLuNb];
#pragma unroll
        for (int t = 0; t < kLuNb; ++t) z[t] = (act && t < kb) ? A[(long long)(r0 + t) * lda + j] : 0.0;
#pragma unroll
        for (int r = kLuNb - 1; r >= 0; --r) {
          if (r < kb) {
            double a = z[r];
#pragma unroll
            for (int t = r + 1; t < kLuNb; ++t) a = fma(-L11[r][t], z[t], a);
            z[r] = a / L11[r][r];
          }
        }
#pragma unroll
        for (int t = 0; t < kLuNb; ++t) {
          Zs[t][tid] = z[t];  // 0 beyond kb and nc
          if (act && t < kb) A[(long long)(r0 + t) * lda + j] = z[t];
        }
      }
      __syncthreads();
      const int lane = tid & 31, warp = tid >> 5, nwarps = T >> 5, q = lane & 3, r8 = lane >> 2;
      for (int i0 = 8 * warp; i0 < r0; i0 += 8 * nwarps) {  // r0 is a multiple of 8
        const int ia = i0 + r8;
        double af[kLuNb / 4];
        // U(ia, r0 + k); no-pivot pass: U = D L^T, so D(ia) L(r0 + k, ia) (the strictly
        // upper part left of the right-hand sides is not kept up to date there)
        const double dia = PIV ? 1.0 : A[(long long)ia * lda + ia];
#pragma unroll
        for (int s4 = 0; s4 < kLuNb / 4; ++s4) {
          const int k = 4 * s4 + q;
          af[s4] = k < kb ? (PIV ? A[(long long)ia * lda + r0 + k] : dia * A[(long long)(r0 + k) * lda + ia]) : 0.0;
        }
        double *yrow = A + (long long)ia * lda + n + cb;
        auto ld = [&](int cj, double &c0, double &c1) {
          const int jc = cj + 2 * q;
          c0 = jc < nc ? yrow[jc] : 0.0;
          c1 = jc + 1 < nc ? yrow[jc + 1] : 0.0;
        };
        double c0, c1;
        ld(0, c0, c1);
        for (int cj = 0; cj < nc; cj += 8) {
          double n0 = 0.0, n1 = 0.0;
          if (cj + 8 < nc) ld(cj + 8, n0, n1);
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int s4 = 0; s4 < kLuNb / 4; ++s4) dmma(d0, d1, af[s4], Zs[4 * s4 + q][cj + r8]);
          const int jc = cj + 2 * q;
          if (jc < nc) yrow[jc] = c0 - d0;
          if (jc + 1 < nc) yrow[jc + 1] = c1 - d1;
          c0 = n0;
          c1 = n1;
        }
      }
    }
  }
  __syncthreads();
  LUP(5)
  const long long ld = (n + 1) & ~1;
  double *Xc = X + x_off[cl];
  for (long long t = tid; t < (long long)nrhs * ld; t += T) {  // row o: RHS column o
    const int o = (int)(t / ld), q = (int)(t - (long long)o * ld);
    double v = 0.0;
    if (q < n) {
      int pp;
      if (q < own_nat) pp = q;
      else if (q < own_nat + n_own) pp = n0 + (q - own_nat);
      else pp = q - n_own;
      v = A[(long long)pp * lda + n + o];
    }
    Xc[t] = v;
  }
  __syncthreads();
  LUP(6)
}

// Persistent LU kernel: one CTA per SM takes the cells of glist (sorted largest first)
// from an atomic counter, so the cell sizes (tens to thousands of points on clustered
// data) balance over the SMs in ONE launch, and the workspace is one slice per CTA.
template <int kLuThreads, bool PIV>
__global__ __launch_bounds__(kLuThreads, 512 / kLuThreads) void k_rasm_setup_lu(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, const int *__restrict__ glist,
    int count, double *__restrict__ ws, long long ws_stride, int *__restrict__ fail_key,
    OvList ov, int *__restrict__ next, int *__restrict__ retry, int *__restrict__ nretry, int pt_smem) {
  extern __shared__ double lu_dyn[];
  __shared__ int s_item;
  double *slice = ws + (long long)blockIdx.x * ws_stride;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= count) break;
    lu_cell<kLuThreads, PIV>(g, st, xy, cell_start, x_off, X, glist[item], slice, fail_key, ov, retry, nretry,
                             pt_smem ? lu_dyn : nullptr);
    __syncthreads();
  }
}

// sort keys of the LU cells: |Omega_c|, plus kLuBreakdown for the cells whose Cholesky
// broke down in the tensor-core pass (glist[n_nonfit:]), so those sort first
constexpr int kLuBreakdown = 1 << 24;
__global__ void k_lu_sizes(Geom g, Strip st, const int *__restrict__ cell_start, const int *__restrict__ glist,
                           int count, int n_nonfit, int *__restrict__ key, OvList ov) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int cl = glist[i];
  Runs R;
  sub_runs(g, cell_start, ov, cl, cl % g.ncx, st.row_lo + cl / g.ncx, R);
  key[i] = R.n_ov + (i >= n_nonfit ? kLuBreakdown : 0);
}

// z[own(c)] = X_c u[Omega_c]: one CTA per cell; u[Omega_c] gathered into shared
// memory once, then each warp streams whole rows of X_c with 16-byte loads (rows are
// 16-byte aligned: ld even, block offsets even), 4 loads in flight per lane.
// Direct-load variant: one CTA per cell.  Each warp issues the 16-byte loads of its
// first X row BEFORE the u[Omega_c] gather, and the next row's loads before the
// current row's reduction, so the HBM stream never waits on the gather.
__global__ __launch_bounds__(kRaThreads) void k_rasm_apply(
    Geom g, Strip st, const int *__restrict__ cell_start, const long long *__restrict__ x_off,
    const double *__restrict__ X, const double *__restrict__ u, double *__restrict__ z, OvList ov,
    int cl_split, int cl_skip) {
  extern __shared__ double su[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = (int)blockIdx.x < cl_split ? (int)blockIdx.x : (int)blockIdx.x + cl_skip;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  const int key = cy * g.ncx + cx;
  const int o0 = cell_start[key], n_own = cell_start[key + 1] - o0;
  if (n_own == 0) return;
  const long long nel = x_off[cl + 1] - x_off[cl];
  const int ld = (int)(nel / n_own), h = ld >> 1;
  const double2 *Xc = reinterpret_cast<const double2 *>(X + x_off[cl]);
  auto load4 = [&](int o, int c0, double2 *xv) {
    const double2 *row = Xc + (long long)o * h + c0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int j = lane + 32 * k;
      xv[k] = (o < n_own && c0 + j < h) ? __ldcs(row + j) : make_double2(0.0, 0.0);
    }
  };
  double2 xv[4];
  load4(warp, 0, xv);  // in flight during the gather below
  Runs R;
  sub_runs(g, cell_start, ov, cl, cx, cy, R);
  const int n = R.n_ov;
  for (int q = tid; q < ld; q += kRaThreads) su[q] = (q < n) ? u[nat_to_global(R, q) - st.ext_lo] : 0.0;
  __syncthreads();
  const double2 *u2 = reinterpret_cast<const double2 *>(su);
  for (int o = warp; o < n_own; o += kRaThreads / 32) {
    double acc = 0.0, acc2 = 0.0;
    for (int c0 = 0; c0 < h; c0 += 128) {
      if (c0 > 0) load4(o, c0, xv);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = c0 + lane + 32 * k;
        if (j < h) {
          const double2 uv = u2[j];
          acc = fma(xv[k].x, uv.x, acc);
          acc2 = fma(xv[k].y, uv.y, acc2);
        }
      }
    }
    load4(o + kRaThreads / 32, 0, xv);  // next row of this warp
    acc += acc2;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) z[o0 + o - st.own_lo] = acc;
  }
}

// ---------------------------------------------------------------------------
// Additive Schwarz, Eq.(8) (reading Q26): z = sum_c R_c^T A_c^-1 R_c u.
// (1) k_asm_local: t_c = A_c^-1 u[Omega_c] for every cell (all n_ov rows of the stored
//     inverse, the RASM GEMV with every row kept), into t at asm_toff[cl];
// (2) k_asm_gather: z_i = sum of the t entries of point i, in ascending cell order
//     (a CSR map built once at setup by a stable sort of (point, t index) pairs), so
//     the sums are deterministic and need no atomics.
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(kRaThreads) void k_asm_local(
    Geom g, Strip st, const int *__restrict__ cell_start, const long long *__restrict__ x_off,
    const long long *__restrict__ t_off, const double *__restrict__ X, const double *__restrict__ u,
    double *__restrict__ t, OvList ov) {
  extern __shared__ double su[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = blockIdx.x;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  Runs R;
  sub_runs(g, cell_start, ov, cl, cx, cy, R);
  if (R.n_own == 0) return;
  const int n = R.n_ov, ld = (n + 1) & ~1, h = ld >> 1;
  for (int q = tid; q < ld; q += kRaThreads) su[q] = (q < n) ? u[nat_to_global(R, q) - st.ext_lo] : 0.0;
  __syncthreads();
  const double2 *u2 = reinterpret_cast<const double2 *>(su);
  const double2 *Xc = reinterpret_cast<const double2 *>(X + x_off[cl]);
  double *tc = t + t_off[cl];
  for (int o = warp; o < n; o += kRaThreads / 32) {
    const double2 *row = Xc + (long long)o * h;
    double acc = 0.0, acc2 = 0.0;
    for (int j = lane; j < h; j += 32) {
      const double2 xv = __ldcs(row + j), uv = u2[j];
      acc = fma(xv.x, uv.x, acc);
      acc2 = fma(xv.y, uv.y, acc2);
    }
    acc += acc2;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) tc[o] = acc;
  }
}

// t sizes (n_ov, or 0 for an empty cell) of the cells of rows [row0, row0 + ncl_e / ncx):
// the strip's own rows plus, across strips, the `rings` rows on each side whose
// subdomains reach into the strip
__global__ void k_asm_tsizes(Geom g, Strip st, const int *__restrict__ cell_start, int row0, int ncl_e,
                             long long *__restrict__ tsizes, OvList ov) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e > ncl_e) return;
  if (e == ncl_e) { tsizes[e] = 0; return; }
  const int cy = row0 + e / g.ncx, cx = e % g.ncx;
  Runs R;  // box-overlap lists exist for the own cells only (ASM across strips needs whole rings)
  sub_runs(g, cell_start, ov, cy - st.row_lo >= 0 ? (cy - st.row_lo) * g.ncx + cx : 0, cx, cy, R);
  tsizes[e] = R.n_own ? R.n_ov : 0;
}

// (point, t index) pairs in (cell, position) order, for the stable sort by point; cells of
// rows [row0, ...) with t offsets t_off; points outside the strip get the key npts (sorted
// last, not summed)
__global__ void k_asm_entries(Geom g, Strip st, const int *__restrict__ cell_start, int row0,
                              const long long *__restrict__ t_off, long long npts, int *__restrict__ key,
                              int *__restrict__ val, OvList ov) {
  const int e = blockIdx.x;
  const int cy = row0 + e / g.ncx, cx = e % g.ncx;
  Runs R;
  sub_runs(g, cell_start, ov, cy - st.row_lo >= 0 ? (cy - st.row_lo) * g.ncx + cx : 0, cx, cy, R);
  if (R.n_own == 0) return;
  const long long o = t_off[e];
  for (int q = threadIdx.x; q < R.n_ov; q += blockDim.x) {
    const long long k = nat_to_global(R, q) - st.own_lo;
    key[o + q] = (int)(k >= 0 && k < npts ? k : npts);
    val[o + q] = (int)(o + q);
  }
}

// CSR offsets from the sorted keys: every point has >= 1 entry (its own cell); the keys
// npts (entries for other strips' points) are last and close the table
__global__ void k_asm_offsets(const int *__restrict__ skey, long long total, long long npts,
                              long long *__restrict__ poff) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k < total && (k == 0 || skey[k] != skey[k - 1]) && skey[k] <= npts) poff[skey[k]] = k;
  if (k == 0 && (total == 0 || skey[total - 1] < npts)) poff[npts] = total;
}

__global__ void k_asm_gather(const long long *__restrict__ poff, const int *__restrict__ map,
                             const double *__restrict__ t, long long npts, double *__restrict__ z) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= npts) return;
  double acc = 0.0;
  for (long long k = poff[i]; k < poff[i + 1]; ++k) acc += t[map[k]];
  z[i] = acc;
}

static OvList ov_of(const rbf_ctx *c) { return OvList{c->ov_idx, c->ov_off, c->ov_own}; }

static int build_asm_map(rbf_ctx *c, int ncl, long long total_own, cudaStream_t s) {
  const long long np = n_loc(c);
  const Geom &g = c->g;
  // across strips: the rings rows on each side whose subdomains reach into this strip
  const int nrows = c->s.row_hi - c->s.row_lo;
  const int rb = (c->nranks > 1 && c->rank > 0) ? g.rings : 0;
  const int ra = (c->nranks > 1 && c->rank < c->nranks - 1) ? g.rings : 0;
  const int row0 = c->s.row_lo - rb, ncl_e = (nrows + rb + ra) * g.ncx;
  ScratchGuard sg(s);
  long long *tsz = nullptr, *toff = nullptr;
  RBF_TRY(sg.alloc(c, &tsz, sizeof(long long) * (size_t)(ncl_e + 1)));
  RBF_TRY(sg.alloc(c, &toff, sizeof(long long) * (size_t)(ncl_e + 1)));
  k_asm_tsizes<<<(ncl_e + 256) / 256, 256, 0, s>>>(g, c->s, c->cell_start, row0, ncl_e, tsz, ov_of(c));
  size_t tb0 = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb0, tsz, toff, ncl_e + 1, s));
  void *tmp0 = nullptr;
  RBF_TRY(sg.alloc(c, &tmp0, tb0));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp0, tb0, tsz, toff, ncl_e + 1, s));
  // block boundaries: below | own | above, and the boundary rows sent to the neighbours
  long long hb[5] = {0, 0, 0, 0, 0};
  const int idx[5] = {rb * g.ncx, (rb + rb) * g.ncx, (rb + nrows - ra) * g.ncx, (rb + nrows) * g.ncx, ncl_e};
  for (int k = 0; k < 5; ++k)
    RBF_CUDA_TRY(cudaMemcpyAsync(&hb[k], toff + idx[k], sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  const long long sb = hb[0], so = hb[3] - hb[0], total = hb[4];
  if (so != total_own) {
    set_error("rbf_setup: ASM local-solution sizes disagree (%lld vs %lld)", so, total_own);
    return RBF_EINVAL;
  }
  if (total >= (1LL << 31)) {
    set_error("rbf_setup: ASM needs %lld local-solution entries (limit 2^31)", total);
    return RBF_EUNSUPPORTED;
  }
  c->asm_sb = sb;
  // t exchange: to rank - 1 the own first rb rows' t, from it the rb rows below; to rank + 1
  // the own last ra rows' t, from it the ra rows above (offsets: send in the own block,
  // receive in the whole buffer)
  c->halo_asm[0] = Halo{0, rb ? hb[1] - sb : 0, 0, sb};
  c->halo_asm[1] = Halo{ra ? hb[2] - sb : 0, ra ? hb[3] - hb[2] : 0, hb[3], total - hb[3]};
  int *key = nullptr, *val = nullptr, *skey = nullptr;
  RBF_TRY(sg.alloc(c, &key, sizeof(int) * (size_t)(total > 0 ? total : 1)));
  RBF_TRY(sg.alloc(c, &val, sizeof(int) * (size_t)(total > 0 ? total : 1)));
  RBF_TRY(sg.alloc(c, &skey, sizeof(int) * (size_t)(total > 0 ? total : 1)));
  RBF_TRY(dalloc(c, (void **)&c->asm_map, sizeof(int) * (size_t)(total > 0 ? total : 1), s));
  RBF_TRY(dalloc(c, (void **)&c->asm_poff, sizeof(long long) * (size_t)(np + 1), s));
  RBF_TRY(dalloc(c, (void **)&c->asm_t, sizeof(double) * (size_t)(total > 0 ? total : 1), s));
  k_asm_entries<<<ncl_e, 128, 0, s>>>(g, c->s, c->cell_start, row0, toff, np, key, val, ov_of(c));
  RBF_CUDA_TRY(cudaGetLastError());
  int end_bit = 1;
  while ((1LL << end_bit) <= np) ++end_bit;  // keys up to np (other strips' points)
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, skey, val, c->asm_map, (int)total, 0,
                                               end_bit, s));
  void *tmp = nullptr;
  RBF_TRY(sg.alloc(c, &tmp, tb));
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, key, skey, val, c->asm_map, (int)total, 0,
                                               end_bit, s));  // stable: cell order kept per point
  k_asm_offsets<<<(int)((total + 255) / 256) + 1, 256, 0, s>>>(skey, total, np, c->asm_poff);
  count_launch(6 + (end_bit + 7) / 8);
  RBF_CUDA_TRY(cudaGetLastError());
  (void)ncl;
  return RBF_OK;
}

int probe_read(long long *out) {
#ifdef RBF_PROBE
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out, g_probe, sizeof(long long) * 64 * 8));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8, g_trace, sizeof(long long) * 65536 * 3));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3, g_col, sizeof(long long) * 512));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3 + 512, g_wcol, sizeof(long long) * 128));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3 + 512 + 128, g_lu_acc, sizeof(long long) * 512 * 10));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3 + 512 + 128 + 5120, g_t2_acc, sizeof(long long) * 512 * 8));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3 + 512 + 128 + 5120 + 4096, g_t2_col, sizeof(long long) * 256));
  RBF_CUDA_TRY(cudaMemcpyFromSymbol(out + 64 * 8 + 65536 * 3 + 512 + 128 + 5120 + 4096 + 256, g_t2_w, sizeof(long long) * 256));
  return RBF_OK;
#else
  (void)out;
  set_error("built without RBF_PROBE");
  return RBF_EUNSUPPORTED;
#endif
}


// Box-overlap index lists (reading Q24): count, scan, fill.
static int build_ov_lists(rbf_ctx *c, int ncl, cudaStream_t s) {
  dfree(c->ov_idx, s);
  dfree(c->ov_off, s);
  dfree(c->ov_own, s);
  c->ov_idx = nullptr;
  long long *sizes = nullptr;
  RBF_TRY(dalloc(c, (void **)&sizes, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&c->ov_off, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&c->ov_own, sizeof(int) * (ncl > 0 ? ncl : 1), s));
  const int blocks = (ncl + 1 + 255) / 256;
  k_ov_lists<0><<<blocks, 256, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, ncl, sizes, nullptr,
                                       nullptr, nullptr);
  RBF_CUDA_TRY(cudaGetLastError());
  size_t tmp_bytes = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes, c->ov_off, ncl + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tmp_bytes, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, c->ov_off, ncl + 1, s));
  long long total = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, c->ov_off + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(tmp, s);
  dfree(sizes, s);
  RBF_TRY(dalloc(c, (void **)&c->ov_idx, sizeof(int) * (size_t)(total > 0 ? total : 1), s));
  k_ov_lists<1><<<blocks, 256, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, ncl, nullptr, c->ov_off,
                                       c->ov_idx, c->ov_own);
  count_launch(3);  // count, scan, fill
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

// Slot plans of k_rasm_setup_tc2 for every tile shape (T <= 29, T1 <= 4): the order in
// which the column loop forms tiles (column j: (j..T-1, j)) and retires them (in column
// j's panel step: row j+1's tiles (j+1, kt < j) and row j's (j, j-1), (j, j), rows of
// L11 only), each new tile taking the lowest free slot.  Uploaded once per device.
static void t2_plan(int T, int T1, unsigned char *rec) {
  std::memset(rec, 0, kT2Rec);
  if (T1 > T) return;
  const int T0 = T - T1;
  std::vector<int> slot(T * (T + 1) / 2, 0);
  std::vector<char> used(512, 0);
  int peak = 0;
  auto tix = [](int it, int jt) { return it * (it + 1) / 2 + jt; };
  for (int j = 0; j < T; ++j) {
    for (int it = j; it < T; ++it) {
      int sl = 0;
      while (used[sl]) ++sl;
      used[sl] = 1;
      slot[tix(it, j)] = sl;
      peak = std::max(peak, sl + 1);
    }
    if (j + 1 < T0)
      for (int kt = 0; kt < j; ++kt) used[slot[tix(j + 1, kt)]] = 0;
    if (j < T0) {
      if (j >= 1) used[slot[tix(j, j - 1)]] = 0;
      used[slot[tix(j, j)]] = 0;
    }
  }
  for (size_t i = 0; i < slot.size(); ++i) rec[i] = (unsigned char)std::min(slot[i], 255);
  int nfree = 0;
  for (int sl = 0; sl < kT2Cap; ++sl)
    if (!used[sl]) rec[kT2RecFree + nfree++] = (unsigned char)sl;
  int *pi = reinterpret_cast<int *>(rec + kT2RecPeak);
  pi[0] = peak;
  pi[1] = nfree;
}

static int t2_plans(const unsigned char **out) {
  static std::mutex mu;
  static std::map<int, unsigned char *> per_dev;
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  unsigned char *&d = per_dev[dev];
  if (!d) {
    std::vector<unsigned char> h((size_t)kT2Recs * kT2Rec);
    for (int T = 1; T <= kTcMaxTiles; ++T)
      for (int T1 = 1; T1 <= kT2MaxT1; ++T1) t2_plan(T, T1, h.data() + (size_t)t2_rec_index(T, T1) * kT2Rec);
    RBF_CUDA_TRY(cudaMalloc((void **)&d, h.size()));
    RBF_CUDA_TRY(cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice));
  }
  *out = d;
  return RBF_OK;
}

int rasm_setup(rbf_ctx *c, cudaStream_t s) {
  const int ncl = owned_cells(c);
  long long *sizes = nullptr;
  int *cnt = nullptr, *glist = nullptr;
  RBF_TRY(dalloc(c, (void **)&sizes, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&c->x_off, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&cnt, sizeof(int) * 8, s));
  RBF_TRY(dalloc(c, (void **)&glist, sizeof(int) * (ncl > 0 ? ncl : 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * 8, s));
  if (c->g.ovw > 0.0) RBF_TRY(build_ov_lists(c, ncl, s));
  const OvList ov = ov_of(c);
  long long *tsizes = nullptr;
  if (c->g.asm_full) {
    RBF_TRY(dalloc(c, (void **)&tsizes, sizeof(long long) * (ncl + 1), s));
    RBF_TRY(dalloc(c, (void **)&c->asm_toff, sizeof(long long) * (ncl + 1), s));
  }
  k_rasm_sizes<<<(ncl + 1 + 255) / 256, 256, 0, s>>>(c->g, c->s, c->cell_start, ncl, sizes, cnt,
                                                     glist, ov, tsizes);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  size_t tmp_bytes = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes, c->x_off, ncl + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tmp_bytes, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, c->x_off, ncl + 1, s));
  count_launch(2);  // init + scan
  long long asm_total = 0;
  if (c->g.asm_full) {
    RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, tsizes, c->asm_toff, ncl + 1, s));
    count_launch(2);
    RBF_CUDA_TRY(cudaMemcpyAsync(&asm_total, c->asm_toff + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  }
  int hc[8];
  long long total = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, c->x_off + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(tmp, s);
  dfree(sizes, s);
  dfree(tsizes, s);
  if (c->g.asm_full && ncl > 0) RBF_TRY(build_asm_map(c, ncl, asm_total, s));
  c->max_ov = hc[0];
  c->max_own = hc[1];
  c->nsub = hc[2];
  c->x_count = total;
  const int n_nonfit = hc[3];  // cells routed to LU by size (before the Cholesky breakdowns)
  RBF_TRY(dalloc(c, (void **)&c->X, sizeof(double) * (size_t)(total > 0 ? total : 2), s));
  if (ncl > 0 && c->nsub > hc[3]) {
    const size_t smem = (size_t)hc[4];  // the largest per-cell layout of the tensor-core cells
    const int skern = (int)opt(OPT_SETUP_KERNEL);
    if (skern == 1 || skern == 2) {
      // 1: two factorisations per SM; 2: factorisation and post phase pipelined on one SM.
      // The cells they cannot take (n_own > 32) are listed for the one-per-SM kernel.
      const unsigned char *plans = nullptr;
      RBF_TRY(t2_plans(&plans));
      int dev = 0, sms = 148, occ = 0;
      RBF_CUDA_TRY(cudaGetDevice(&dev));
      RBF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      if (skern == 1) {
        RBF_TRY(ensure_dyn_smem((const void *)k_rasm_setup_tc2, kT2Smem));
        RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rasm_setup_tc2, kT2Threads, kT2Smem));
      } else {
        RBF_TRY(ensure_dyn_smem((const void *)k_rasm_setup_tc3, kT3Smem));
        RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rasm_setup_tc3, kT3Threads, kT3Smem));
      }
      const int grid = std::max(1, std::min(ncl, std::max(occ, 1) * sms));
#ifdef RBF_PROBE
      fprintf(stderr, "[probe] k_rasm_setup_tc2/3: %d CTAs per SM, grid %d, %zu B dynamic shared memory\n", occ, grid,
              kT2Smem);
      {
        static long long zero[512 * 8];
        RBF_CUDA_TRY(cudaMemcpyToSymbolAsync(g_t2_acc, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s));
      }
#endif
      double *ws2 = nullptr;
      int *w2 = nullptr;
      RBF_TRY(dalloc(c, (void **)&ws2, sizeof(double) * 64 * (size_t)kT2WsTiles * grid * (skern == 2 ? 2 : 1), s));
      RBF_TRY(dalloc(c, (void **)&w2, sizeof(int) * (2 + (size_t)ncl), s));
      RBF_CUDA_TRY(cudaMemsetAsync(w2, 0, 2 * sizeof(int), s));
      if (skern == 1)
        k_rasm_setup_tc2<<<grid, kT2Threads, kT2Smem, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off, c->X,
                                                            cnt, glist, ov, plans, ws2, w2, w2 + 2, ncl);
      else
        k_rasm_setup_tc3<<<grid, kT3Threads, kT3Smem, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off, c->X,
                                                            cnt, glist, ov, plans, ws2, w2, w2 + 2, ncl);
      count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
      RBF_TRY(prebuild_solve(c, s));  // host work while the kernel runs (krylov.cu)
      int nd = 0;
      RBF_CUDA_TRY(cudaMemcpyAsync(&nd, w2 + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
      RBF_CUDA_TRY(cudaStreamSynchronize(s));
      if (nd > 0) {
        RBF_TRY(ensure_dyn_smem((const void *)k_rasm_setup_tc, smem));
        k_rasm_setup_tc<<<nd, kTcThreads, smem, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off, c->X, cnt,
                                                     glist, ov, w2 + 2);
        count_launch(1);
        RBF_CUDA_TRY(cudaGetLastError());
      }
      RBF_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
      RBF_CUDA_TRY(cudaStreamSynchronize(s));
      dfree(w2, s);
      dfree(ws2, s);
    } else {
      RBF_TRY(ensure_dyn_smem((const void *)k_rasm_setup_tc, smem));
      k_rasm_setup_tc<<<ncl, kTcThreads, smem, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off,
                                                    c->X, cnt, glist, ov, nullptr);
      count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
      // host work while the kernel runs: GMRES workspace and the solve graph (krylov.cu)
      RBF_TRY(prebuild_solve(c, s));
      RBF_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
      RBF_CUDA_TRY(cudaStreamSynchronize(s));
    }
  }
  const int nglobal = hc[3];  // big cells + Cholesky breakdowns (ASM: every cell)
  if (ncl > 0 && c->nsub == nglobal) RBF_TRY(prebuild_solve(c, s));  // no tensor-core pass
  int hfail = 0x7fffffff;
  if (nglobal > 0) {
    int *fail = cnt + 4;
    RBF_CUDA_TRY(cudaMemcpyAsync(fail, &hfail, sizeof(int), cudaMemcpyHostToDevice, s));
    const long long no = c->max_own;
    // largest subdomains first (longest-processing-time order for the work queue), ties
    // by cell index: glist's order comes from atomics, so it is sorted by cell first (the
    // radix sort is stable) and the probe wave below is the same cells on every run
    int *keys = nullptr, *skeys = nullptr, *sorted = nullptr, *keys2 = nullptr, *cells2 = nullptr;
    int *next = cnt + 5;
    RBF_TRY(dalloc(c, (void **)&keys, sizeof(int) * nglobal, s));
    RBF_TRY(dalloc(c, (void **)&skeys, sizeof(int) * nglobal, s));
    RBF_TRY(dalloc(c, (void **)&sorted, sizeof(int) * nglobal, s));
    RBF_TRY(dalloc(c, (void **)&keys2, sizeof(int) * nglobal, s));
    RBF_TRY(dalloc(c, (void **)&cells2, sizeof(int) * nglobal, s));
    k_lu_sizes<<<(nglobal + 255) / 256, 256, 0, s>>>(c->g, c->s, c->cell_start, glist, nglobal, n_nonfit,
                                                      keys, ov);
    size_t tb = 0, tb2 = 0;
    RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, glist, cells2, keys, keys2, nglobal, 0, 32, s));
    RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb2, keys2, skeys, cells2, sorted, nglobal, 0,
                                                           32, s));
    tb = std::max(tb, tb2);
    void *tmp = nullptr;
    RBF_TRY(dalloc(c, &tmp, tb, s));
    RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, glist, cells2, keys, keys2, nglobal, 0, 32, s));
    RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, keys2, skeys, cells2, sorted, nglobal, 0,
                                                           32, s));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Cholesky breakdowns (numerically indefinite A_c, sorted first): partial pivoting
    // right away.  The cells routed here by size: a pass without row exchanges (SPD
    // subdomains), then the pivoting pass for those whose pivots were not all positive.
    // Each pass: 512 threads one CTA per SM if its largest cell exceeds kLuBigN points,
    // else 256 threads two per SM.
    std::vector<int> hk(nglobal);
    RBF_CUDA_TRY(cudaMemcpyAsync(hk.data(), skeys, sizeof(int) * nglobal, cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    int nbd = 0;
    while (nbd < nglobal && hk[nbd] >= kLuBreakdown) ++nbd;
    const int nsz = nglobal - nbd;
    const long long n_bd = nbd > 0 ? hk[0] - kLuBreakdown : 0, n_sz = nsz > 0 ? hk[nbd] : 0;
    auto stride_of = [&](long long nn) {
      const long long oo = no < nn ? no : nn;  // rows of X_c <= |Omega_c|
      return (((nn * (nn + oo) + (long long)kLuNb * nn + 1) & ~1LL) + 2 * nn + 1) & ~1LL;
    };
    auto grid_of = [&](long long nn, int cnt_) {
      const int per_sm = nn > kLuBigN ? 1 : 2;
      return cnt_ < per_sm * sms ? cnt_ : per_sm * sms;
    };
    const int probe = grid_of(n_sz, nsz), rest = nsz - probe;  // see the no-pivot probe below
    const long long n_rest = rest > 0 ? hk[nbd + probe] : 0;
    const long long wsz = std::max({stride_of(n_bd) * grid_of(n_bd, nbd), stride_of(n_sz) * grid_of(n_sz, nsz),
                                    stride_of(n_rest) * grid_of(n_rest, rest)});
    double *ws = nullptr;
    RBF_TRY(dalloc(c, (void **)&ws, sizeof(double) * (size_t)(wsz > 0 ? wsz : 1), s));
    int *retry = keys, *nretry = cnt + 6;  // keys are free after the sort
    // the transposed panel (kLuNb x n, re-read and re-written once per panel column) in
    // dynamic shared memory whenever that keeps the CTAs per SM of the global-memory
    // layout; option lu_smem_panel = 0 keeps it in the workspace (A/B knob)
    const bool sm_panel = opt(OPT_LU_SMEM_PANEL) != 0;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    auto launch = [&](auto kern, int threads, bool with_retry, const int *list, int count, long long nn) -> int {
      int grid = grid_of(nn, count);
      size_t dyn = 0;
      if (sm_panel) {
        const size_t need = sizeof(double) * kLuNb * (size_t)nn;
        cudaFuncAttributes fa;
        RBF_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
        if (need + fa.sharedSizeBytes <= (size_t)optin) {
          RBF_TRY(ensure_dyn_smem((const void *)kern, need));
          int occ = 0;
          RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, need));
          if (occ >= (nn > kLuBigN ? 1 : 2)) dyn = need;
        }
      }
      RBF_CUDA_TRY(cudaMemsetAsync(next, 0, sizeof(int), s));
      kern<<<grid, threads, dyn, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off, c->X, list, count, ws,
                                      stride_of(nn), fail, ov, next, with_retry ? retry : nullptr,
                                      with_retry ? nretry : nullptr, dyn > 0);
      count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
      return RBF_OK;
    };
    auto pass = [&](bool piv, const int *list, int count, long long nn) -> int {
      if (nn > kLuBigN)
        return piv ? launch(k_rasm_setup_lu<512, true>, 512, false, list, count, nn)
                   : launch(k_rasm_setup_lu<512, false>, 512, true, list, count, nn);
      return piv ? launch(k_rasm_setup_lu<256, true>, 256, false, list, count, nn)
                 : launch(k_rasm_setup_lu<256, false>, 256, true, list, count, nn);
    };
    if (nbd > 0) RBF_TRY(pass(true, sorted, nbd, n_bd));
    const bool nopiv = opt(OPT_LU_NOPIV) != 0;  // 0: pivot every LU cell (A/B knob)
    int hretry = 0;
    bool rest_piv = false;
    if (nsz > 0 && !nopiv) RBF_TRY(pass(true, sorted + nbd, nsz, n_sz));
    if (nsz > 0 && nopiv) {
      // probe: the largest cells, one wave, without pivoting.  If more than a quarter of
      // them need pivoting the data is numerically indefinite at this size and the rest
      // take the pivoting pass directly.  The decision depends only on the data, so the
      // factors (and every result) are reproducible run to run.
      RBF_CUDA_TRY(cudaMemsetAsync(nretry, 0, sizeof(int), s));
      RBF_TRY(pass(false, sorted + nbd, probe, n_sz));
      RBF_CUDA_TRY(cudaMemcpyAsync(&hretry, nretry, sizeof(int), cudaMemcpyDeviceToHost, s));
      RBF_CUDA_TRY(cudaStreamSynchronize(s));
      rest_piv = 4 * hretry > probe;
      if (rest_piv) {
        // one pivoting pass over the probe's failed cells (the largest) followed by the
        // rest, so that the largest cells start first (longest-processing-time order)
        // instead of forming a last wave of their own
        if (rest > 0)
          RBF_CUDA_TRY(cudaMemcpyAsync(retry + hretry, sorted + nbd + probe, sizeof(int) * (size_t)rest,
                                       cudaMemcpyDeviceToDevice, s));
        if (hretry + rest > 0) RBF_TRY(pass(true, retry, hretry + rest, hretry > 0 ? n_sz : n_rest));
      } else {
        if (rest > 0) RBF_TRY(pass(false, sorted + nbd + probe, rest, n_rest));
        if (rest > 0) {
          RBF_CUDA_TRY(cudaMemcpyAsync(&hretry, nretry, sizeof(int), cudaMemcpyDeviceToHost, s));
          RBF_CUDA_TRY(cudaStreamSynchronize(s));
        }
        if (hretry > 0) RBF_TRY(pass(true, retry, hretry, n_sz));
      }
    }
    c->n_lu_pivot = nbd + (nopiv ? hretry + (rest_piv ? rest : 0) : nsz);  // cells factored with partial pivoting
    count_launch(9);  // sizes, two sorts
    RBF_CUDA_TRY(cudaGetLastError());
    dfree(tmp, s);
    dfree(keys, s);
    dfree(skeys, s);
    dfree(sorted, s);
    dfree(keys2, s);
    dfree(cells2, s);
    RBF_CUDA_TRY(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    dfree(ws, s);
  }
  c->n_lu = nglobal;
  dfree(cnt, s);
  dfree(glist, s);
  if (hfail != 0x7fffffff) {
    set_error("rbf_setup: subdomain matrix A_c is singular (zero pivot in LU with partial "
              "pivoting) in cell %d (cx=%d, cy=%d)", hfail, hfail % c->g.ncx, hfail / c->g.ncx);
    return RBF_EFACTOR;
  }
  return RBF_OK;
}

int launch_asm_local(const rbf_ctx *c, const double *r_ext, cudaStream_t s) {
  const int ncl = owned_cells(c);
  if (ncl <= 0 || c->nsub == 0) return RBF_OK;
  const size_t smem = sizeof(double) * (size_t)(c->max_ov + 2);
  RBF_TRY(ensure_dyn_smem((const void *)k_asm_local, smem));
  k_asm_local<<<ncl, kRaThreads, smem, s>>>(c->g, c->s, c->cell_start, c->x_off, c->asm_toff, c->X, r_ext,
                                            c->asm_t + c->asm_sb, ov_of(c));
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_asm_gather(const rbf_ctx *c, double *z_loc, cudaStream_t s) {
  const long long np = n_loc(c);
  if (np <= 0) return RBF_OK;
  k_asm_gather<<<(int)((np + 255) / 256), 256, 0, s>>>(c->asm_poff, c->asm_map, c->asm_t, np, z_loc);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_rasm_apply(const rbf_ctx *c, const double *r_ext, double *z_loc, cudaStream_t s, int part) {
  const int ncl = owned_cells(c);
  if (ncl <= 0 || c->nsub == 0) return RBF_OK;
  const size_t smem = sizeof(double) * (size_t)(c->max_ov + 2);
  if (c->g.asm_full) {  // Eq.(8): local solutions, then the per-point sums (one strip; across
                        // strips dist_rasm_apply exchanges the boundary rows' t in between)
    if (part == 2) return RBF_OK;
    RBF_TRY(launch_asm_local(c, r_ext, s));
    return launch_asm_gather(c, z_loc, s);
  }
  // cell rows next to a strip edge with a neighbour rank read the halo (rings rows)
  const int nrows = c->s.row_hi - c->s.row_lo, ncx = c->g.ncx;
  int rb = (c->nranks > 1 && c->rank > 0) ? c->g.rings : 0;
  int ra = (c->nranks > 1 && c->rank < c->nranks - 1) ? c->g.rings : 0;
  rb = rb < nrows ? rb : nrows;
  ra = ra < nrows - rb ? ra : nrows - rb;
  int grid = ncl, split = ncl, skip = 0;
  if (part == 1) {
    grid = (nrows - ra - rb) * ncx;
    split = 0;
    skip = rb * ncx;
  } else if (part == 2) {
    grid = (rb + ra) * ncx;
    split = rb * ncx;
    skip = (nrows - ra - rb) * ncx;
  }
  if (grid <= 0) return RBF_OK;
  RBF_TRY(ensure_dyn_smem((const void *)k_rasm_apply, smem));
  k_rasm_apply<<<grid, kRaThreads, smem, s>>>(c->g, c->s, c->cell_start, c->x_off, c->X, r_ext, z_loc,
                                              ov_of(c), split, skip);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

}  // namespace rbf
