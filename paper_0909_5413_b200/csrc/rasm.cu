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

#include "common.cuh"

namespace rbf {

constexpr int kMaxRuns = 15;   // rings <= 7
constexpr int kRsThreads = 256;
constexpr int kRaThreads = 128;

struct Runs {
  int n;                 // number of runs (block rows inside the grid)
  int lo[kMaxRuns];      // global sorted start of each run
  int len[kMaxRuns];
  int n_ov, n_own, own_nat_lo;
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
  for (int r = 0; r < R.n; ++r) {
    const int by = by0 + r;
    R.lo[r] = cell_start[by * g.ncx + bx0];
    R.len[r] = cell_start[by * g.ncx + bx1 + 1] - R.lo[r];
    if (by == cy) R.own_nat_lo = R.n_ov + (cell_start[key] - R.lo[r]);
    R.n_ov += R.len[r];
  }
  R.n_own = cell_start[key + 1] - cell_start[key];
}

__device__ __forceinline__ int nat_to_global(const Runs &R, int q) {
  int r = 0;
  while (q >= R.len[r]) { q -= R.len[r]; ++r; }
  return R.lo[r] + q;
}

__device__ __forceinline__ long long tri(int i) { return (long long)i * (i + 1) / 2; }

// flat index f of a lower triangle (row a >= col b) -> (a, b)
__device__ __forceinline__ void tri_index(int f, int &a, int &b) {
  a = (int)((sqrtf(8.0f * (float)f + 1.0f) - 1.0f) * 0.5f);
  while ((long long)a * (a + 1) / 2 > f) --a;
  while ((long long)(a + 1) * (a + 2) / 2 <= f) ++a;
  b = f - a * (a + 1) / 2;
}

// Shared-memory layout for one subdomain of n points, n_own own points.
struct SetupSmem {
  size_t off_B, off_pos, off_gidx, total;
  __host__ __device__ SetupSmem(int n, int n_own) {
    size_t a = (size_t)n * (n + 1) / 2 * sizeof(double);
    off_B = a;
    size_t b = off_B + (size_t)n_own * n_own * sizeof(double);
    off_pos = (b + 15) & ~(size_t)15;
    off_gidx = off_pos + (size_t)n * sizeof(double2);
    total = off_gidx + (size_t)n * sizeof(int);
  }
};

// Per owned cell: X block size, maxima, and the list of cells whose factor does
// not fit in shared memory (they go to the global-memory LU kernel).
__global__ void k_rasm_sizes(Geom g, Strip st, const int *__restrict__ cell_start, int ncl,
                             size_t smem_limit, long long *__restrict__ sizes,
                             int *__restrict__ maxes, int *__restrict__ glist) {
  int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl) {
    if (cl == ncl) sizes[cl] = 0;
    return;
  }
  int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  Runs R;
  block_runs(g, cell_start, cx, cy, R);
  long long ld = (R.n_ov + 1) & ~1;
  sizes[cl] = R.n_own ? (long long)R.n_own * ld : 0;
  if (R.n_own) {
    atomicMax(&maxes[0], R.n_ov);
    atomicMax(&maxes[1], R.n_own);
    atomicAdd(&maxes[2], 1);
    if (SetupSmem(R.n_ov, R.n_own).total > smem_limit) glist[atomicAdd(&maxes[3], 1)] = cl;
  }
}

__global__ __launch_bounds__(kRsThreads) void k_rasm_setup(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, size_t smem_limit,
    int *__restrict__ counts, int *__restrict__ glist) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Runs R;
  const int tid = threadIdx.x, T = blockDim.x;
  const int cl = blockIdx.x;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  if (tid == 0) block_runs(g, cell_start, cx, cy, R);
  __syncthreads();
  const int n = R.n_ov, n_own = R.n_own, n0 = n - n_own;
  if (n_own == 0) return;
  const int own_nat = R.own_nat_lo;
  SetupSmem L(n, n_own);
  if (L.total > smem_limit) return;  // handled by k_rasm_setup_lu
  double *A = reinterpret_cast<double *>(smem);
  double *B = reinterpret_cast<double *>(smem + L.off_B);
  double2 *pos = reinterpret_cast<double2 *>(smem + L.off_pos);

  // factor order p -> natural order q: own(c) moved to the end
  for (int p = tid; p < n; p += T) {
    int q = (p < n0) ? (p < own_nat ? p : p + n_own) : own_nat + (p - n0);
    pos[p] = xy[nat_to_global(R, q) - st.ext_lo];
  }
  __syncthreads();
  // A_c = R_c A_rc R_c^T, packed lower triangle (reading Q10)
  {
    const int warp = tid >> 5, lane = tid & 31, nw = T >> 5;
    for (int i = warp; i < n; i += nw) {
      const double2 pi = pos[i];
      for (int j = lane; j <= i; j += 32) {
        const double2 pj = pos[j];
        const double dx = pi.x - pj.x, dy = pi.y - pj.y;
        const double r2 = fma(dx, dx, dy * dy);
        A[tri(i) + j] = (r2 < g.rc2) ? exp(r2 * g.neg_inv_2s2) * g.norm : 0.0;
      }
    }
  }
  for (int t = tid; t < n_own * n_own; t += T) B[t] = ((t / n_own) == (t % n_own)) ? 1.0 : 0.0;
  __syncthreads();

  // Right-looking Cholesky, one barrier per column: step k updates the trailing
  // triangle with a_ik a_jk / d_k (column k still unscaled) and finalises
  // column k-1 (not read in step k).
  bool failed = false;
  double l_prev_inv = 0.0;
  for (int k = 0; k < n; ++k) {
    const double d = A[tri(k) + k];
    if (!(d > 0.0)) { failed = true; break; }  // uniform: every thread reads the same d
    const double inv_d = 1.0 / d;
    const int m = n - 1 - k;
    const int nt = m * (m + 1) / 2;
    if (nt > 0) {
      int a, b;
      tri_index(tid, a, b);
      for (int f = tid; f < nt; f += T) {
        const int i = k + 1 + a, j = k + 1 + b;
        A[tri(i) + j] -= A[tri(i) + k] * A[tri(j) + k] * inv_d;
        b += T;
        while (b > a) { b -= a + 1; ++a; }
      }
    }
    if (k > 0) {  // finalise column k-1
      for (int i = k + tid; i < n; i += T) A[tri(i) + k - 1] *= l_prev_inv;
      if (tid == 0) A[tri(k - 1) + k - 1] = 1.0 / l_prev_inv;
    }
    const double l = sqrt(d);
    l_prev_inv = 1.0 / l;
    __syncthreads();
  }
  if (failed) {  // Cholesky broke down: redo this cell with LU (reading Q11)
    if (tid == 0) glist[atomicAdd(&counts[3], 1)] = cl;
    return;
  }
  if (tid == 0) A[tri(n - 1) + n - 1] = 1.0 / l_prev_inv;
  __syncthreads();

  // W = L21 L11^-1 in place over L21 (rows n0.., cols ..n0), column j finished at
  // step j and scaled one step later.
  for (int j = n0 - 1; j >= 0; --j) {
    const double inv = 1.0 / A[tri(j) + j];
    const int nt = n_own * j;
    for (int f = tid; f < nt; f += T) {
      const int r = f / j, kk = f - r * j;
      const long long row = tri(n0 + r);
      A[row + kk] -= A[row + j] * inv * A[tri(j) + kk];
    }
    if (j + 1 < n0) {
      const double inv1 = 1.0 / A[tri(j + 1) + j + 1];
      for (int r = tid; r < n_own; r += T) A[tri(n0 + r) + j + 1] *= inv1;
    }
    __syncthreads();
  }
  if (n0 > 0) {
    const double inv0 = 1.0 / A[0];
    for (int r = tid; r < n_own; r += T) A[tri(n0 + r) + 0] *= inv0;
  }
  __syncthreads();

  // Columns of S^-1 [-W, I]: per column, L22 y = b then L22^T x = y.
  for (int p = tid; p < n; p += T) {
    // column storage: W part in A (row n0+r, col p), identity part in B (row r, col p-n0)
    const bool wpart = p < n0;
    const long long bcol = p - n0;
    auto colp = [&](int r) -> double & {
      return wpart ? A[tri(n0 + r) + p] : B[(long long)r * n_own + bcol];
    };
    for (int r = 0; r < n_own; ++r) {
      double s = wpart ? -colp(r) : colp(r);
      const long long row = tri(n0 + r) + n0;
      for (int c2 = 0; c2 < r; ++c2) s -= A[row + c2] * colp(c2);
      colp(r) = s / A[row + r];
    }
    for (int r = n_own - 1; r >= 0; --r) {
      double s = colp(r);
      for (int c2 = r + 1; c2 < n_own; ++c2) s -= A[tri(n0 + c2) + n0 + r] * colp(c2);
      colp(r) = s / A[tri(n0 + r) + n0 + r];
    }
  }
  __syncthreads();

  // X_c[o][q] (natural column order), ld = n rounded up to even
  const long long ld = (n + 1) & ~1;
  double *Xc = X + x_off[cl];
  for (int o = 0; o < n_own; ++o) {
    for (int q = tid; q < ld; q += T) {
      double v = 0.0;
      if (q < n) {
        int p;
        if (q < own_nat) p = q;
        else if (q < own_nat + n_own) p = n0 + (q - own_nat);
        else p = q - n_own;
        v = (p < n0) ? A[tri(n0 + o) + p] : B[(long long)o * n_own + (p - n0)];
      }
      Xc[o * ld + q] = v;
    }
  }
}

// Global-memory local solve for subdomains whose factor does not fit in shared
// memory, and for cells whose Cholesky broke down (reading Q11): LU with partial
// pivoting (largest |a|, lowest row on ties) of the full A_c in factor order, then
// A_c Z = E_own by forward/back substitution; X_c = Z^T.  One CTA per cell, the
// matrix lives in a per-CTA slice of a global workspace (L2-resident).
constexpr int kLuThreads = 512;

__global__ __launch_bounds__(kLuThreads) void k_rasm_setup_lu(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const long long *__restrict__ x_off, double *__restrict__ X, const int *__restrict__ glist,
    int first, int count, double *__restrict__ ws, long long ws_stride, int *__restrict__ fail_key) {
  __shared__ Runs R;
  __shared__ double red_v[kLuThreads / 32];
  __shared__ int red_i[kLuThreads / 32];
  __shared__ int s_piv;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  if ((int)blockIdx.x >= count) return;
  const int cl = glist[first + blockIdx.x];
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  if (tid == 0) block_runs(g, cell_start, cx, cy, R);
  __syncthreads();
  const int n = R.n_ov, n_own = R.n_own, n0 = n - n_own, own_nat = R.own_nat_lo;
  double *A = ws + (long long)blockIdx.x * ws_stride;  // n x n row-major
  double *Z = A + (long long)n * n;                    // n x n_own row-major
  double2 *pos = reinterpret_cast<double2 *>(A + (((long long)n * n + (long long)n * n_own + 1) & ~1LL));
  for (int p = tid; p < n; p += T) {
    int q = (p < n0) ? (p < own_nat ? p : p + n_own) : own_nat + (p - n0);
    pos[p] = xy[nat_to_global(R, q) - st.ext_lo];
  }
  __syncthreads();
  for (long long t = tid; t < (long long)n * n; t += T) {
    const int i = (int)(t / n), j = (int)(t - (long long)i * n);
    const double dx = pos[i].x - pos[j].x, dy = pos[i].y - pos[j].y;
    const double r2 = fma(dx, dx, dy * dy);
    A[t] = (r2 < g.rc2) ? exp(r2 * g.neg_inv_2s2) * g.norm : 0.0;
  }
  for (long long t = tid; t < (long long)n * n_own; t += T) {
    const int i = (int)(t / n_own), r = (int)(t - (long long)i * n_own);
    Z[t] = (i == n0 + r) ? 1.0 : 0.0;  // E_own in factor order
  }
  __syncthreads();
  bool singular = false;
  for (int k = 0; k < n; ++k) {
    // pivot: largest |A[i][k]|, i >= k, lowest index on ties
    double best = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += T) {
      const double v = fabs(A[(long long)i * n + k]);
      if (v > best) { best = v; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (v2 > best || (v2 == best && i2 < bi)) { best = v2; bi = i2; }
    }
    if (lane == 0) { red_v[warp] = best; red_i[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = red_v[0];
      int ii = red_i[0];
      for (int w = 1; w < T / 32; ++w)
        if (red_v[w] > b || (red_v[w] == b && red_i[w] < ii)) { b = red_v[w]; ii = red_i[w]; }
      s_piv = (b > 0.0) ? ii : -1;
    }
    __syncthreads();
    const int p = s_piv;
    if (p < 0) { singular = true; break; }
    if (p != k) {  // swap rows k and p of A and of the right-hand sides
      for (int j = tid; j < n; j += T) {
        const double t = A[(long long)k * n + j];
        A[(long long)k * n + j] = A[(long long)p * n + j];
        A[(long long)p * n + j] = t;
      }
      for (int r = tid; r < n_own; r += T) {
        const double t = Z[(long long)k * n_own + r];
        Z[(long long)k * n_own + r] = Z[(long long)p * n_own + r];
        Z[(long long)p * n_own + r] = t;
      }
    }
    __syncthreads();
    const double inv = 1.0 / A[(long long)k * n + k];
    const int m = n - 1 - k;
    for (long long t = tid; t < (long long)m * (m + n_own); t += T) {
      const int i = k + 1 + (int)(t / (m + n_own));
      const int jj = (int)(t % (m + n_own));
      const double l = A[(long long)i * n + k] * inv;
      if (jj < m) A[(long long)i * n + k + 1 + jj] -= l * A[(long long)k * n + k + 1 + jj];
      else Z[(long long)i * n_own + (jj - m)] -= l * Z[(long long)k * n_own + (jj - m)];
    }
    __syncthreads();
  }
  if (singular) {
    if (tid == 0) atomicMin(fail_key, cy * g.ncx + cx);
    return;
  }
  // back substitution U Z = (L^-1 P E_own), column-oriented
  for (int k = n - 1; k >= 0; --k) {
    const double inv = 1.0 / A[(long long)k * n + k];
    __syncthreads();
    for (int r = tid; r < n_own; r += T) Z[(long long)k * n_own + r] *= inv;
    __syncthreads();
    for (long long t = tid; t < (long long)k * n_own; t += T) {
      const int i = (int)(t / n_own), r = (int)(t - (long long)i * n_own);
      Z[(long long)i * n_own + r] -= A[(long long)i * n + k] * Z[(long long)k * n_own + r];
    }
  }
  __syncthreads();
  const long long ld = (n + 1) & ~1;
  double *Xc = X + x_off[cl];
  for (long long t = tid; t < (long long)n_own * ld; t += T) {
    const int o = (int)(t / ld), q = (int)(t - (long long)o * ld);
    double v = 0.0;
    if (q < n) {
      int pp;
      if (q < own_nat) pp = q;
      else if (q < own_nat + n_own) pp = n0 + (q - own_nat);
      else pp = q - n_own;
      v = Z[(long long)pp * n_own + o];
    }
    Xc[t] = v;
  }
}

__global__ __launch_bounds__(kRaThreads) void k_rasm_apply_v1(
    Geom g, Strip st, const int *__restrict__ cell_start, const long long *__restrict__ x_off,
    const double *__restrict__ X, const double *__restrict__ u, double *__restrict__ z) {
  extern __shared__ double su[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = blockIdx.x;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  Runs R;
  block_runs(g, cell_start, cx, cy, R);
  if (R.n_own == 0) return;
  const int n = R.n_ov;
  for (int q = tid; q < n; q += kRaThreads) su[q] = u[nat_to_global(R, q) - st.ext_lo];
  __syncthreads();
  const long long ld = (n + 1) & ~1;
  const double *Xc = X + x_off[cl];
  const int o0 = cell_start[cy * g.ncx + cx];
  for (int o = warp; o < R.n_own; o += kRaThreads / 32) {
    double acc = 0.0;
    for (int q = lane; q < n; q += 32) acc = fma(Xc[o * ld + q], su[q], acc);
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
    if (lane == 0) z[o0 + o - st.own_lo] = acc;
  }
}

int rasm_setup(rbf_ctx *c, cudaStream_t s) {
  const int ncl = owned_cells(c);
  int dev = 0, smem_optin = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  RBF_CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  RBF_CUDA_TRY(cudaFuncGetAttributes(&fa, k_rasm_setup));
  const size_t smem_limit = (size_t)smem_optin - fa.sharedSizeBytes;  // dynamic part
  long long *sizes = nullptr;
  int *cnt = nullptr, *glist = nullptr;
  RBF_TRY(dalloc(c, (void **)&sizes, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&c->x_off, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&cnt, sizeof(int) * 8, s));
  RBF_TRY(dalloc(c, (void **)&glist, sizeof(int) * (ncl > 0 ? ncl : 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * 8, s));
  k_rasm_sizes<<<(ncl + 1 + 255) / 256, 256, 0, s>>>(c->g, c->s, c->cell_start, ncl, smem_limit,
                                                     sizes, cnt, glist); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  size_t tmp_bytes = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes, c->x_off, ncl + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tmp_bytes, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, sizes, c->x_off, ncl + 1, s));
  count_launch(2);  // init + scan
  int hc[8];
  long long total = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, c->x_off + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(tmp, s);
  dfree(sizes, s);
  c->max_ov = hc[0];
  c->max_own = hc[1];
  c->nsub = hc[2];
  c->x_count = total;
  RBF_TRY(dalloc(c, (void **)&c->X, sizeof(double) * (size_t)(total > 0 ? total : 2), s));
  if (ncl > 0 && c->nsub > 0 && hc[3] < c->nsub) {
    SetupSmem L(c->max_ov, c->max_own);
    size_t smem = L.total < smem_limit ? L.total : smem_limit;
    RBF_CUDA_TRY(cudaFuncSetAttribute(k_rasm_setup, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    k_rasm_setup<<<ncl, kRsThreads, smem, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off,
                                               c->X, smem, cnt, glist); count_launch(1);
    RBF_CUDA_TRY(cudaGetLastError());
    RBF_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
  }
  const int nglobal = hc[3];  // big cells + Cholesky breakdowns
  int hfail = 0x7fffffff;
  if (nglobal > 0) {
    int *fail = cnt + 4;
    RBF_CUDA_TRY(cudaMemcpyAsync(fail, &hfail, sizeof(int), cudaMemcpyHostToDevice, s));
    const long long n = c->max_ov, no = c->max_own;
    const long long stride = (((n * n + n * no + 1) & ~1LL) + 2 * n + 1) & ~1LL;
    const long long budget = 4LL << 30;  // bytes of workspace per batch
    long long batch = budget / (stride * 8);
    if (batch < 1) batch = 1;
    if (batch > nglobal) batch = nglobal;
    double *ws = nullptr;
    RBF_TRY(dalloc(c, (void **)&ws, sizeof(double) * (size_t)(stride * batch), s));
    for (int first = 0; first < nglobal; first += (int)batch) {
      int count = nglobal - first < batch ? nglobal - first : (int)batch;
      k_rasm_setup_lu<<<count, kLuThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->x_off,
                                                   c->X, glist, first, count, ws, stride, fail); count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
    }
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

int launch_rasm_apply(const rbf_ctx *c, const double *r_ext, double *z_loc, cudaStream_t s) {
  const int ncl = owned_cells(c);
  if (ncl <= 0 || c->nsub == 0) return RBF_OK;
  size_t smem = sizeof(double) * (size_t)c->max_ov;
  k_rasm_apply_v1<<<ncl, kRaThreads, smem, s>>>(c->g, c->s, c->cell_start, c->x_off, c->X, r_ext,
                                                z_loc); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

}  // namespace rbf
