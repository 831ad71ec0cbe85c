// matvec.cu -- fp64 cutoff-Gaussian matvec (Eq.(12)).
//
//   y_i = norm * sum_{j : fma(dx,dx,dy*dy) < rc^2} w_j exp(-r2_ij / (2 sigma^2))
//
// over the (2kh+1)^2 cell stencil around the target's cell (row-major keys make it
// 2kh+1 contiguous runs of the sorted arrays).
//
// The truncated operator is applied matrix-free in its VALUES (every entry is
// recomputed, "without actually storing the matrix"), but its sparsity
// pattern -- which of the stencil's sources lie within rc of each target -- is
// found once in rbf_setup (exact fp64 test) and kept as an ELLPACK-style list of
// 32-bit source indices, 4 bytes per in-cutoff pair (O(N) storage).  A matvec then
// spends its FP64 pipe only on in-cutoff pairs: one warp per chunk of <= 32 targets
// of a cell, lanes walk their own lists in lock step (coalesced list loads, gathers
// of the sources from L1/L2), table-driven exp on the FP64 pipe.
//
// The per-target summation order is the stencil order (rows, then sorted order),
// independent of the strip decomposition: results are deterministic and bitwise
// identical for any number of strips (reading Q20).
#include <cub/cub.cuh>

#include "common.cuh"

namespace rbf {

constexpr int kMvWarps = 4;  // target chunks per CTA
constexpr int kMvThreads = 32 * kMvWarps;
constexpr int kPad = -1;

// exp_neg()'s constants in the constant bank, so the DFMAs read them as c[][]
// operands instead of re-materialising 64-bit immediates in every iteration.
__constant__ double kExpC[8] = {6755399441055744.0,   92.33248261689366,
                                -0.010830417275428772, -7.420820373486988e-09,
                                1.0 / 120.0,           1.0 / 24.0,
                                1.0 / 6.0,             0.5};

__device__ __forceinline__ double exp_neg_smem(double x, const double *tab) {
  // exp_neg() without the underflow guard (rbf_setup requires rc <= 37 sigma, so
  // every in-range argument is > -685) and with the table in shared memory.
  const double t = fma(x, kExpC[1], kExpC[0]);
  const double kd = t - kExpC[0];
  const int k = __double2loint(t);
  double r = fma(kd, kExpC[2], x);
  r = fma(kd, kExpC[3], r);
  double p = fma(r, kExpC[4], kExpC[5]);
  p = fma(r, p, kExpC[6]);
  p = fma(r, p, kExpC[7]);
  p = fma(r, p, 1.0);
  p = r * p;
  const double T = tab[k & 63];
  const double e = fma(T, p, T);
  return __hiloint2double(__double2hiint(e) + ((k >> 6) << 20), __double2loint(e));
}

// ---------------------------------------------------------------------------
// Neighbour-list build (setup).  Chunks: ceil(n_t / 32) per owned cell.
// ---------------------------------------------------------------------------
__global__ void k_chunk_count(Geom g, Strip st, const int *__restrict__ cell_start, int ncl,
                              int *__restrict__ nchunk) {
  int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl > ncl) return;
  if (cl == ncl) {
    nchunk[cl] = 0;
    return;
  }
  const int key = (st.row_lo + cl / g.ncx) * g.ncx + cl % g.ncx;
  nchunk[cl] = (cell_start[key + 1] - cell_start[key] + 31) / 32;
}

__global__ void k_chunk_fill(const int *__restrict__ chunk_first, int ncl,
                             int *__restrict__ chunk_cell) {
  int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl) return;
  for (int c = chunk_first[cl]; c < chunk_first[cl + 1]; ++c) chunk_cell[c] = cl;
}

// MODE 0: per-chunk list length (max over lanes); MODE 1: write the entries.
template <int MODE>
__global__ __launch_bounds__(kMvThreads) void k_nlist(
    Geom g, Strip st, const double2 *__restrict__ xy, const int *__restrict__ cell_start,
    const int *__restrict__ chunk_cell, const int *__restrict__ chunk_first, int nchunks,
    int *__restrict__ chunk_len, const long long *__restrict__ chunk_off,
    int *__restrict__ list) {
  const int lane = threadIdx.x & 31;
  const int ch = blockIdx.x * kMvWarps + (threadIdx.x >> 5);
  if (ch >= nchunks) return;
  const int cl = chunk_cell[ch];
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  const int key = cy * g.ncx + cx;
  const int t = cell_start[key] + 32 * (ch - chunk_first[cl]) + lane;
  const bool active = t < cell_start[key + 1];
  const int bx0 = max(cx - g.kh, 0), bx1 = min(cx + g.kh, g.ncx - 1);
  const int by0 = max(cy - g.kh, 0), by1 = min(cy + g.kh, g.ncy - 1);
  const double2 *xye = xy - st.ext_lo;
  const double2 p = xye[active ? t : cell_start[key]];
  int cnt = 0;
  long long base = 0;
  if (MODE == 1) base = chunk_off[ch];
  for (int by = by0; by <= by1; ++by) {
    const int s0 = cell_start[by * g.ncx + bx0], s1 = cell_start[by * g.ncx + bx1 + 1];
    for (int s = s0; s < s1; ++s) {
      const double2 o = xye[s];
      const double dx = p.x - o.x, dy = p.y - o.y;
      if (active && fma(dx, dx, dy * dy) < g.rc2) {
        if (MODE == 1) list[base + ((long long)(cnt >> 2) * 32 + lane) * 4 + (cnt & 3)] = s;
        ++cnt;
      }
    }
  }
  const int kmax = (__reduce_max_sync(0xffffffffu, cnt) + 3) & ~3;  // groups of 4
  if (MODE == 0) {
    if (lane == 0) chunk_len[ch] = kmax;
  } else {
    for (int k = cnt; k < kmax; ++k) list[base + ((long long)(k >> 2) * 32 + lane) * 4 + (k & 3)] = kPad;
  }
}

__global__ void k_len_to_entries(const int *__restrict__ len, int n, long long *__restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = 32LL * len[i];
}

// ---------------------------------------------------------------------------
// The matvec: one warp per target chunk, lanes walk their lists in lock step.
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(kMvThreads) void k_matvec_ell(
    Geom g, Strip st, const double2 *__restrict__ xy, const double *__restrict__ w,
    const int *__restrict__ cell_start, const int *__restrict__ chunk_cell,
    const int *__restrict__ chunk_first, int nchunks, const int *__restrict__ chunk_len,
    const long long *__restrict__ chunk_off, const int *__restrict__ list,
    double *__restrict__ y) {
  __shared__ double s_tab[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 64) s_tab[threadIdx.x] = kExp2Tab64[threadIdx.x];
  __syncthreads();
  const int ch = blockIdx.x * kMvWarps + warp;
  if (ch >= nchunks) return;
  const int cl = chunk_cell[ch];
  const int key = (st.row_lo + cl / g.ncx) * g.ncx + cl % g.ncx;
  const int t = cell_start[key] + 32 * (ch - chunk_first[cl]) + lane;
  const bool active = t < cell_start[key + 1];
  const double2 *xye = xy - st.ext_lo;
  const double *we = w - st.ext_lo;
  const int self = active ? t : cell_start[key];
  const double2 p = xye[self];
  const int K = chunk_len[ch];  // multiple of 4
  const int4 *lp = reinterpret_cast<const int4 *>(list + chunk_off[ch]) + lane;
  const double nscale = g.neg_inv_2s2;
  double acc = 0.0;
  // 4 entries per 16-byte load, the next group prefetched; padding entries point at
  // the target itself with weight 0, so the loop is branch-free with 4 pairs in flight.
  int4 nxt = (K > 0) ? __ldcs(lp) : make_int4(kPad, kPad, kPad, kPad);
  for (int k = 0; k < K; k += 4) {
    const int4 ev = nxt;
    if (k + 4 < K) nxt = __ldcs(lp + ((k >> 2) + 1) * 32);
    const int es[4] = {ev.x, ev.y, ev.z, ev.w};
    double2 o[4];
    double wq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int src = es[u] < 0 ? self : es[u];
      o[u] = xye[src];
      wq[u] = es[u] < 0 ? 0.0 : we[src];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double dx = p.x - o[u].x, dy = p.y - o[u].y;
      const double r2 = fma(dx, dx, dy * dy);
      acc = fma(wq[u], exp_neg_smem(r2 * nscale, s_tab), acc);
    }
  }
  if (active) y[t - st.own_lo] = acc * g.norm;
}

int build_nlist(rbf_ctx *c, cudaStream_t s) {
  const int ncl = owned_cells(c);
  if (ncl <= 0) return RBF_OK;
  int *first = nullptr;
  RBF_TRY(dalloc(c, (void **)&first, sizeof(int) * (ncl + 1), s));
  k_chunk_count<<<(ncl + 1 + 255) / 256, 256, 0, s>>>(c->g, c->s, c->cell_start, ncl, first);
  count_launch(1);
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, first, first, ncl + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tb, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, first, first, ncl + 1, s));
  count_launch(2);
  int nch = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&nch, first + ncl, sizeof(int), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(tmp, s);
  c->nchunks = nch;
  c->chunk_first = first;
  RBF_TRY(dalloc(c, (void **)&c->chunk_cell, sizeof(int) * (nch > 0 ? nch : 1), s));
  RBF_TRY(dalloc(c, (void **)&c->chunk_len, sizeof(int) * (nch > 0 ? nch : 1), s));
  RBF_TRY(dalloc(c, (void **)&c->chunk_off, sizeof(long long) * (nch + 1), s));
  if (nch == 0) return RBF_OK;
  k_chunk_fill<<<(ncl + 255) / 256, 256, 0, s>>>(first, ncl, c->chunk_cell);
  count_launch(1);
  const int blocks = (nch + kMvWarps - 1) / kMvWarps;
  k_nlist<0><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->chunk_cell,
                                           first, nch, c->chunk_len, nullptr, nullptr);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  // offsets (in entries) = exclusive scan of 32 * len
  long long *w64 = nullptr;
  RBF_TRY(dalloc(c, (void **)&w64, sizeof(long long) * (nch + 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(w64 + nch, 0, sizeof(long long), s));
  k_len_to_entries<<<(nch + 255) / 256, 256, 0, s>>>(c->chunk_len, nch, w64);
  count_launch(1);
  tb = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, w64, c->chunk_off, nch + 1, s));
  RBF_TRY(dalloc(c, &tmp, tb, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, w64, c->chunk_off, nch + 1, s));
  count_launch(2);
  long long total = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, c->chunk_off + nch, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(tmp, s);
  dfree(w64, s);
  c->nlist_entries = total;
  RBF_TRY(dalloc(c, (void **)&c->nlist, sizeof(int) * (size_t)(total > 0 ? total : 1), s));
  k_nlist<1><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, c->chunk_cell,
                                           first, nch, c->chunk_len, c->chunk_off, c->nlist);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_matvec(const rbf_ctx *c, const double *w_ext, double *y_loc, cudaStream_t s) {
  if (c->nchunks <= 0) return RBF_OK;
  k_matvec_ell<<<(c->nchunks + kMvWarps - 1) / kMvWarps, kMvThreads, 0, s>>>(
      c->g, c->s, c->xy_ext, w_ext, c->cell_start, c->chunk_cell, c->chunk_first, c->nchunks,
      c->chunk_len, c->chunk_off, c->nlist, y_loc);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

}  // namespace rbf
