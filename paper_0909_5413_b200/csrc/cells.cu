// cells.cu -- GPU cell-list build (index sets of P:250, 268).
//
// key = cy*ncx + cx with cx = clamp(floor((x-x0)/c), 0, ncx-1) computed with IEEE
// division (reading Q5), then a stable LSD radix sort of (key, caller index) with
// CUB, cell_start by boundary detection, and a gather of the sorted positions as
// double2 (16-byte aligned, one LDG.128 per point in the matvec).
#include <cub/cub.cuh>

#include "common.cuh"

namespace rbf {

__device__ __forceinline__ int cell_coord(double v, double v0, double c, int ncells) {
  double t = floor(__ddiv_rn(__dsub_rn(v, v0), c));
  t = fmax(t, 0.0);
  t = fmin(t, (double)(ncells - 1));
  return (int)t;
}

__global__ void k_cell_keys(const double *__restrict__ xy, int n, Geom g, int *__restrict__ keys,
                            int *__restrict__ vals, int *__restrict__ bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = xy[2 * (long long)i], y = xy[2 * (long long)i + 1];
  bool ok = isfinite(x) && isfinite(y) && x >= g.x0 && x <= g.x1 && y >= g.y0 && y <= g.y1;
  if (!ok) atomicMin(bad, i);
  int cx = ok ? cell_coord(x, g.x0, g.cell, g.ncx) : 0;
  int cy = ok ? cell_coord(y, g.y0, g.cell, g.ncy) : 0;
  keys[i] = cy * g.ncx + cx;
  vals[i] = i;
}

// cell_start[k] = first sorted position with key >= k (ncells+1 entries).
__global__ void k_cell_start(const int *__restrict__ skeys, int n, int ncells,
                             int *__restrict__ cell_start) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int k1 = skeys[s];
  int k0 = (s == 0) ? -1 : skeys[s - 1];
  for (int k = k0 + 1; k <= k1; ++k) cell_start[k] = s;
  if (s == n - 1)
    for (int k = k1 + 1; k <= ncells; ++k) cell_start[k] = n;
}

// Sorted positions (fp64, double2).
__global__ void k_gather_xy(const double *__restrict__ xy, const int *__restrict__ perm,
                            long long lo, long long cnt, double2 *__restrict__ out) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  long long i = perm[lo + t];
  out[t] = make_double2(xy[2 * i], xy[2 * i + 1]);
}

__global__ void k_max_cell(const int *__restrict__ cell_start, int ncells, int *__restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  int v = (k < ncells) ? cell_start[k + 1] - cell_start[k] : 0;
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(out, v);
}

__global__ void k_row_start(const int *__restrict__ cell_start, int ncx, int ncy,
                            long long *__restrict__ out) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > ncy) return;
  out[r] = cell_start[(long long)r * ncx];
}

__global__ void k_to_local(const double *__restrict__ vc, const int *__restrict__ perm,
                           long long own_lo, long long cnt, double *__restrict__ vl) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < cnt) vl[t] = vc[perm[own_lo + t]];
}

__global__ void k_from_local(const double *__restrict__ vl, const int *__restrict__ perm,
                             long long own_lo, long long cnt, double *__restrict__ vc) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < cnt) vc[perm[own_lo + t]] = vl[t];
}

__global__ void k_local_index(const int *__restrict__ perm, long long own_lo, long long cnt,
                              int64_t *__restrict__ idx) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < cnt) idx[t] = perm[own_lo + t];
}

static int blocks_for(long long n, int t) { return (int)((n + t - 1) / t); }

// Coincident points (reading Q30): equal coordinates fall into the same cell, so each
// cell compares its points pairwise; out[0] = the smallest caller index that repeats an
// earlier point, out[1] = the caller index it repeats (lowest such pair).
__global__ void k_dup_check(const double *__restrict__ xy, const int *__restrict__ perm,
                            const int *__restrict__ cell_start, int ncells,
                            unsigned long long *__restrict__ out) {
  for (int cl = blockIdx.x; cl < ncells; cl += gridDim.x) {
    const int s0 = cell_start[cl], s1 = cell_start[cl + 1];
    for (int a = s0 + (int)threadIdx.x; a < s1; a += blockDim.x) {
      const int ia = perm[a];
      const double xa = xy[2LL * ia], ya = xy[2LL * ia + 1];
      for (int b = a + 1; b < s1; ++b) {
        const int ib = perm[b];
        if (xy[2LL * ib] == xa && xy[2LL * ib + 1] == ya) {
          const unsigned lo = ia < ib ? ia : ib, hi = ia < ib ? ib : ia;
          atomicMin(out, ((unsigned long long)hi << 32) | lo);
        }
      }
    }
  }
}

int build_cell_list(rbf_ctx *c, const double *xy, cudaStream_t s) {
  const int n = (int)c->n;
  const int ncells = c->g.ncx * c->g.ncy;
  int *keys = nullptr, *vals = nullptr, *skeys = nullptr, *bad = nullptr;
  RBF_TRY(dalloc(c, (void **)&keys, sizeof(int) * n, s));
  RBF_TRY(dalloc(c, (void **)&vals, sizeof(int) * n, s));
  RBF_TRY(dalloc(c, (void **)&skeys, sizeof(int) * n, s));
  RBF_TRY(dalloc(c, (void **)&bad, sizeof(int) * 2, s));
  RBF_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int) * 2, s));
  RBF_TRY(dalloc(c, (void **)&c->perm, sizeof(int) * n, s));
  RBF_TRY(dalloc(c, (void **)&c->cell_start, sizeof(int) * ((size_t)ncells + 1), s));
  int init_bad = 0x7fffffff;
  RBF_CUDA_TRY(cudaMemcpyAsync(bad, &init_bad, sizeof(int), cudaMemcpyHostToDevice, s));
  k_cell_keys<<<blocks_for(n, 256), 256, 0, s>>>(xy, n, c->g, keys, vals, bad); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  int end_bit = 1;
  while ((1LL << end_bit) < (long long)ncells) ++end_bit;
  size_t tmp_bytes = 0;
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, skeys, vals, c->perm, n,
                                               0, end_bit, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tmp_bytes, s));
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, skeys, vals, c->perm, n, 0,
                                               end_bit, s));
  count_launch(1 + (end_bit + 7) / 8);  // onesweep: histogram + one pass per 8-bit digit
  k_cell_start<<<blocks_for(n, 256), 256, 0, s>>>(skeys, n, ncells, c->cell_start); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  // row starts (host copy drives the strip plan and the halo ranges)
  long long *rs = nullptr;
  RBF_TRY(dalloc(c, (void **)&rs, sizeof(long long) * (c->g.ncy + 1), s));
  k_row_start<<<blocks_for(c->g.ncy + 1, 256), 256, 0, s>>>(c->cell_start, c->g.ncx, c->g.ncy, rs); count_launch(1);
  k_max_cell<<<blocks_for(ncells, 256), 256, 0, s>>>(c->cell_start, ncells, bad + 1);
  count_launch(1);
  unsigned long long *dup = nullptr, hdup = ~0ULL;
  RBF_TRY(dalloc(c, (void **)&dup, sizeof(unsigned long long), s));
  RBF_CUDA_TRY(cudaMemsetAsync(dup, 0xff, sizeof(unsigned long long), s));
  k_dup_check<<<ncells < 4096 ? ncells : 4096, 128, 0, s>>>(xy, c->perm, c->cell_start, ncells, dup);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  RBF_CUDA_TRY(cudaMemcpyAsync(&hdup, dup, sizeof(hdup), cudaMemcpyDeviceToHost, s));
  int hmax = 0;
  c->row_start.assign(c->g.ncy + 1, 0);
  int hbad = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(c->row_start.data(), rs, sizeof(long long) * (c->g.ncy + 1),
                               cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&hmax, bad + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  c->max_cell = hmax;
  dfree(tmp, s);
  dfree(keys, s);
  dfree(vals, s);
  dfree(skeys, s);
  dfree(bad, s);
  dfree(rs, s);
  dfree(dup, s);
  if (hbad != 0x7fffffff) {
    set_error("rbf_setup: point %d is non-finite or outside the box [%g,%g]x[%g,%g]", hbad,
              c->g.x0, c->g.x1, c->g.y0, c->g.y1);
    return RBF_EINVAL;
  }
  if (hdup != ~0ULL) {
    set_error("rbf_setup: points %u and %u coincide (the interpolation matrix is singular for "
              "repeated nodes; SPEC S:53)", (unsigned)(hdup & 0xffffffffULL), (unsigned)(hdup >> 32));
    return RBF_EINVAL;
  }
  return RBF_OK;
}

int gather_positions(rbf_ctx *c, const double *xy, cudaStream_t s) {
  long long cnt = c->s.ext_hi - c->s.ext_lo;
  RBF_TRY(dalloc(c, (void **)&c->xy_ext, sizeof(double2) * (size_t)(cnt > 0 ? cnt : 1), s));
  if (cnt > 0) {
    k_gather_xy<<<blocks_for(cnt, 256), 256, 0, s>>>(xy, c->perm, c->s.ext_lo, cnt, c->xy_ext);
    count_launch(1);
    RBF_CUDA_TRY(cudaGetLastError());
  }
  return RBF_OK;
}

int launch_to_local(const rbf_ctx *c, const double *vc, double *vl, cudaStream_t s) {
  long long cnt = n_loc(c);
  if (cnt > 0) {
    k_to_local<<<blocks_for(cnt, 256), 256, 0, s>>>(vc, c->perm, c->s.own_lo, cnt, vl);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_from_local(const rbf_ctx *c, const double *vl, double *vc, cudaStream_t s) {
  long long cnt = n_loc(c);
  if (cnt > 0) {
    k_from_local<<<blocks_for(cnt, 256), 256, 0, s>>>(vl, c->perm, c->s.own_lo, cnt, vc);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_local_index(const rbf_ctx *c, int64_t *idx, cudaStream_t s) {
  long long cnt = n_loc(c);
  if (cnt > 0) {
    k_local_index<<<blocks_for(cnt, 256), 256, 0, s>>>(c->perm, c->s.own_lo, cnt, idx);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

// In-cutoff pair count of the owned rows (diagnostics / Gpairs/s denominator).
__global__ void k_count_pairs(Geom g, Strip st, const double2 *__restrict__ xy,
                              const int *__restrict__ cell_start,
                              unsigned long long *__restrict__ out) {
  int cl = blockIdx.x;
  int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  int key = cy * g.ncx + cx;
  int t0 = cell_start[key], t1 = cell_start[key + 1];
  int bx0 = max(cx - g.kh, 0), bx1 = min(cx + g.kh, g.ncx - 1);
  int by0 = max(cy - g.kh, 0), by1 = min(cy + g.kh, g.ncy - 1);
  unsigned long long cnt = 0;
  const CellBox tb = cell_box(g, cx, cy, g.tw);  // T-box rows (reading Q25)
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    double2 p = xy[t - st.ext_lo];
    for (int by = by0; by <= by1; ++by) {
      int s0 = cell_start[by * g.ncx + bx0], s1 = cell_start[by * g.ncx + bx1 + 1];
      for (int q = s0; q < s1; ++q) {
        double2 o = xy[q - st.ext_lo];
        double dx = p.x - o.x, dy = p.y - o.y;
        if (g.tw > 0.0 ? in_box(tb, o.x, o.y) : fma(dx, dx, dy * dy) < g.rc2) ++cnt;
      }
    }
  }
  if (cnt) atomicAdd(out, cnt);
}

int count_pairs(rbf_ctx *c, long long *out, cudaStream_t s) {
  unsigned long long *d = nullptr, h = 0;
  RBF_TRY(dalloc(c, (void **)&d, sizeof(unsigned long long), s));
  RBF_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
  int nc = owned_cells(c);
  if (nc > 0) {
    k_count_pairs<<<nc, 64, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, d);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  RBF_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(d, s);
  *out = (long long)h;
  return RBF_OK;
}

// Strip cost of each cell row (cfg5's cluster core must be split by work,
// not by points): per cell, n_own (0.28 S + n_ov) scaled by 25 to integers, where S is
// the number of points in the matvec stencil (about 0.28 S of them within rc: pairs) and
// n_ov the subdomain size (the RASM apply streams n_own n_ov entries of X); one pair and
// one X entry cost about the same (FP64-bound matvec vs HBM-bound apply).  Integer sums,
// so every rank computes the same partition.
__global__ void k_row_costs(Geom g, const int *__restrict__ cell_start, unsigned long long *__restrict__ cost) {
  const long long cl = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (cl >= (long long)g.ncx * g.ncy) return;
  const int cy = (int)(cl / g.ncx), cx = (int)(cl - (long long)cy * g.ncx);
  const long long own = cell_start[cl + 1] - cell_start[cl];
  if (own == 0) return;
  auto box = [&](int k) {
    long long n = 0;
    const int x0 = max(cx - k, 0), x1 = min(cx + k, g.ncx - 1);
    for (int y = max(cy - k, 0); y <= min(cy + k, g.ncy - 1); ++y)
      n += cell_start[y * g.ncx + x1 + 1] - cell_start[y * g.ncx + x0];
    return n;
  };
  atomicAdd(&cost[cy], (unsigned long long)(own * (7 * box(g.kh) + 25 * box(g.rings > 0 ? g.rings : 1))));
}

int row_costs(rbf_ctx *c, cudaStream_t s, std::vector<long long> &out) {
  const Geom &g = c->g;
  out.assign(g.ncy, 0);
  unsigned long long *d = nullptr;
  ScratchGuard sg(s);
  RBF_TRY(sg.alloc(c, &d, sizeof(unsigned long long) * (size_t)g.ncy));
  RBF_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * (size_t)g.ncy, s));
  const long long ncl = (long long)g.ncx * g.ncy;
  k_row_costs<<<(int)((ncl + 255) / 256), 256, 0, s>>>(g, c->cell_start, d);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  RBF_CUDA_TRY(cudaMemcpyAsync(out.data(), d, sizeof(long long) * (size_t)g.ncy, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  return RBF_OK;
}

}  // namespace rbf
