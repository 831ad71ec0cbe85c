// evaluate.cu -- interpolant evaluation at query points:
//
//   s(q) = norm * sum_{j : |q - x_j| < rc} lambda_j exp(-|q - x_j|^2 / (2 sigma^2))
//
// (with the T-box of reading Q25: j in the query cell's box grown by trunc_width)
//
// the RBF interpolant of Eq.(1) with the Gaussian of Eq.(12) and the
// truncation of reading Q1 -- the paper's application, interpolation from
// scattered points onto a lattice.
//
// The queries are binned into the context's cell grid (CUB radix sort of their
// cell keys), so a warp of consecutive sorted queries walks the same (2kh+1)
// contiguous source runs of the cell-sorted records {x, y, lambda} (one 256-bit
// gather per candidate, L1-resident across the warp), tests the exact fp64
// cutoff and accumulates in ascending source order with the matvec's table-free
// exp: at a data point the result is bitwise the matvec row.
#include <cub/cub.cuh>

#include "common.cuh"

namespace rbf {

__global__ void k_query_keys(const double *__restrict__ q, long long m, Geom g, int *__restrict__ keys,
                             int *__restrict__ vals, long long *__restrict__ bad) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const double x = q[2 * k], y = q[2 * k + 1];
  const bool ok = isfinite(x) && isfinite(y) && x >= g.x0 && x <= g.x1 && y >= g.y0 && y <= g.y1;
  if (!ok) atomicMin((unsigned long long *)bad, (unsigned long long)k);
  int cx = 0, cy = 0;
  if (ok) {
    cx = (int)fmin(fmax(floor(__ddiv_rn(__dsub_rn(x, g.x0), g.cell)), 0.0), (double)(g.ncx - 1));
    cy = (int)fmin(fmax(floor(__ddiv_rn(__dsub_rn(y, g.y0), g.cell)), 0.0), (double)(g.ncy - 1));
  }
  keys[k] = cy * g.ncx + cx;
  vals[k] = (int)k;
}

__global__ __launch_bounds__(256) void k_evaluate(Geom g, const double *__restrict__ q, long long m,
                                                   const int *__restrict__ skeys,
                                                   const int *__restrict__ order,
                                                   const int *__restrict__ cell_start,
                                                   const double4 *__restrict__ rec,
                                                   double *__restrict__ s) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int k = order[t], key = skeys[t];
  const int cx = key % g.ncx, cy = key / g.ncx;
  const double qx = q[2LL * k], qy = q[2LL * k + 1];
  const int bx0 = max(cx - g.kh, 0), bx1 = min(cx + g.kh, g.ncx - 1);
  const int by0 = max(cy - g.kh, 0), by1 = min(cy + g.kh, g.ncy - 1);
  const CellBox tb = cell_box(g, cx, cy, g.tw);  // the query cell's T-box (reading Q25)
  const bool tbox = g.tw > 0.0;
  double acc = 0.0;
  for (int by = by0; by <= by1; ++by) {
    const int s0 = cell_start[by * g.ncx + bx0], s1 = cell_start[by * g.ncx + bx1 + 1];
    for (int j = s0; j < s1; ++j) {
      const double4 o = ld_rec(rec + j);
      const double dx = qx - o.x, dy = qy - o.y;
      const double r2 = fma(dx, dx, dy * dy);
      if (tbox ? in_box(tb, o.x, o.y) : r2 < g.rc2) acc = fma(o.z, gauss_exp2<kExpDeg>(r2, g.esc), acc);
    }
  }
  s[k] = acc * g.norm;
}

int launch_pack_w(const rbf_ctx *c, const double *w_ext, cudaStream_t s);  // matvec.cu

int evaluate(rbf_ctx *c, const double *q, long long m, const double *lam, double *out,
             cudaStream_t s) {
  if (c->nranks > 1) {
    set_error("rbf_evaluate: single-rank contexts only (queries are not partitioned by strip)");
    return RBF_EUNSUPPORTED;
  }
  if (m == 0) return RBF_OK;
  if (m >= (1LL << 31)) {
    set_error("rbf_evaluate: m = %lld queries (at most 2^31 - 1 per call)", m);
    return RBF_EINVAL;
  }
  int *keys = nullptr, *vals = nullptr, *skeys = nullptr, *order = nullptr;
  long long *bad = nullptr;
  ScratchGuard sg(s);
  RBF_TRY(sg.alloc(nullptr, &keys, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &vals, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &skeys, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &order, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &bad, sizeof(long long)));
  RBF_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(long long), s));
  const int blocks = (int)((m + 255) / 256);
  k_query_keys<<<blocks, 256, 0, s>>>(q, m, c->g, keys, vals, bad);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  const int ncells = c->g.ncx * c->g.ncy;
  int end_bit = 1;
  while ((1LL << end_bit) < (long long)ncells) ++end_bit;
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, vals, order, (int)m, 0, end_bit, s));
  void *tmp = nullptr;
  RBF_TRY(sg.alloc(nullptr, &tmp, tb));
  RBF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, vals, order, (int)m, 0, end_bit, s));
  count_launch(1 + (end_bit + 7) / 8);
  RBF_TRY(launch_pack_w(c, lam, s));
  k_evaluate<<<blocks, 256, 0, s>>>(c->g, q, m, skeys, order, c->cell_start, c->rec, out);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  long long hbad = -1;
  RBF_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad != -1) {
    set_error("rbf_evaluate: query %lld is non-finite or outside the box [%g,%g]x[%g,%g]", hbad,
              c->g.x0, c->g.x1, c->g.y0, c->g.y1);
    return RBF_EINVAL;
  }
  return RBF_OK;
}

}  // namespace rbf
