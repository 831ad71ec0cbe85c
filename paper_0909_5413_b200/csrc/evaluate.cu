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

// One thread per query, the queries in cell order: the 32 lanes of a warp usually share
// one or two cells, so they walk the same (2kh+1) contiguous source runs of the
// cell-sorted records {x, y, lambda} (one 256-bit gather per candidate, L1-resident
// across the warp; measured faster than a walk over the warp's union box with
// broadcast loads, and than one thread per pair of queries -- DESIGN.md §6), test the
// exact fp64 cutoff and accumulate in ascending source order with the matvec's
// table-free exp: at a data point the result is bitwise the matvec row.  COUNT:
// in-cutoff pairs instead of values.  Queries outside this rank's strip of cell rows
// get 0 (another rank owns them).
template <bool COUNT>
__global__ __launch_bounds__(256) void k_evaluate(Geom g, Strip st, const double *__restrict__ q,
                                                   long long m, const int *__restrict__ skeys,
                                                   const int *__restrict__ order,
                                                   const int *__restrict__ cell_start,
                                                   const double4 *__restrict__ rec,
                                                   double *__restrict__ s,
                                                   unsigned long long *__restrict__ npairs) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int k = order[t], key = skeys[t];
  const int cx = key % g.ncx, cy = key / g.ncx;
  const double qx = q[2LL * k], qy = q[2LL * k + 1];
  const bool act = cy >= st.row_lo && cy < st.row_hi;
  const int bx0 = max(cx - g.kh, 0), bx1 = act ? min(cx + g.kh, g.ncx - 1) : -1;
  const int by0 = max(cy - g.kh, 0), by1 = act ? min(cy + g.kh, g.ncy - 1) : -1;
  const CellBox tb = cell_box(g, cx, cy, g.tw);  // the query cell's T-box (reading Q25)
  const bool tbox = g.tw > 0.0;
  double acc = 0.0;
  unsigned long long cnt = 0;
  // radial cutoff: per cell row, only the cells the disc |q - x| < rc reaches in x (the
  // row's distance from q, less a margin, bounds |dy| from below); the skipped sources
  // all fail the exact test, so the sum (same sources, same order) is unchanged
  const double mg = 1e-9 * g.cell;
  for (int by = by0; by <= by1; ++by) {
    int xa = bx0, xb = bx1;
    if (!tbox) {
      const double lo = g.y0 + by * g.cell, hi = lo + g.cell;
      const double dy = fmax(fmax(fmax(lo - qy, qy - hi), 0.0) - mg, 0.0);
      const double w2 = g.rc2 - dy * dy;
      if (!(w2 > 0.0)) continue;
      const double wx = sqrt(w2) + mg;
      xa = max(bx0, (int)floor((qx - wx - g.x0) / g.cell));
      xb = min(bx1, (int)floor((qx + wx - g.x0) / g.cell));
      if (xa > xb) continue;
    }
    const int s0 = cell_start[by * g.ncx + xa], s1 = cell_start[by * g.ncx + xb + 1];
    for (int j = s0; j < s1; ++j) {
      const double4 o = ld_rec(rec + (j - st.ext_lo));
      const double dx = qx - o.x, dy = qy - o.y;
      const double r2 = fma(dx, dx, dy * dy);
      if (tbox ? in_box(tb, o.x, o.y) : r2 < g.rc2) {
        if (COUNT) ++cnt;
        else acc = fma(o.z, gauss_exp2<kExpDeg>(r2, g.esc), acc);
      }
    }
  }
  if (COUNT) {
    if (cnt) atomicAdd(npairs, cnt);
    return;
  }
  s[k] = act ? acc * g.norm : 0.0;
}

int launch_pack_w(const rbf_ctx *c, const double *w_ext, cudaStream_t s);  // matvec.cu

int evaluate(rbf_ctx *c, const double *q, long long m, const double *lam, double *out,
             cudaStream_t s, unsigned long long *pairs_out) {
  if (m == 0) {
    if (pairs_out) *pairs_out = 0;
    return RBF_OK;
  }
  if (m >= (1LL << 31)) {
    set_error("rbf_evaluate: m = %lld queries (at most 2^31 - 1 per call)", m);
    return RBF_EINVAL;
  }
  if (c->nranks > 1 && c->comm_mode == RBF_COMM_NONE) {
    set_error("rbf_evaluate: a virtual strip context (RBF_COMM_NONE) cannot combine the strips' results");
    return RBF_EUNSUPPORTED;
  }
  int *keys = nullptr, *vals = nullptr, *skeys = nullptr, *order = nullptr;
  long long *bad = nullptr;
  unsigned long long *np = nullptr;
  ScratchGuard sg(s);
  RBF_TRY(sg.alloc(nullptr, &keys, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &vals, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &skeys, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &order, sizeof(int) * m));
  RBF_TRY(sg.alloc(nullptr, &bad, sizeof(long long)));
  RBF_TRY(sg.alloc(nullptr, &np, sizeof(unsigned long long)));
  RBF_CUDA_TRY(cudaMemsetAsync(bad, 0xff, sizeof(long long), s));
  RBF_CUDA_TRY(cudaMemsetAsync(np, 0, sizeof(unsigned long long), s));
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
  // the weights of the ext range: this strip's plus the matvec halo (multi-rank)
  if (!pairs_out) {
    if (c->nranks > 1) {
      RBF_TRY(halo_exchange(c, lam, c->w_ext, true, s));
      RBF_TRY(launch_pack_w(c, c->w_ext, s));
    } else {
      RBF_TRY(launch_pack_w(c, lam, s));
    }
  }
  if (pairs_out)
    k_evaluate<true><<<blocks, 256, 0, s>>>(c->g, c->s, q, m, skeys, order, c->cell_start, c->rec, out, np);
  else
    k_evaluate<false><<<blocks, 256, 0, s>>>(c->g, c->s, q, m, skeys, order, c->cell_start, c->rec, out, np);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  // every query is evaluated by exactly one strip (the others write 0): the sum over
  // ranks is exact in any order
  if (!pairs_out && c->nranks > 1) RBF_TRY(allreduce_vector(c, out, m, s));
  long long hbad = -1;
  unsigned long long hnp = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&hnp, np, sizeof(hnp), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad != -1) {
    set_error("rbf_evaluate: query %lld is non-finite or outside the box [%g,%g]x[%g,%g]", hbad,
              c->g.x0, c->g.x1, c->g.y0, c->g.y1);
    return RBF_EINVAL;
  }
  if (pairs_out) {
    *pairs_out = hnp;
    if (c->nranks > 1) {
      // in-cutoff pairs of all strips (one all-gather of the per-rank counts)
      double *d = nullptr;
      RBF_TRY(sg.alloc(nullptr, &d, sizeof(double) * (1 + c->nranks)));
      const double v = (double)hnp;
      RBF_CUDA_TRY(cudaMemcpyAsync(d, &v, sizeof(double), cudaMemcpyHostToDevice, s));
      RBF_TRY(allgather_scalars(c, d, d + 1, 1, s));
      std::vector<double> h(c->nranks);
      RBF_CUDA_TRY(cudaMemcpyAsync(h.data(), d + 1, sizeof(double) * c->nranks, cudaMemcpyDeviceToHost, s));
      RBF_CUDA_TRY(cudaStreamSynchronize(s));
      unsigned long long tot = 0;
      for (double x : h) tot += (unsigned long long)x;
      *pairs_out = tot;
    }
  }
  return RBF_OK;
}

}  // namespace rbf
