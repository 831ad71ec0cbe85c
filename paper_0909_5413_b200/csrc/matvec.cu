// matvec.cu -- fp64 cutoff-Gaussian matvec (Eq.(12)).
//
//   y_i = norm * sum_{j : fma(dx,dx,dy*dy) < rc^2} w_j exp(-r2_ij / (2 sigma^2))
//
// over the (2kh+1)^2 cell stencil around the target's cell.  With row-major cell
// keys the stencil is 2kh+1 contiguous runs of the sorted arrays.  The per-target
// sum order (stencil rows ascending, sources ascending) depends only on the point
// set, never on the strip, so per-point results are bitwise identical for any
// number of ranks (reading Q20).
#include "common.cuh"

namespace rbf {

constexpr int kMvWarps = 4;  // cells per CTA (one warp per target cell)

__global__ __launch_bounds__(32 * kMvWarps) void k_matvec_v1(
    Geom g, Strip st, const double2 *__restrict__ xy, const double *__restrict__ w,
    const int *__restrict__ cell_start, int ncells_owned, double *__restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int cl = blockIdx.x * kMvWarps + (threadIdx.x >> 5);
  if (cl >= ncells_owned) return;
  const int cy = st.row_lo + cl / g.ncx, cx = cl % g.ncx;
  const int key = cy * g.ncx + cx;
  const int t0 = cell_start[key], t1 = cell_start[key + 1];
  const int bx0 = max(cx - g.kh, 0), bx1 = min(cx + g.kh, g.ncx - 1);
  const int by0 = max(cy - g.kh, 0), by1 = min(cy + g.kh, g.ncy - 1);
  const long long e0 = st.ext_lo;
  for (int tb = t0; tb < t1; tb += 32) {
    const int t = tb + lane;
    const bool active = t < t1;
    const double2 p = xy[(active ? t : t0) - e0];
    double acc = 0.0;
    for (int by = by0; by <= by1; ++by) {
      const int s0 = cell_start[by * g.ncx + bx0], s1 = cell_start[by * g.ncx + bx1 + 1];
      for (int q = s0; q < s1; ++q) {
        const double2 o = xy[q - e0];
        const double dx = p.x - o.x, dy = p.y - o.y;
        const double r2 = fma(dx, dx, dy * dy);
        if (r2 < g.rc2) acc = fma(w[q - e0], exp(r2 * g.neg_inv_2s2), acc);
      }
    }
    if (active) y[t - st.own_lo] = acc * g.norm;
  }
}

int launch_matvec(const rbf_ctx *c, const double *w_ext, double *y_loc, cudaStream_t s) {
  int nc = owned_cells(c);
  if (nc <= 0) return RBF_OK;
  int blocks = (nc + kMvWarps - 1) / kMvWarps;
  k_matvec_v1<<<blocks, 32 * kMvWarps, 0, s>>>(c->g, c->s, c->xy_ext, w_ext, c->cell_start, nc,
                                               y_loc); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

}  // namespace rbf
