/*
 * oracle/rbf_oracle.c -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * A plain, slow, obviously-correct CPU implementation of what the PetRBF hot
 * path computes (Yokota, Barba, Knepley, arXiv 0909.5413; /root/reference/PAPER.md,
 * cited below as P:<line>).  It shares no code, header, table or constant with
 * the CUDA path in paper_0909_5413_b200/ and includes no CUDA header.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.
 *
 * Arithmetic is IEEE fp64, compiled with -ffp-contract=off so that every fused
 * multiply-add below is one that is written out with fma().
 *
 * Readings of the paper (numbered Q1..Q20 as in SURVEY.md §8.c.2 and DESIGN.md):
 *   Q1  per-pair radial cutoff: j contributes to row i iff r2_ij < rc*rc,
 *       r2_ij = fma(dx, dx, dy*dy), dx = x_i - x_j, dy = y_i - y_j.
 *   Q2  normalised Gaussian A_ij = exp(-r^2/(2 sigma^2)) / (2 pi sigma^2), Eq.(12) P:244-246.
 *   Q5  cell grid with origin (x0,y0), side c, ncx = ceil((x1-x0)/c);
 *       cx = clamp(floor((x - x0)/c), 0, ncx-1); key = cy*ncx + cx.
 *   Q9  one subdomain per non-empty cell; Omega_c = the (2*rings+1)^2 block of
 *       cells around c clipped to the grid, visited row-major (cy then cx),
 *       points inside a cell in ascending caller index; Omega~_c = own(c).
 *   Q10 the local matrix A_c is the principal submatrix of the truncated A_rc.
 *   Q11 Cholesky (lower); if a pivot is <= 0, LU with partial pivoting (largest
 *       |a|, lowest row index on ties).  The oracle applies A_c^-1 by
 *       forward/back substitution.
 *   Q12 left-preconditioned restarted GMRES(m), modified Gram-Schmidt, Givens
 *       rotations, x0 = 0; stop when |g_{k+1}| <= max(rtol*||M^-1 f||, atol);
 *       explicit preconditioned residual at each restart; happy breakdown when
 *       h_{k+1,k} == 0.
 *   Q25 (optional) the paper's T-box matvec truncation: row i
 *       keeps the sources inside target i's cell box grown by tau (closed); the
 *       local matrices of the preconditioner stay principal submatrices of A_rc.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 2
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-2)
#define ORC_EFACTOR (-5)
#define ORC_ENUMERIC (-6)

/* ------------------------------------------------------------------------ */
/* Kernel entries, Eq.(12)                                         */
/* ------------------------------------------------------------------------ */

/* phi(r2) = exp(-r2 / (2 sigma^2)) / (2 pi sigma^2)   (Eq.(12)) */
double orc_phi(double sigma, double r2) {
  double two_s2 = 2.0 * sigma * sigma;
  return exp(-r2 / two_s2) / (M_PI * two_s2);
}

/* squared distance, reading Q1 */
static double sqdist(const double *xy, int64_t i, int64_t j) {
  double dx = xy[2 * i] - xy[2 * j];
  double dy = xy[2 * i + 1] - xy[2 * j + 1];
  return fma(dx, dx, dy * dy);
}

/* sigma * sqrt(-2 ln t): the radius where exp(-r^2/2sigma^2) = t */
double orc_cutoff_radius(double sigma, double rel_tol) {
  return sigma * sqrt(-2.0 * log(rel_tol));
}

/* Dense A (exact when rc <= 0, else A_rc with the Q1 indicator), row-major n x n.
 * Eq.(4) Phi block, with the entries of Eq.(12). */
void orc_assemble_dense(int64_t n, const double *xy, double sigma, double rc,
                        double *A) {
  double rc2 = rc * rc;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double r2 = sqdist(xy, i, j);
      A[i * n + j] = (rc <= 0.0 || r2 < rc2) ? orc_phi(sigma, r2) : 0.0;
    }
}

/* ------------------------------------------------------------------------ */
/* Matrix-vector product, P:248 ("sparse matrix-vector multiplication with   */
/* controllable accuracy") and Q1.                                           */
/* ------------------------------------------------------------------------ */

/* Plain definition, O(N^2): y_i = sum_{j=0..n-1} [r2_ij < rc^2] w_j phi(r2_ij),
 * summed in ascending j.  exact != 0 drops the indicator (the untruncated A).
 * rows == NULL computes every row (y has n entries); otherwise y[k] is row
 * rows[k] (used for sampled parity at full sizes). */
void orc_matvec_brute(int64_t n, const double *xy, const double *w, double sigma,
                      double rc, int exact, int64_t nrows, const int64_t *rows,
                      double *y) {
  double rc2 = rc * rc;
  int64_t m = rows ? nrows : n;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = rows ? rows[k] : k;
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double r2 = sqdist(xy, i, j);
      if (exact || r2 < rc2) acc += w[j] * orc_phi(sigma, r2);
    }
    y[k] = acc;
  }
}

/* Interpolant evaluation s(q_k) = sum_{j=0..n-1} [r2 < rc^2] lambda_j phi(r2), r2 =
 * |q_k - x_j|^2 (Eq.(1) P:76-79 with the Gaussian of Eq.(12) and the truncation of
 * reading Q1), brute force over all j in ascending order.  exact != 0
 * drops the indicator.  At q_k = x_k this is row k of orc_matvec_brute. */
void orc_evaluate(int64_t m, const double *q, int64_t n, const double *xy, const double *lam,
                  double sigma, double rc, int exact, double *s) {
  double rc2 = rc * rc;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < m; ++k) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double dx = q[2 * k] - xy[2 * j];
      double dy = q[2 * k + 1] - xy[2 * j + 1];
      double r2 = fma(dx, dx, dy * dy);
      if (exact || r2 < rc2) acc += lam[j] * orc_phi(sigma, r2);
    }
    s[k] = acc;
  }
}

/* Neglected row mass sum_{j: r2_ij >= rc^2} phi(r2_ij), brute force. */
void orc_neglected_row_mass(int64_t n, const double *xy, double sigma, double rc,
                            int64_t nrows, const int64_t *rows, double *out) {
  double rc2 = rc * rc;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < nrows; ++k) {
    int64_t i = rows[k];
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double r2 = sqdist(xy, i, j);
      if (!(r2 < rc2)) acc += orc_phi(sigma, r2);
    }
    out[k] = acc;
  }
}

/* ------------------------------------------------------------------------ */
/* Cell grid and cell list (reading Q5; index sets of P:250, 268)            */
/* ------------------------------------------------------------------------ */

typedef struct {
  double x0, y0, cell;
  int64_t ncx, ncy;
} orc_grid;

static orc_grid make_grid(double x0, double y0, double x1, double y1, double cell) {
  orc_grid g;
  g.x0 = x0;
  g.y0 = y0;
  g.cell = cell;
  g.ncx = (int64_t)ceil((x1 - x0) / cell);
  g.ncy = (int64_t)ceil((y1 - y0) / cell);
  if (g.ncx < 1) g.ncx = 1;
  if (g.ncy < 1) g.ncy = 1;
  return g;
}

void orc_grid_dims(double x0, double y0, double x1, double y1, double cell,
                   int64_t *ncx, int64_t *ncy) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  *ncx = g.ncx;
  *ncy = g.ncy;
}

static int64_t cell_coord(double v, double v0, double c, int64_t ncells) {
  double t = floor((v - v0) / c);
  if (t < 0.0) t = 0.0;
  if (t > (double)(ncells - 1)) t = (double)(ncells - 1);
  return (int64_t)t;
}

static int64_t cell_key(const orc_grid *g, double x, double y) {
  return cell_coord(y, g->y0, g->cell, g->ncy) * g->ncx +
         cell_coord(x, g->x0, g->cell, g->ncx);
}

/* Stable counting sort of the points by cell key.
 * key[i]        cell of caller point i
 * perm[s]       caller index of the s-th point in sorted order
 * cell_start[k] first sorted position of cell k (ncx*ncy + 1 entries) */
void orc_cell_list(int64_t n, const double *xy, double x0, double y0, double x1,
                   double y1, double cell, int64_t *key, int64_t *perm,
                   int64_t *cell_start) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t ncells = g.ncx * g.ncy;
  for (int64_t k = 0; k <= ncells; ++k) cell_start[k] = 0;
  for (int64_t i = 0; i < n; ++i) {
    key[i] = cell_key(&g, xy[2 * i], xy[2 * i + 1]);
    cell_start[key[i] + 1] += 1;
  }
  for (int64_t k = 0; k < ncells; ++k) cell_start[k + 1] += cell_start[k];
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells > 0 ? ncells : 1));
  for (int64_t k = 0; k < ncells; ++k) fill[k] = cell_start[k];
  for (int64_t i = 0; i < n; ++i) perm[fill[key[i]]++] = i; /* ascending i: stable */
  free(fill);
}

/* number of cell rings the matvec must search so that every pair with
 * r < rc is found: kh = ceil(rc/c), bumped when rc/c is (nearly) integral */
static int64_t search_rings(double rc, double cell) {
  return (int64_t)ceil(rc / cell * (1.0 + 1e-12));
}

/* Cell-list version of orc_matvec_brute: the same sum restricted to the cells
 * within search_rings() of the target's cell (an acceleration only; pinned to
 * orc_matvec_brute by tests).  Caller order in and out. */
int orc_matvec_cells(int64_t n, const double *xy, const double *w, double sigma,
                     double rc, double x0, double y0, double x1, double y1,
                     double cell, double *y) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t ncells = g.ncx * g.ncy;
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
  if (!key || !perm || !start) {
    free(key); free(perm); free(start);
    return ORC_ENOMEM;
  }
  orc_cell_list(n, xy, x0, y0, x1, y1, cell, key, perm, start);
  int64_t kh = search_rings(rc, cell);
  double rc2 = rc * rc;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int64_t cx = key[i] % g.ncx, cy = key[i] / g.ncx;
    double acc = 0.0;
    for (int64_t by = cy - kh; by <= cy + kh; ++by) {
      if (by < 0 || by >= g.ncy) continue;
      for (int64_t bx = cx - kh; bx <= cx + kh; ++bx) {
        if (bx < 0 || bx >= g.ncx) continue;
        int64_t c = by * g.ncx + bx;
        for (int64_t s = start[c]; s < start[c + 1]; ++s) {
          int64_t j = perm[s];
          double r2 = sqdist(xy, i, j);
          if (r2 < rc2) acc += w[j] * orc_phi(sigma, r2);
        }
      }
    }
    y[i] = acc;
  }
  free(key);
  free(perm);
  free(start);
  return ORC_OK;
}

/* Count of in-cutoff pairs (i, j) including i == j, by cell search. */
int64_t orc_count_pairs(int64_t n, const double *xy, double rc, double x0,
                        double y0, double x1, double y1, double cell) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t ncells = g.ncx * g.ncy;
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
  orc_cell_list(n, xy, x0, y0, x1, y1, cell, key, perm, start);
  int64_t kh = search_rings(rc, cell);
  double rc2 = rc * rc;
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (int64_t i = 0; i < n; ++i) {
    int64_t cx = key[i] % g.ncx, cy = key[i] / g.ncx;
    for (int64_t by = cy - kh; by <= cy + kh; ++by) {
      if (by < 0 || by >= g.ncy) continue;
      for (int64_t bx = cx - kh; bx <= cx + kh; ++bx) {
        if (bx < 0 || bx >= g.ncx) continue;
        int64_t c = by * g.ncx + bx;
        for (int64_t s = start[c]; s < start[c + 1]; ++s)
          if (sqdist(xy, i, perm[s]) < rc2) total += 1;
      }
    }
  }
  free(key);
  free(perm);
  free(start);
  return total;
}

/* ------------------------------------------------------------------------ */
/* T-box truncation (the paper's own matvec rule; reading Q25): */
/* "an additional subdomain with size T, which defines the non-zero entries   */
/* for the matrix-vector multiplication.  Everything outside of this region   */
/* is neglected when calculating A x for Omega~_i", T = B + 4 sigma*/
/* for h/sigma >= 0.9 and B + 6 sigma for 0.8.  Row i keeps      */
/* source j iff x_j lies in the closed box of target i's cell (the B box)     */
/* grown by tau = (T - B)/2 on every side:                                    */
/*   [x0 + cx c - tau, x0 + (cx+1) c + tau] x [same in y],                    */
/* edges formed as in reading Q24.  No radial test; the matrix is not         */
/* symmetric (targets of one cell share one box).                             */
/* ------------------------------------------------------------------------ */

static int in_tbox(const double *p, int64_t cx, int64_t cy, double x0, double y0, double cell,
                   double tau) {
  const double lx = x0 + (double)cx * cell, hx = x0 + (double)(cx + 1) * cell;
  const double ly = y0 + (double)cy * cell, hy = y0 + (double)(cy + 1) * cell;
  return p[0] >= lx - tau && p[0] <= hx + tau && p[1] >= ly - tau && p[1] <= hy + tau;
}

/* Plain definition, O(N^2): y_i = sum_{j=0..n-1} [x_j in T(cell(i))] w_j phi(r2_ij),
 * ascending j.  rows as in orc_matvec_brute. */
void orc_matvec_tbox(int64_t n, const double *xy, const double *w, double sigma, double x0,
                     double y0, double x1, double y1, double cell, double tau, int64_t nrows,
                     const int64_t *rows, double *y) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t m = rows ? nrows : n;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = rows ? rows[k] : k;
    int64_t cx = cell_coord(xy[2 * i], g.x0, g.cell, g.ncx);
    int64_t cy = cell_coord(xy[2 * i + 1], g.y0, g.cell, g.ncy);
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j)
      if (in_tbox(&xy[2 * j], cx, cy, x0, y0, cell, tau))
        acc += w[j] * orc_phi(sigma, sqdist(xy, i, j));
    y[k] = acc;
  }
}

/* Interpolant with the T-box (Eq.(1), reading Q25): s(q_k) = sum_j [x_j in
 * T(cell(q_k))] lambda_j phi(|q_k - x_j|^2), ascending j.  At q_k = x_k: row k of
 * orc_matvec_tbox. */
void orc_evaluate_tbox(int64_t m, const double *q, int64_t n, const double *xy,
                       const double *lam, double sigma, double x0, double y0, double x1,
                       double y1, double cell, double tau, double *s) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < m; ++k) {
    int64_t cx = cell_coord(q[2 * k], g.x0, g.cell, g.ncx);
    int64_t cy = cell_coord(q[2 * k + 1], g.y0, g.cell, g.ncy);
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (!in_tbox(&xy[2 * j], cx, cy, x0, y0, cell, tau)) continue;
      double dx = q[2 * k] - xy[2 * j];
      double dy = q[2 * k + 1] - xy[2 * j + 1];
      acc += lam[j] * orc_phi(sigma, fma(dx, dx, dy * dy));
    }
    s[k] = acc;
  }
}

/* Cell-list version (an acceleration only, pinned to orc_matvec_tbox): the box
 * reaches floor(tau/c) + 1 cells beyond the target's cell at most. */
int orc_matvec_tbox_cells(int64_t n, const double *xy, const double *w, double sigma,
                          double x0, double y0, double x1, double y1, double cell, double tau,
                          double *y) {
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t ncells = g.ncx * g.ncy;
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
  if (!key || !perm || !start) {
    free(key); free(perm); free(start);
    return ORC_ENOMEM;
  }
  orc_cell_list(n, xy, x0, y0, x1, y1, cell, key, perm, start);
  int64_t kh = (int64_t)floor(tau / cell * (1.0 + 1e-12)) + 1;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int64_t cx = key[i] % g.ncx, cy = key[i] / g.ncx;
    double acc = 0.0;
    for (int64_t by = cy - kh; by <= cy + kh; ++by) {
      if (by < 0 || by >= g.ncy) continue;
      for (int64_t bx = cx - kh; bx <= cx + kh; ++bx) {
        if (bx < 0 || bx >= g.ncx) continue;
        int64_t c = by * g.ncx + bx;
        for (int64_t s = start[c]; s < start[c + 1]; ++s) {
          int64_t j = perm[s];
          if (in_tbox(&xy[2 * j], cx, cy, x0, y0, cell, tau))
            acc += w[j] * orc_phi(sigma, sqdist(xy, i, j));
        }
      }
    }
    y[i] = acc;
  }
  free(key);
  free(perm);
  free(start);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Dense local factorizations ("-sub_pc_type lu -sub_mat_type dense";  */
/* reading Q11)                                                              */
/* ------------------------------------------------------------------------ */

/* In-place Cholesky A = L L^T of a row-major n x n matrix (lower triangle
 * overwritten by L).  Returns the failing column + 1 when a pivot is <= 0. */
static int64_t cholesky(int64_t n, double *A) {
  for (int64_t j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int64_t k = 0; k < j; ++k) d -= A[j * n + k] * A[j * n + k];
    if (!(d > 0.0)) return j + 1;
    double ljj = sqrt(d);
    A[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = A[i * n + j];
      for (int64_t k = 0; k < j; ++k) s -= A[i * n + k] * A[j * n + k];
      A[i * n + j] = s / ljj;
    }
  }
  return 0;
}

/* In-place LU with partial pivoting (Doolittle, unit lower L).  piv[k] is the
 * row swapped with row k at step k.  Returns column + 1 on an exactly zero pivot. */
static int64_t lu_factor(int64_t n, double *A, int64_t *piv) {
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = fabs(A[k * n + k]);
    for (int64_t i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > best) { best = fabs(A[i * n + k]); p = i; }
    piv[k] = p;
    if (best == 0.0) return k + 1;
    if (p != k)
      for (int64_t j = 0; j < n; ++j) {
        double t = A[k * n + j]; A[k * n + j] = A[p * n + j]; A[p * n + j] = t;
      }
    for (int64_t i = k + 1; i < n; ++i) {
      double l = A[i * n + k] / A[k * n + k];
      A[i * n + k] = l;
      for (int64_t j = k + 1; j < n; ++j) A[i * n + j] -= l * A[k * n + j];
    }
  }
  return 0;
}

static void cholesky_solve(int64_t n, const double *L, double *b) {
  for (int64_t i = 0; i < n; ++i) { /* L y = b */
    double s = b[i];
    for (int64_t k = 0; k < i; ++k) s -= L[i * n + k] * b[k];
    b[i] = s / L[i * n + i];
  }
  for (int64_t i = n - 1; i >= 0; --i) { /* L^T x = y */
    double s = b[i];
    for (int64_t k = i + 1; k < n; ++k) s -= L[k * n + i] * b[k];
    b[i] = s / L[i * n + i];
  }
}

static void lu_solve(int64_t n, const double *LU, const int64_t *piv, double *b) {
  for (int64_t k = 0; k < n; ++k)
    if (piv[k] != k) { double t = b[k]; b[k] = b[piv[k]]; b[piv[k]] = t; }
  for (int64_t i = 0; i < n; ++i) {
    double s = b[i];
    for (int64_t k = 0; k < i; ++k) s -= LU[i * n + k] * b[k];
    b[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int64_t k = i + 1; k < n; ++k) s -= LU[i * n + k] * b[k];
    b[i] = s / LU[i * n + i];
  }
}

/* Dense SPD factor/solve exposed for the linalg pins. */
int orc_dense_factor_solve(int64_t n, const double *A, const double *b, double *x,
                           int *used_lu) {
  double *F = (double *)malloc(sizeof(double) * (size_t)(n * n));
  int64_t *piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!F || !piv) { free(F); free(piv); return ORC_ENOMEM; }
  memcpy(F, A, sizeof(double) * (size_t)(n * n));
  memcpy(x, b, sizeof(double) * (size_t)n);
  *used_lu = 0;
  int rc = ORC_OK;
  if (cholesky(n, F) == 0) {
    cholesky_solve(n, F, x);
  } else {
    *used_lu = 1;
    memcpy(F, A, sizeof(double) * (size_t)(n * n));
    if (lu_factor(n, F, piv) != 0) rc = ORC_EFACTOR;
    else lu_solve(n, F, piv, x);
  }
  free(F);
  free(piv);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Restricted additive Schwarz preconditioner, Eqs.(5),(9)-(11) P:180-226    */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t n_own, n_ov;
  int64_t *ov;      /* caller indices of Omega_c in local order (R_c, Eq.(5)) */
  int64_t *own_pos; /* local positions of own(c) inside Omega_c (R~_c, Eq.(9)) */
  double *F;        /* factor of A_c = R_c A R_c^T, n_ov x n_ov row-major */
  int64_t *piv;     /* LU pivots, NULL when Cholesky succeeded */
} orc_sub;

typedef struct {
  int64_t n, nsub, ncells;
  orc_sub *sub;
  int64_t n_lu; /* subdomains that needed the LU fallback */
  int64_t bad_cell;
  int status;
} orc_rasm;

/* Set up M^-1 = sum_c R~_c^T A_c^-1 R_c (Eq.(11)) with one subdomain
 * per non-empty cell (Q9), A_c the principal submatrix of A_rc (Q10), factored
 * by Cholesky with LU fallback (Q11).  variant_asm != 0 keeps the ASM form
 * (Eq.(8)): every point of Omega_c receives the local solution. */
orc_rasm *orc_rasm_setup_box(int64_t n, const double *xy, double sigma, double rc,
                             double x0, double y0, double x1, double y1, double cell,
                             int64_t rings, double delta);

orc_rasm *orc_rasm_setup(int64_t n, const double *xy, double sigma, double rc,
                         double x0, double y0, double x1, double y1, double cell,
                         int64_t rings) {
  return orc_rasm_setup_box(n, xy, sigma, rc, x0, y0, x1, y1, cell, rings, 0.0);
}

/* Box overlap (reading Q24, the paper's "overlapping subdomains of size D"):
 * with delta > 0, Omega_c keeps, of the block's points, own(c) and every point inside
 * cell c's box grown by delta on each side, [x0 + cx c - delta, x0 + (cx+1) c + delta]
 * x [same in y] (closed; D = c + 2 delta).  The order stays the block order. */
static int in_grown_box(const double *p, int64_t cx, int64_t cy, double x0, double y0,
                        double cell, double delta) {
  const double lx = x0 + (double)cx * cell, hx = x0 + (double)(cx + 1) * cell;
  const double ly = y0 + (double)cy * cell, hy = y0 + (double)(cy + 1) * cell;
  return p[0] >= lx - delta && p[0] <= hx + delta && p[1] >= ly - delta && p[1] <= hy + delta;
}

orc_rasm *orc_rasm_setup_box(int64_t n, const double *xy, double sigma, double rc,
                             double x0, double y0, double x1, double y1, double cell,
                             int64_t rings, double delta) {
  orc_rasm *P = (orc_rasm *)calloc(1, sizeof(orc_rasm));
  orc_grid g = make_grid(x0, y0, x1, y1, cell);
  int64_t ncells = g.ncx * g.ncy;
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
  orc_cell_list(n, xy, x0, y0, x1, y1, cell, key, perm, start);
  P->n = n;
  P->ncells = ncells;
  P->bad_cell = -1;
  /* subdomain list: every non-empty cell, in key order */
  int64_t nsub = 0;
  for (int64_t c = 0; c < ncells; ++c) if (start[c + 1] > start[c]) ++nsub;
  P->nsub = nsub;
  P->sub = (orc_sub *)calloc((size_t)(nsub > 0 ? nsub : 1), sizeof(orc_sub));
  int64_t *cell_of_sub = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nsub > 0 ? nsub : 1));
  for (int64_t c = 0, s = 0; c < ncells; ++c) if (start[c + 1] > start[c]) cell_of_sub[s++] = c;
  double rc2 = rc * rc;
  int64_t n_lu = 0, bad = -1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : n_lu)
  for (int64_t s = 0; s < nsub; ++s) {
    int64_t c = cell_of_sub[s];
    int64_t cx = c % g.ncx, cy = c / g.ncx;
    orc_sub *S = &P->sub[s];
    /* R_c: the block's cells row-major, each cell's points in sorted order */
    int64_t cnt = 0;
    for (int64_t by = cy - rings; by <= cy + rings; ++by)
      for (int64_t bx = cx - rings; bx <= cx + rings; ++bx)
        if (by >= 0 && by < g.ncy && bx >= 0 && bx < g.ncx) {
          int64_t b = by * g.ncx + bx;
          for (int64_t t = start[b]; t < start[b + 1]; ++t)
            if (delta <= 0.0 || b == c || in_grown_box(&xy[2 * perm[t]], cx, cy, x0, y0, cell, delta))
              ++cnt;
        }
    S->n_ov = cnt;
    S->n_own = start[c + 1] - start[c];
    S->ov = (int64_t *)malloc(sizeof(int64_t) * (size_t)cnt);
    S->own_pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)S->n_own);
    int64_t q = 0, o = 0;
    for (int64_t by = cy - rings; by <= cy + rings; ++by)
      for (int64_t bx = cx - rings; bx <= cx + rings; ++bx) {
        if (by < 0 || by >= g.ncy || bx < 0 || bx >= g.ncx) continue;
        int64_t b = by * g.ncx + bx;
        for (int64_t t = start[b]; t < start[b + 1]; ++t) {
          if (!(delta <= 0.0 || b == c || in_grown_box(&xy[2 * perm[t]], cx, cy, x0, y0, cell, delta)))
            continue;
          if (b == c) S->own_pos[o++] = q;
          S->ov[q++] = perm[t];
        }
      }
    /* A_c = R_c A_rc R_c^T */
    int64_t m = cnt;
    S->F = (double *)malloc(sizeof(double) * (size_t)(m * m));
    for (int64_t p = 0; p < m; ++p)
      for (int64_t r = 0; r < m; ++r) {
        double r2 = sqdist(xy, S->ov[p], S->ov[r]);
        S->F[p * m + r] = (r2 < rc2) ? orc_phi(sigma, r2) : 0.0;
      }
    S->piv = NULL;
    if (cholesky(m, S->F) != 0) {
      /* Q11 fallback: re-assemble and LU-factor with partial pivoting */
      n_lu += 1;
      for (int64_t p = 0; p < m; ++p)
        for (int64_t r = 0; r < m; ++r) {
          double r2 = sqdist(xy, S->ov[p], S->ov[r]);
          S->F[p * m + r] = (r2 < rc2) ? orc_phi(sigma, r2) : 0.0;
        }
      S->piv = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
      if (lu_factor(m, S->F, S->piv) != 0) {
#pragma omp critical
        { if (bad < 0 || c < bad) bad = c; }
      }
    }
  }
  P->n_lu = n_lu;
  P->bad_cell = bad;
  P->status = (bad >= 0) ? ORC_EFACTOR : ORC_OK;
  free(cell_of_sub);
  free(key);
  free(perm);
  free(start);
  return P;
}

int orc_rasm_status(const orc_rasm *P, int64_t *bad_cell, int64_t *nsub, int64_t *n_lu) {
  *bad_cell = P->bad_cell;
  *nsub = P->nsub;
  *n_lu = P->n_lu;
  return P->status;
}

/* Local data of subdomain s (for the index-set pins): sizes, then arrays. */
void orc_rasm_sub_info(const orc_rasm *P, int64_t s, int64_t *n_own, int64_t *n_ov) {
  *n_own = P->sub[s].n_own;
  *n_ov = P->sub[s].n_ov;
}
void orc_rasm_sub_sets(const orc_rasm *P, int64_t s, int64_t *ov, int64_t *own_pos) {
  memcpy(ov, P->sub[s].ov, sizeof(int64_t) * (size_t)P->sub[s].n_ov);
  memcpy(own_pos, P->sub[s].own_pos, sizeof(int64_t) * (size_t)P->sub[s].n_own);
}

/* z = sum_c R~_c^T A_c^-1 R_c r   (Eq.(10)/(11)).  With asm != 0,
 * z = sum_c R_c^T A_c^-1 R_c r   (Eq.(8)) summed in subdomain order. */
void orc_rasm_apply(const orc_rasm *P, const double *r, double *z, int asm_variant) {
  int64_t n = P->n;
  for (int64_t i = 0; i < n; ++i) z[i] = 0.0;
  if (!asm_variant) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < P->nsub; ++s) {
      const orc_sub *S = &P->sub[s];
      double *y = (double *)malloc(sizeof(double) * (size_t)S->n_ov);
      for (int64_t q = 0; q < S->n_ov; ++q) y[q] = r[S->ov[q]]; /* R_c r */
      if (S->piv) lu_solve(S->n_ov, S->F, S->piv, y);          /* A_c^-1 */
      else cholesky_solve(S->n_ov, S->F, y);
      for (int64_t o = 0; o < S->n_own; ++o)                   /* R~_c^T */
        z[S->ov[S->own_pos[o]]] = y[S->own_pos[o]];
      free(y);
    }
  } else {
    for (int64_t s = 0; s < P->nsub; ++s) {
      const orc_sub *S = &P->sub[s];
      double *y = (double *)malloc(sizeof(double) * (size_t)S->n_ov);
      for (int64_t q = 0; q < S->n_ov; ++q) y[q] = r[S->ov[q]];
      if (S->piv) lu_solve(S->n_ov, S->F, S->piv, y);
      else cholesky_solve(S->n_ov, S->F, y);
      for (int64_t q = 0; q < S->n_ov; ++q) z[S->ov[q]] += y[q]; /* R_c^T */
      free(y);
    }
  }
}

void orc_rasm_free(orc_rasm *P) {
  if (!P) return;
  for (int64_t s = 0; s < P->nsub; ++s) {
    free(P->sub[s].ov);
    free(P->sub[s].own_pos);
    free(P->sub[s].F);
    free(P->sub[s].piv);
  }
  free(P->sub);
  free(P);
}

/* ------------------------------------------------------------------------ */
/* Linear operators for GMRES                                                */
/* ------------------------------------------------------------------------ */

typedef void (*orc_apply_fn)(void *ctx, const double *x, double *y);

enum { ORC_OP_IDENTITY = 0, ORC_OP_DENSE = 1, ORC_OP_RBF = 2, ORC_OP_RASM = 3,
       ORC_OP_RBF_BRUTE = 4, ORC_OP_RBF_TBOX = 5 };

typedef struct {
  int kind;
  int64_t n;
  const double *A; /* dense */
  const double *xy; double sigma, rc, x0, y0, x1, y1, cell; /* rbf */
  double tau;                                                /* rbf T-box (Q25) */
  const orc_rasm *P; int asm_variant;                        /* rasm */
} orc_op;

static void op_apply(const orc_op *op, const double *x, double *y) {
  int64_t n = op->n;
  switch (op->kind) {
  case ORC_OP_IDENTITY:
    for (int64_t i = 0; i < n; ++i) y[i] = x[i];
    break;
  case ORC_OP_DENSE:
#pragma omp parallel for
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < n; ++j) s += op->A[i * n + j] * x[j];
      y[i] = s;
    }
    break;
  case ORC_OP_RBF:
    orc_matvec_cells(n, op->xy, x, op->sigma, op->rc, op->x0, op->y0, op->x1, op->y1,
                     op->cell, y);
    break;
  case ORC_OP_RBF_BRUTE:
    orc_matvec_brute(n, op->xy, x, op->sigma, op->rc, 0, 0, NULL, y);
    break;
  case ORC_OP_RBF_TBOX:
    orc_matvec_tbox_cells(n, op->xy, x, op->sigma, op->x0, op->y0, op->x1, op->y1, op->cell,
                          op->tau, y);
    break;
  case ORC_OP_RASM:
    orc_rasm_apply(op->P, x, y, op->asm_variant);
    break;
  }
}

static double dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* GMRES report (all residuals relative) */
typedef struct {
  int64_t iterations;
  int64_t restarts;
  int converged;
  int status;
  double resid_est;      /* |g_{k+1}| / beta0 at exit (recurrence)           */
  double resid_precond;  /* ||M^-1 (b - A x)|| / ||M^-1 b|| (explicit)      */
  double resid_true;     /* ||b - A x|| / ||b||                             */
  double beta0;          /* ||M^-1 b||                                      */
} orc_report;

/* Left-preconditioned restarted GMRES(m) with Givens rotations ("we use the
 * GMRES"; reading Q12).  x0 = 0.  orth selects the Arnoldi
 * orthogonalisation: 0 = modified Gram-Schmidt (Q12, BJ:5), 1 = classical
 * Gram-Schmidt applied twice (CGS2: h = V^T w, w -= V h, twice, H column = the sum
 * of both passes; SURVEY §8.f3 -- the communication-avoiding variant, reading Q23).
 * history[k] = |g_{k+1}| / beta0 after iteration k (up to hist_cap entries).
 * V_out (optional, (m+1) x n) receives the Krylov basis of the last cycle and
 * *v_count the number of basis vectors in it (for the orthogonality pin). */
static int gmres_dcgs2(const orc_op *A, const orc_op *M, const double *b, int64_t restart,
                       int64_t max_iters, double rtol, double atol, double *x, double *history,
                       int64_t hist_cap, orc_report *rep, double *V_out, int64_t *v_count);

int orc_gmres_orth(const orc_op *A, const orc_op *M, const double *b, int64_t restart,
                   int64_t max_iters, double rtol, double atol, int orth, double *x,
                   double *history, int64_t hist_cap, orc_report *rep, double *V_out,
                   int64_t *v_count) {
  int64_t n = A->n, m = restart;
  memset(rep, 0, sizeof(*rep));
  if (m < 1 || rtol < 0.0 || atol < 0.0 || orth < 0 || orth > 2) return ORC_EINVAL;
  if (orth == 2)
    return gmres_dcgs2(A, M, b, restart, max_iters, rtol, atol, x, history, hist_cap, rep, V_out,
                       v_count);
  double *hp = (double *)malloc(sizeof(double) * (size_t)(m + 1)); /* one CGS pass */
  double *V = (double *)malloc(sizeof(double) * (size_t)((m + 1) * n));
  double *H = (double *)calloc((size_t)((m + 1) * m), sizeof(double)); /* H[i*m + k] */
  double *cs = (double *)malloc(sizeof(double) * (size_t)m);
  double *sn = (double *)malloc(sizeof(double) * (size_t)m);
  double *g = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *yk = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *t = (double *)malloc(sizeof(double) * (size_t)n);
  double *r = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  /* r0 = M^-1 (b - A x0) = M^-1 b */
  op_apply(M, b, r);
  double beta0 = sqrt(dot(n, r, r));
  rep->beta0 = beta0;
  double bnorm = sqrt(dot(n, b, b));
  int64_t it = 0;
  int converged = 0;
  int status = ORC_OK;
  if (v_count) *v_count = 0;
  if (beta0 == 0.0) {
    converged = 1;
  } else {
    double tol = fmax(rtol * beta0, atol);
    double beta = beta0;
    for (;;) {
      /* v_0 = r / beta, g = beta e_1 */
      for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
      for (int64_t i = 0; i <= m; ++i) g[i] = 0.0;
      g[0] = beta;
      int64_t k_end = 0;
      int done = 0;
      for (int64_t k = 0; k < m; ++k) {
        double *w = &V[(k + 1) * n];
        op_apply(A, &V[k * n], t); /* w = M^-1 A v_k */
        op_apply(M, t, w);
        if (orth == 0) {
          for (int64_t j = 0; j <= k; ++j) { /* modified Gram-Schmidt */
            double h = dot(n, w, &V[j * n]);
            H[j * m + k] = h;
            for (int64_t i = 0; i < n; ++i) w[i] -= h * V[j * n + i];
          }
        } else {
          for (int64_t j = 0; j <= k; ++j) H[j * m + k] = 0.0;
          for (int pass = 0; pass < 2; ++pass) { /* classical Gram-Schmidt, twice */
            for (int64_t j = 0; j <= k; ++j) hp[j] = dot(n, w, &V[j * n]);
            for (int64_t j = 0; j <= k; ++j) {
              H[j * m + k] += hp[j];
              for (int64_t i = 0; i < n; ++i) w[i] -= hp[j] * V[j * n + i];
            }
          }
        }
        double hn = sqrt(dot(n, w, w));
        H[(k + 1) * m + k] = hn;
        if (!isfinite(hn)) { status = ORC_ENUMERIC; done = 1; k_end = k; break; }
        if (hn != 0.0)
          for (int64_t i = 0; i < n; ++i) w[i] /= hn;
        for (int64_t j = 0; j < k; ++j) { /* previous rotations on column k */
          double a = H[j * m + k], c = H[(j + 1) * m + k];
          H[j * m + k] = cs[j] * a + sn[j] * c;
          H[(j + 1) * m + k] = -sn[j] * a + cs[j] * c;
        }
        double a = H[k * m + k], c = H[(k + 1) * m + k];
        double den = hypot(a, c);
        cs[k] = a / den;
        sn[k] = c / den;
        H[k * m + k] = den;
        H[(k + 1) * m + k] = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
        ++it;
        if (it - 1 < hist_cap) history[it - 1] = fabs(g[k + 1]) / beta0;
        k_end = k + 1;
        if (fabs(g[k + 1]) <= tol || hn == 0.0) { converged = 1; done = 1; break; }
        if (it >= max_iters) { done = 1; break; }
      }
      if (V_out) {
        int64_t nv = k_end + 1;
        memcpy(V_out, V, sizeof(double) * (size_t)(nv * n));
        if (v_count) *v_count = nv;
      }
      /* y = H^-1 g (upper triangular k_end x k_end), x += V y */
      for (int64_t i = k_end - 1; i >= 0; --i) {
        double s = g[i];
        for (int64_t j = i + 1; j < k_end; ++j) s -= H[i * m + j] * yk[j];
        yk[i] = s / H[i * m + i];
      }
      for (int64_t j = 0; j < k_end; ++j)
        for (int64_t i = 0; i < n; ++i) x[i] += yk[j] * V[j * n + i];
      rep->resid_est = fabs(g[k_end]) / beta0;
      if (done) break;
      /* restart: r = M^-1 (b - A x), explicitly */
      op_apply(A, x, t);
      for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
      op_apply(M, t, r);
      beta = sqrt(dot(n, r, r));
      rep->restarts += 1;
      if (beta <= tol) { converged = 1; rep->resid_est = beta / beta0; break; }
    }
  }
  /* explicit residuals for the report */
  op_apply(A, x, t);
  for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
  rep->resid_true = (bnorm > 0.0) ? sqrt(dot(n, t, t)) / bnorm : 0.0;
  op_apply(M, t, r);
  rep->resid_precond = (beta0 > 0.0) ? sqrt(dot(n, r, r)) / beta0 : 0.0;
  rep->iterations = it;
  rep->converged = converged;
  if (status == ORC_OK && !converged) status = ORC_NOT_CONVERGED;
  rep->status = status;
  free(V); free(H); free(cs); free(sn); free(g); free(yk); free(t); free(r); free(hp);
  return status;
}

/* GMRES with delayed classical Gram-Schmidt reorthogonalisation, one reduction per
 * Arnoldi step (orth = 2; SURVEY §8.f3 "one allreduce per iteration"; reading Q27).
 * The low-synchronisation Arnoldi of Swirydowicz, Langou, Ananthan, Yang, Thomas
 * (2020) and Bielich et al. (2022) ("DCGS2"), restated:
 *   slot k of V holds u_k = the k-th direction after ONE classical Gram-Schmidt pass,
 *   not yet reorthogonalised nor normalised (u_0 = the preconditioned residual).
 *   Step k (k = 0..m):
 *     w = B u_k (B = M^-1 A; skipped at k = m)
 *     one block reduction:  a_j = <v_j, u_k>, alpha = <u_k, u_k>,
 *                           b_j = <v_j, w>,   gamma = <u_k, w>        (j < k)
 *     rho = sqrt(alpha - sum a_j^2)            (Pythagoras: ||u_k - V a||)
 *     column k-1 of the Arnoldi relation:  H(j, k-1) = s_j + a_j,  H(k, k-1) = rho
 *       (s = the first-pass coefficients of u_k), then the Givens update (Q12);
 *       k = 0: beta = rho, g = beta e_1
 *     v_k = (u_k - sum_j a_j v_j) / rho
 *     c = V_{0..k}^T w / ... :  c_j = b_j (j < k),  c_k = (gamma - a^T b) / rho
 *     next first pass of B v_k = (w - B V a)/rho with B V a = V H a (Arnoldi):
 *       s_j = (c_j - sum_{i<k} H(j, i) a_i) / rho        (j = 0..k)
 *       u_{k+1} = (w - V_{0..k} c) / rho = (w - sum_{j<k} (b_j - e a_j) v_j - e u_k) / rho,
 *       e = c_k / rho
 *   Column k-1's residual estimate is known at step k, one matvec after it was
 *   started; the iteration count is the number of finished columns, as for MGS.
 *   A rho that is zero (or alpha - |a|^2 <= 0 in rounding) is a happy breakdown. */
static int gmres_dcgs2(const orc_op *A, const orc_op *M, const double *b, int64_t restart,
                       int64_t max_iters, double rtol, double atol, double *x, double *history,
                       int64_t hist_cap, orc_report *rep, double *V_out, int64_t *v_count) {
  int64_t n = A->n, m = restart;
  double *V = (double *)malloc(sizeof(double) * (size_t)((m + 1) * n));
  double *Hr = (double *)calloc((size_t)((m + 1) * m), sizeof(double)); /* unrotated */
  double *H = (double *)calloc((size_t)((m + 1) * m), sizeof(double));  /* rotated */
  double *cs = (double *)malloc(sizeof(double) * (size_t)m);
  double *sn = (double *)malloc(sizeof(double) * (size_t)m);
  double *g = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *yk = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *aa = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *bb = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *cc = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *s = (double *)malloc(sizeof(double) * (size_t)(m + 1));
  double *w = (double *)malloc(sizeof(double) * (size_t)n);
  double *t = (double *)malloc(sizeof(double) * (size_t)n);
  double *r = (double *)malloc(sizeof(double) * (size_t)n);
  double *vk = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  op_apply(M, b, r);
  double beta0 = sqrt(dot(n, r, r));
  rep->beta0 = beta0;
  double bnorm = sqrt(dot(n, b, b));
  int64_t it = 0;
  int converged = 0, status = ORC_OK;
  if (v_count) *v_count = 0;
  if (beta0 == 0.0) {
    converged = 1;
  } else {
    double tol = fmax(rtol * beta0, atol);
    for (;;) {
      for (int64_t i = 0; i < n; ++i) V[i] = r[i]; /* u_0 */
      int64_t k_end = 0;
      int done = 0;
      for (int64_t k = 0; k <= m; ++k) {
        double *u = &V[k * n];
        int more = k < m;
        if (more) {
          op_apply(A, u, t);
          op_apply(M, t, w);
        }
        for (int64_t j = 0; j < k; ++j) aa[j] = dot(n, &V[j * n], u);
        double alpha = dot(n, u, u), gamma = 0.0;
        if (more) {
          for (int64_t j = 0; j < k; ++j) bb[j] = dot(n, &V[j * n], w);
          gamma = dot(n, u, w);
        }
        double asq = 0.0;
        for (int64_t j = 0; j < k; ++j) asq += aa[j] * aa[j];
        double rho2 = alpha - asq;
        double rho = rho2 > 0.0 ? sqrt(rho2) : 0.0;
        if (!isfinite(rho)) { status = ORC_ENUMERIC; done = 1; k_end = k > 0 ? k - 1 : 0; break; }
        /* v_k = (u_k - sum_j a_j v_j) / rho */
        for (int64_t i = 0; i < n; ++i) {
          double v = u[i];
          for (int64_t j = 0; j < k; ++j) v -= aa[j] * V[j * n + i];
          vk[i] = rho > 0.0 ? v / rho : 0.0;
        }
        if (k == 0) {
          for (int64_t i = 0; i <= m; ++i) g[i] = 0.0;
          g[0] = rho;
        } else {
          int64_t kc = k - 1; /* finish column k-1 */
          for (int64_t j = 0; j < k; ++j) Hr[j * m + kc] = s[j] + aa[j];
          Hr[k * m + kc] = rho;
          for (int64_t j = 0; j <= k; ++j) H[j * m + kc] = Hr[j * m + kc];
          for (int64_t j = 0; j < kc; ++j) {
            double p = H[j * m + kc], q = H[(j + 1) * m + kc];
            H[j * m + kc] = cs[j] * p + sn[j] * q;
            H[(j + 1) * m + kc] = -sn[j] * p + cs[j] * q;
          }
          double p = H[kc * m + kc], q = H[k * m + kc];
          double den = hypot(p, q);
          cs[kc] = p / den;
          sn[kc] = q / den;
          H[kc * m + kc] = den;
          H[k * m + kc] = 0.0;
          g[k] = -sn[kc] * g[kc];
          g[kc] = cs[kc] * g[kc];
          ++it;
          if (it - 1 < hist_cap) history[it - 1] = fabs(g[k]) / beta0;
          k_end = k;
          int stop = 0;
          if (fabs(g[k]) <= tol || rho == 0.0) { converged = 1; stop = 1; }
          else if (it >= max_iters) stop = 1;
          if (stop) { /* slot k = v_k: the basis of the last cycle is complete (V_out) */
            memcpy(u, vk, sizeof(double) * (size_t)n);
            done = 1;
            break;
          }
        }
        if (!more) { memcpy(u, vk, sizeof(double) * (size_t)n); break; }
        /* the first pass of the next direction (u_k still unnormalised here) */
        double ab = 0.0;
        for (int64_t j = 0; j < k; ++j) ab += aa[j] * bb[j];
        for (int64_t j = 0; j < k; ++j) cc[j] = bb[j];
        cc[k] = (gamma - ab) / rho;
        for (int64_t j = 0; j <= k; ++j) {
          double ha = 0.0;
          for (int64_t i = 0; i < k; ++i) ha += Hr[j * m + i] * aa[i];
          s[j] = (cc[j] - ha) / rho;
        }
        double e = cc[k] / rho;
        double *un = &V[(k + 1) * n];
        for (int64_t i = 0; i < n; ++i) {
          double nx = w[i] - e * u[i];
          for (int64_t j = 0; j < k; ++j) nx -= (bb[j] - e * aa[j]) * V[j * n + i];
          un[i] = nx / rho;
        }
        memcpy(u, vk, sizeof(double) * (size_t)n);
      }
      if (V_out) {
        int64_t nv = k_end + 1;
        memcpy(V_out, V, sizeof(double) * (size_t)(nv * n));
        if (v_count) *v_count = nv;
      }
      for (int64_t i = k_end - 1; i >= 0; --i) {
        double sum = g[i];
        for (int64_t j = i + 1; j < k_end; ++j) sum -= H[i * m + j] * yk[j];
        yk[i] = sum / H[i * m + i];
      }
      for (int64_t j = 0; j < k_end; ++j)
        for (int64_t i = 0; i < n; ++i) x[i] += yk[j] * V[j * n + i];
      rep->resid_est = fabs(g[k_end]) / beta0;
      if (done) break;
      op_apply(A, x, t);
      for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
      op_apply(M, t, r);
      double beta = sqrt(dot(n, r, r));
      rep->restarts += 1;
      if (beta <= tol) { converged = 1; rep->resid_est = beta / beta0; break; }
    }
  }
  op_apply(A, x, t);
  for (int64_t i = 0; i < n; ++i) t[i] = b[i] - t[i];
  rep->resid_true = (bnorm > 0.0) ? sqrt(dot(n, t, t)) / bnorm : 0.0;
  op_apply(M, t, r);
  rep->resid_precond = (beta0 > 0.0) ? sqrt(dot(n, r, r)) / beta0 : 0.0;
  rep->iterations = it;
  rep->converged = converged;
  if (status == ORC_OK && !converged) status = ORC_NOT_CONVERGED;
  rep->status = status;
  free(V); free(Hr); free(H); free(cs); free(sn); free(g); free(yk); free(aa); free(bb);
  free(cc); free(s); free(w); free(t); free(r); free(vk);
  return status;
}

int orc_gmres(const orc_op *A, const orc_op *M, const double *b, int64_t restart,
              int64_t max_iters, double rtol, double atol, double *x, double *history,
              int64_t hist_cap, orc_report *rep, double *V_out, int64_t *v_count) {
  return orc_gmres_orth(A, M, b, restart, max_iters, rtol, atol, 0, x, history, hist_cap, rep,
                        V_out, v_count);
}

/* Convenience constructors used by the ctypes binding. */
void orc_op_identity(orc_op *op, int64_t n) {
  memset(op, 0, sizeof(*op)); op->kind = ORC_OP_IDENTITY; op->n = n;
}
void orc_op_dense(orc_op *op, int64_t n, const double *A) {
  memset(op, 0, sizeof(*op)); op->kind = ORC_OP_DENSE; op->n = n; op->A = A;
}
void orc_op_rbf(orc_op *op, int64_t n, const double *xy, double sigma, double rc,
                double x0, double y0, double x1, double y1, double cell, int brute) {
  memset(op, 0, sizeof(*op));
  op->kind = brute ? ORC_OP_RBF_BRUTE : ORC_OP_RBF;
  op->n = n; op->xy = xy; op->sigma = sigma; op->rc = rc;
  op->x0 = x0; op->y0 = y0; op->x1 = x1; op->y1 = y1; op->cell = cell;
}
/* the T-box operator of reading Q25 (cell-list form) */
void orc_op_rbf_tbox(orc_op *op, int64_t n, const double *xy, double sigma, double x0,
                     double y0, double x1, double y1, double cell, double tau) {
  memset(op, 0, sizeof(*op));
  op->kind = ORC_OP_RBF_TBOX;
  op->n = n; op->xy = xy; op->sigma = sigma; op->tau = tau;
  op->x0 = x0; op->y0 = y0; op->x1 = x1; op->y1 = y1; op->cell = cell;
}
void orc_op_rasm(orc_op *op, const orc_rasm *P, int asm_variant) {
  memset(op, 0, sizeof(*op)); op->kind = ORC_OP_RASM; op->n = P->n; op->P = P;
  op->asm_variant = asm_variant;
}
int64_t orc_op_size(void) { return (int64_t)sizeof(orc_op); }
int64_t orc_report_size(void) { return (int64_t)sizeof(orc_report); }
