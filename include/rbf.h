/*
 * rbf.h -- C ABI of librbf.so, the B200 (sm_100a) hot path of PetRBF
 * (Yokota, Barba, Knepley, "PetRBF -- A parallel O(N) algorithm for radial
 * basis function interpolation", arXiv 0909.5413; PAPER.md line numbers are
 * cited as P:<line>).
 *
 * The library solves the Gaussian RBF interpolation problem of Eqs.(1)-(4)
 * without polynomial part (the Gaussian is positive definite,
 * P:81):   A_rc lambda = f,   A_ij = exp(-|x_i-x_j|^2/(2 sigma^2))/(2 pi sigma^2)
 * (Eq.(12)) truncated to pairs with |x_i-x_j| < rc (reading
 * Q1 of DESIGN.md), by GMRES left-preconditioned with the restricted
 * additive Schwarz method M^-1 = sum_i R~_i^T A_i^-1 R_i (Eq.(11)),
 * one subdomain per cell of a uniform cell grid, overlap = rings of
 * neighbouring cells (reading Q9).
 *
 * Conventions (all entry points):
 *  - Every pointer argument named *_dev is DEVICE memory of the current CUDA
 *    device; *_host is host memory.  The caller owns every buffer it passes and
 *    keeps it alive until the stream work that uses it has completed.
 *  - All device work is enqueued on `stream` (a cudaStream_t passed as void*,
 *    NULL = legacy default stream); calls that return results to the host
 *    (reports, counts) synchronise that stream.
 *  - Vectors are RANK-LOCAL and in LIBRARY (cell-sorted) ORDER: entry s of a
 *    local vector belongs to caller point rbf_local_index()[s].  A single-GPU
 *    run has one rank owning all N points.
 *  - fp64 throughout.  N < 2^31.  A context is not thread-safe.
 *  - Return value: RBF_OK (0) on success, RBF_NOT_CONVERGED (2) when a solve
 *    stopped at max_iters (the last iterate is returned), or a
 *    negative error code; rbf_last_error() then holds a thread-local message.
 *    There is no CPU fallback: without a usable CUDA device every call fails
 *    with RBF_ECUDA.
 */
#ifndef RBF_H
#define RBF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rbf_ctx rbf_ctx; /* opaque, owned by the library */

enum {
  RBF_OK = 0,
  RBF_NOT_CONVERGED = 2,
  RBF_EINVAL = -1,      /* invalid argument (message names it)                    */
  RBF_ENOMEM = -2,      /* device allocation failed                                */
  RBF_ECUDA = -3,       /* CUDA runtime error                                      */
  RBF_ENCCL = -4,       /* NCCL error                                              */
  RBF_EFACTOR = -5,     /* zero pivot even after the LU fallback; message names the cell */
  RBF_ENUMERIC = -6,    /* NaN/Inf produced                                        */
  RBF_EUNSUPPORTED = -7 /* valid input this build does not handle (message says why) */
};

/* Geometry and kernel parameters (readings Q1, Q5, Q9).
 *  sigma          Gaussian width, > 0 (Eq.(12)).
 *  cell           cell side c > 0; cells tile the box from (x0, y0):
 *                 ncx = ceil((x1-x0)/c), ncy = ceil((y1-y0)/c);
 *                 cell of a point: cx = clamp(floor((x-x0)/c), 0, ncx-1), same for y;
 *                 cells are numbered key = cy*ncx + cx (row-major).
 *  rc             per-pair cutoff radius > 0: pair (i,j) enters A_rc iff
 *                 fma(dx,dx,dy*dy) < rc*rc (reading Q1).
 *  overlap_rings  >= 0: Omega_c = the (2r+1)^2 block of cells around cell c,
 *                 clipped to the grid (reading Q9); 0 = block Jacobi.
 *  schwarz        RBF_SCHWARZ_RASM (0, default): restricted additive Schwarz, Eq.(11)
 *                 (P:221-225), each subdomain writes its own points only.
 *                 RBF_SCHWARZ_ASM (1): additive Schwarz, Eq.(8), M^-1 =
 *                 sum_c R_c^T A_c^-1 R_c: every subdomain adds its whole local solution
 *                 (sums in ascending cell order, reading Q26).  Stores the full A_c^-1
 *                 (|Omega_c|^2 doubles per cell, ~9x the RASM blocks) and solves every
 *                 subdomain with the LU path.  Across strips the t_c entries of the
 *                 overlap_rings cell rows next to each strip edge are exchanged with the
 *                 neighbours (rbf_rasm_apply; the sums stay in ascending cell order, so
 *                 bitwise equal to one strip); needs overlap_width 0 there, and
 *                 rbf_rasm_apply_ext returns EUNSUPPORTED for it.
 *  x0,y0,x1,y1    domain box; every point must satisfy x0 <= x <= x1, y0 <= y <= y1.
 *  overlap_width  >= 0.  0: Omega_c is the whole block (above).  > 0: the paper's box
 *                 overlap ("overlapping subdomains of size D"; reading Q24):
 *                 Omega_c = own(c) and the block's points inside cell c's box grown
 *                 by overlap_width on every side (closed), in block order; D = cell +
 *                 2 overlap_width (D = 1.9 B: overlap_width = 0.45 cell).  Points
 *                 outside the block are never included (choose overlap_rings >=
 *                 overlap_width / cell).
 *  trunc_width    >= 0, <= 8 cell.  0: the matvec keeps the pairs with r < rc (Q1).  > 0:
 *                 the paper's T-box truncation ("an additional subdomain with
 *                 size T, which defines the non-zero entries for the matrix-vector
 *                 multiplication"; T = B + 4 sigma for h/sigma >= 0.9, B + 6 sigma at 0.8,
 *                 P:307, 348; reading Q25): row i of A keeps the sources inside target i's
 *                 cell box grown by trunc_width on every side (closed, edges as in Q24),
 *                 with no radial test; the matrix is then not symmetric.  It applies to
 *                 rbf_matvec, rbf_solve (A_T lambda = f), rbf_evaluate (the query's cell
 *                 box) and rbf_count_pairs; the preconditioner's local matrices stay the
 *                 principal submatrices of A_rc (rc still required). */
enum { RBF_SCHWARZ_RASM = 0, RBF_SCHWARZ_ASM = 1 };
typedef struct {
  double sigma;
  double cell;
  double rc;
  int32_t overlap_rings;
  int32_t schwarz;
  double x0, y0, x1, y1;
  double overlap_width;
  double trunc_width;
} rbf_params;

/* Domain decomposition into strips of cell rows.  The rows
 * are cut by a work model computed identically on every rank (per cell: n_own (0.28 S +
 * n_ov), S = points in the matvec stencil, n_ov = subdomain size -- matvec pairs plus
 * RASM apply entries), so a dense cluster is split across strips; on uniform data this
 * is the same as balancing points.
 *  rank, nranks   this process's strip and the strip count (1 <= nranks).
 *  comm           RBF_COMM_NCCL: halos/reductions go through an NCCL communicator
 *                 created from nccl_id (one process per GPU; the caller selects the
 *                 device first).  RBF_COMM_NONE: "virtual strip" -- the context owns
 *                 strip `rank` of `nranks` but never communicates; only the *_ext
 *                 entry points (caller-supplied halos) are usable.
 *                 RBF_COMM_THREADS: all nranks contexts live in ONE process on ONE
 *                 device, each driven by its own host thread (own stream); halos and
 *                 the reductions' all-gathers are device copies out of the peer
 *                 context, ordered by stream synchronisation and a host barrier.  Same
 *                 semantics and reduction order as NCCL; a transport for running and
 *                 checking the multi-strip path on one GPU, not a performance path.
 *                 Every collective call (rbf_matvec, rbf_rasm_apply, rbf_solve) must
 *                 be made by all nranks threads, or the callers block.
 *  nccl_id        NCCL: from rbf_get_nccl_id() on rank 0, broadcast by the caller.  The
 *                 first context set up with an id creates the communicator; later
 *                 contexts with the same id (same rank, rank count and device) reuse it --
 *                 a unique id seeds one communicator -- and it lives until process exit.
 *                 THREADS: any 128-byte key shared by the group's contexts. */
enum { RBF_COMM_NONE = 0, RBF_COMM_NCCL = 1, RBF_COMM_THREADS = 2 };
/* flags: RBF_DIST_NO_OVERLAP -- exchange the halo first, then apply the whole operator.
 * Default (0): rbf_matvec / rbf_rasm_apply / rbf_solve overlap the halo exchange with the
 * interior work -- the targets (matvec) and cells (RASM) whose stencils stay inside the
 * strip are computed while the halo is in flight (NCCL on a high-priority stream), the
 * ones next to a strip edge after it has arrived.  Results are bitwise
 * identical either way. */
enum { RBF_DIST_NO_OVERLAP = 1 };
typedef struct {
  int32_t rank;
  int32_t nranks;
  int32_t comm;
  int32_t flags;
  unsigned char nccl_id[128];
} rbf_dist;

/* GMRES parameters (reading Q12).
 *  restart    m >= 1 (30).      max_iters  >= 1 (1000).
 *  rtol, atol >= 0: stop when the recurrence residual |g_{k+1}| <= max(rtol*||M^-1 f||, atol).
 *  timing     nonzero: record per-phase CUDA-event times into the report (adds events).
 *  orth       Arnoldi orthogonalisation: RBF_ORTH_MGS (0, default; Q12, BJ:5),
 *             RBF_ORTH_CGS2 (classical Gram-Schmidt twice, reading Q23: 3 reductions per
 *             step instead of k+2) or RBF_ORTH_DCGS2 (CGS2 with the second pass delayed
 *             into the next step and Pythagorean normalisation, reading Q27: ONE reduction
 *             per step -- one all-gather across GPUs; a column's residual is known one
 *             operator application later).  CGS2/DCGS2 require restart <=
 *             RBF_CGS2_MAX_RESTART, else EINVAL. */
enum { RBF_ORTH_MGS = 0, RBF_ORTH_CGS2 = 1, RBF_ORTH_DCGS2 = 2 };
#define RBF_CGS2_MAX_RESTART 32
typedef struct {
  int32_t restart;
  int32_t max_iters;
  double rtol;
  double atol;
  int32_t timing;
  int32_t orth;
} rbf_gmres_params;

/* Solve report.  Residuals are relative: resid_est = |g|/||M^-1 f|| (recurrence),
 * resid_precond = ||M^-1(f - A lambda)||/||M^-1 f||, resid_true = ||f - A lambda||/||f||.
 * Phase times (ms, when timing != 0) follow the paper's breakdown.
 * history: optional caller array (host) of history_cap doubles receiving resid_est
 * after each iteration; history_len = entries written. */
typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t restarts;
  int32_t status;
  double resid_est, resid_precond, resid_true, beta0;
  double ms_setup, ms_matmult, ms_pcapply, ms_orth, ms_total;
  int64_t n_pairs;      /* in-cutoff pairs of this rank's rows (filled by rbf_count_pairs) */
  int64_t n_cells;      /* non-empty owned cells = subdomains of this rank */
  int64_t bytes_device; /* device bytes held by the context */
  double *history;
  int32_t history_cap;
  int32_t history_len;
} rbf_report;

/* NCCL unique id for a multi-GPU context (call on rank 0 only). */
int rbf_get_nccl_id(unsigned char out[128]);

/* Build the cell list, choose this rank's strip, and set up the
 * RASM preconditioner: per non-empty owned cell assemble A_c = R_c A_rc R_c^T,
 * factor it (Cholesky; LU with partial pivoting on breakdown, reading Q11)
 * and store the rows of A_c^-1 belonging to the cell's own points (PCSetUp).
 *  xy_dev  N x 2 interleaved fp64 (x0,y0,x1,y1,...) in caller order; every rank
 *          passes the full, identical point set.  Copied; may be freed afterwards.
 *  dist    NULL = single GPU.
 * Errors: EINVAL (n < 1, non-finite or out-of-box points, two points with equal
 * coordinates -- A is singular for repeated nodes, reading Q30 --, bad params, strips
 * thinner than the halo), ENOMEM, EFACTOR, ECUDA, ENCCL, EUNSUPPORTED (a
 * subdomain larger than this build's local-solve limit). */
int rbf_setup(rbf_ctx **ctx, const double *xy_dev, int64_t n, const rbf_params *p,
              const rbf_dist *dist, void *stream);

/* Rank-local sizes: owned points, and the extended range (owned + halo rows). */
int64_t rbf_local_count(const rbf_ctx *ctx);
int64_t rbf_ext_count(const rbf_ctx *ctx);
/* Position of this rank's owned / extended points in the GLOBAL sorted order:
 * out[0] = ext_lo, out[1] = own_lo, out[2] = own_hi, out[3] = ext_hi. */
int rbf_ranges(const rbf_ctx *ctx, int64_t out[4]);
/* idx_dev[s] (int64, rbf_local_count entries) = caller index of local entry s. */
int rbf_local_index(const rbf_ctx *ctx, int64_t *idx_dev, void *stream);
/* Global cell list export (tests): perm_dev (int64, N) = caller index of global sorted
 * entry s; cell_start_dev (int64, ncx*ncy+1).  dims_host[0..1] = ncx, ncy. */
int rbf_cell_list(const rbf_ctx *ctx, int64_t *perm_dev, int64_t *cell_start_dev,
                  int64_t dims_host[2], void *stream);
/* Permute a caller-order vector (N entries, device) into this rank's local order,
 * and back (scatter writes only this rank's entries). */
int rbf_to_local(const rbf_ctx *ctx, const double *v_caller_dev, double *v_loc_dev, void *stream);
int rbf_from_local(const rbf_ctx *ctx, const double *v_loc_dev, double *v_caller_dev, void *stream);

/* y = A_rc w on this rank's points (MatMult): halo exchange of w
 * (ceil(rc/c) cell rows from each strip neighbour; floor(trunc_width/c) + 1 rows
 * with the T-box) then the cutoff matvec (y = A_T w with the T-box, reading Q25). */
int rbf_matvec(rbf_ctx *ctx, const double *w_loc_dev, double *y_loc_dev, void *stream);
/* z = M^-1 r (PCApply / MatSolve, Eq.(10)-(11)): halo exchange of r
 * (overlap_rings rows), then z[own(c)] = (A_c^-1 R_c r)[own(c)] for every cell
 * (with RBF_SCHWARZ_ASM: t_c = A_c^-1 R_c r per cell, the boundary rows' t_c exchanged
 * with the neighbouring strips, then z_i = sum of the t_c entries of point i over the
 * subdomains containing it, ascending cell order, Eq.(8)). */
int rbf_rasm_apply(rbf_ctx *ctx, const double *r_loc_dev, double *z_loc_dev, void *stream);
/* Same two operators with the halo supplied by the caller: w_ext_dev holds
 * rbf_ext_count() entries = global sorted entries [ext_lo, ext_hi). */
int rbf_matvec_ext(rbf_ctx *ctx, const double *w_ext_dev, double *y_loc_dev, void *stream);
int rbf_rasm_apply_ext(rbf_ctx *ctx, const double *r_ext_dev, double *z_loc_dev, void *stream);

/* Solve A_rc lambda = f (KSPSolve): left-preconditioned restarted
 * GMRES(m) with modified Gram-Schmidt and Givens rotations, x0 = 0 (reading Q12).
 * f_loc_dev, lambda_loc_dev: rank-local, library order.  rep may be NULL.
 * A zero right-hand side returns lambda = 0 after 0 iterations. */
int rbf_solve(rbf_ctx *ctx, const double *f_loc_dev, const rbf_gmres_params *g,
              double *lambda_loc_dev, rbf_report *rep, void *stream);

/* One-call interpolation with HOST buffers in caller order (single GPU):
 * copies xy/f to the device, rbf_setup, rbf_solve, copies lambda back. */
int rbf_interpolate_host(const double *xy_host, const double *f_host, int64_t n,
                         const rbf_params *p, const rbf_gmres_params *g,
                         double *lambda_host, rbf_report *rep, void *stream);

/* Interpolant evaluation (the paper's application):
 *   s(q_k) = sum_{j : |q_k - x_j| < rc} lambda_j exp(-|q_k - x_j|^2/(2 sigma^2)) / (2 pi sigma^2)
 * (Eq.(1) P:76-79 with Eq.(12) and the truncation of reading Q1).
 *  q_xy_dev        m x 2 interleaved query points (any order), inside the box.
 *  lambda_loc_dev  weights, rank-local library order (e.g. rbf_solve's output).
 *  s_dev           m values, in the order of the queries.
 * Multi-rank: every rank passes all m queries; each evaluates the queries in its strip of
 * cell rows (its weights plus the matvec halo, exchanged here) and the results are summed
 * over the ranks (each query has one nonzero contribution, so the sum is exact), so every
 * rank receives all m values.  Collective: all ranks call it.  EINVAL for a query that is
 * non-finite or outside the box (message names the first one); EUNSUPPORTED on a virtual
 * strip (RBF_COMM_NONE).  Synchronises. */
int rbf_evaluate(rbf_ctx *ctx, const double *q_xy_dev, int64_t m, const double *lambda_loc_dev,
                 double *s_dev, void *stream);

/* In-cutoff (query, source) pair count of an evaluation (all ranks; for Gpairs/s). */
int rbf_evaluate_count_pairs(rbf_ctx *ctx, const double *q_xy_dev, int64_t m, int64_t *n_pairs,
                             void *stream);

/* In-cutoff pair count of this rank's rows (for Gpairs/s; synchronises). */
int rbf_count_pairs(rbf_ctx *ctx, int64_t *n_pairs, void *stream);

/* Deterministic local dot product and norm (GMRES building blocks, exported for
 * tests): *out_host = <a, b> over this rank's entries, summed in a fixed order. */
int rbf_dot(rbf_ctx *ctx, const double *a_dev, const double *b_dev, double *out_host, void *stream);

/* Strip planner (host only, no GPU): cell-row boundaries row_bounds[0..nranks]
 * for ncy rows with row_counts[r] points, balanced by cumulative count, each
 * strip at least min_rows rows.  Returns EINVAL if impossible. */
int rbf_plan_strips(const int64_t *row_counts, int64_t ncy, int32_t nranks, int64_t min_rows,
                    int64_t *row_bounds);

/* Context facts: out[0] = doubles stored in the X blocks (RASM apply streams
 * 8*out[0] bytes per application), out[1] = subdomains, out[2] = largest
 * |Omega_c|, out[3] = largest |own(c)| (rows of X per cell; |Omega_c| with ASM), out[4] = subdomains solved by the
 * global-memory LU path, out[5..6] = ncx, ncy, out[7] = device bytes held. */
int rbf_info(const rbf_ctx *ctx, int64_t out[8]);

/* Matvec layout facts: out[0] = lanes (target groups), out[1] = chunks of 32 lanes,
 * out[2] = neighbour-list entries stored (ELL, with padding; 4 bytes each),
 * out[3] = sum over lanes of the union-list lengths (entries without padding). */
int rbf_matvec_stats(const rbf_ctx *ctx, int64_t out[4]);

/* RASM setup facts (reading Q11): out[0] = subdomains solved by the global-memory LU
 * path, out[1] = of those, the ones factored with partial pivoting (Cholesky breakdowns
 * of the tensor-core pass, cells whose no-pivot factorisation met a non-positive pivot,
 * and every remaining cell when the probe wave of largest cells needed pivoting in more
 * than a quarter of cases).  EINVAL on NULL. */
int rbf_lu_stats(const rbf_ctx *ctx, int64_t out[2]);

/* Test hook (Krylov orthogonality, reading Q28): copy the first nvec vectors of the
 * context's GMRES basis workspace -- after rbf_solve, the basis v_0, v_1, ... of its last
 * restart cycle (MGS/CGS2: orthonormal vectors; DCGS2: slot k holds the unnormalised
 * first-pass vector of step k) -- into V_dev (nvec x rbf_local_count doubles, row-major,
 * device).  EINVAL when no solve has allocated the basis or nvec exceeds restart + 1.
 * Synchronises. */
int rbf_debug_krylov_basis(const rbf_ctx *ctx, double *V_dev, int32_t nvec, void *stream);

/* Test hook: fill the shared memory of every SM with 0xFF bytes (NaN in every double)
 * on the current device and synchronise, so that a following kernel that reads shared
 * memory it did not write produces NaN in the parity tests.  The option "poison" (below)
 * does the same for every device buffer the library allocates.  Changes no library
 * state.  ECUDA on a CUDA error. */
int rbf_debug_poison_shared(void);

/* Device time (ms, CUDA events) of rbf_setup's phases for this context:
 * out[0] = cell list, out[1] = positions + matvec neighbour list,
 * out[2] = RASM setup (assemble + factor + X), out[3] = whole rbf_setup. */
int rbf_setup_times(const rbf_ctx *ctx, double out[4]);

/* Number of kernel launches this library has issued so far (process-wide). */
int64_t rbf_launch_count(void);

/* Halo plan (host only, no GPU) used by rbf_setup for strip `rank`: row_start[r] =
 * global sorted position of the first point of cell row r (ncy+1 entries),
 * row_bounds from rbf_plan_strips, kh = ceil(rc/c) matvec halo rows, rings = RASM
 * overlap rings.  out = {ext_lo, own_lo, own_hi, ext_hi,
 *   below: send_off, send_cnt, recv_off, recv_cnt,   above: same four}
 * for the matvec halo (send offsets relative to the owned vector, receive offsets
 * relative to the extended vector [ext_lo, ext_hi)). */
int rbf_plan_halo(const int64_t *row_start, int64_t ncy, const int64_t *row_bounds, int32_t nranks,
                  int32_t rank, int32_t kh, int32_t rings, int64_t out[12]);

/* Device memory.  Buffers from 16 MB up that a context frees are kept by the library
 * (with an event on the freeing stream) and handed to the next context that asks for
 * the same size, so repeated setups of one configuration do not go back to the memory
 * pool's fit rules (which stalled cudaMallocAsync for 0.1-1 s at random steps on cfg4).
 * An allocation that fails returns them to the pool and retries.  rbf_trim_memory()
 * releases the kept buffers and trims the device's default memory pool to zero
 * (synchronises the device): call it before handing the memory to another allocator.
 * ECUDA without a device. */
int rbf_trim_memory(void);

/* Process-wide options: test and A/B switches of the hot path (the library reads no
 * environment variables).  None changes a result beyond rounding; the defaults are the
 * product path and are what every benchmark uses.  Read at rbf_setup / rbf_solve time;
 * set them between contexts, not concurrently with library calls on other threads.
 *   "poison"              0   1: NaN-fill every new device buffer (uninitialised reads)
 *   "lu_nopiv"            1   LU path: no-pivot first pass for cells routed there by size
 *                              (reading Q11); 0: partial pivoting for every LU cell
 *   "lu_smem_panel"       1   LU path: transposed panel in shared memory when it fits
 *   "mv_targets_per_lane" 2   matvec union lists of 1..3 targets per lane
 *   "mv_pair_targets"     1   matvec: nearest-neighbour target groups; 0: consecutive targets
 *   "mv_sort_lanes"       1   matvec: lanes sorted by list length within windows
 *   "mv_variant"          0   matvec kernel variant 0..5 (A/B measurements; 5: the
 *                              sources of each CTA staged in shared memory by bulk copies)
 *   "solve_graph"         1   single-rank solve as one CUDA graph; 0: host-driven loop
 *   "fused_arnoldi"       1   single-rank fused cooperative Arnoldi kernel; 0: per-step kernels
 *   "mgs_pairs"           1   fused MGS: two projections per grid barrier (reading Q28)
 *   "arnoldi_ctas_per_sm" 2   fused Arnoldi CTAs per SM (1..4)
 *   "log_slow_alloc"      0   diagnostics: report device allocations slower than N ms (stderr)
 *   "mv_index16"          0   1: 16-bit neighbour-list entries when every row offset fits (half
 *                              the list bytes; measured 8-10% slower)
 *   "setup_kernel"        0   RASM setup kernel for the tensor-core cells:
 *                              0 k_rasm_setup_tc, one factorisation per SM;
 *                              1 k_rasm_setup_tc2, two per SM, finished rows of L11 retired to
 *                                an L2 workspace (measured at parity with 0);
 *                              2 k_rasm_setup_tc3, factorisation of cell i and W / S^-1 / X of
 *                                cell i-1 pipelined on one SM
 * EINVAL for an unknown name or a value out of range. */
int rbf_set_option(const char *name, int64_t value);
int rbf_get_option(const char *name, int64_t *value);

const char *rbf_last_error(void);
void rbf_destroy(rbf_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* RBF_H */
