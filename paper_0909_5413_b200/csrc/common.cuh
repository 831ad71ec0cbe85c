// common.cuh -- internal declarations shared by the librbf.so translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Boundary").
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../include/rbf.h"

namespace rbf {

void set_error(const char *fmt, ...);
void count_launch(int k);  // kernel launches issued by this library (rbf_launch_count)

#define RBF_CUDA_TRY(call)                                                               \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      ::rbf::set_error("CUDA error %s (%s) at %s:%d", cudaGetErrorString(e_), #call,      \
                       __FILE__, __LINE__);                                              \
      return (e_ == cudaErrorMemoryAllocation) ? RBF_ENOMEM : RBF_ECUDA;                 \
    }                                                                                    \
  } while (0)

#define RBF_NCCL_TRY(call)                                                               \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      ::rbf::set_error("NCCL error %s (%s) at %s:%d", ncclGetErrorString(r_), #call,      \
                       __FILE__, __LINE__);                                              \
      return RBF_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

// Process-wide library options (rbf_set_option, include/rbf.h): test and A/B switches
// that never change results beyond rounding; the defaults are the product path.
enum Opt {
  OPT_POISON = 0,        // NaN-fill every new device buffer (uninitialised-read tests)
  OPT_LU_NOPIV,          // LU path: no-pivot first pass for cells routed by size (1)
  OPT_LU_SMEM_PANEL,     // LU path: transposed panel in shared memory when it fits (1)
  OPT_MV_G,              // matvec targets per lane (union lists), 1..3 (2)
  OPT_MV_PAIR,           // matvec: nearest-neighbour target groups (1) or consecutive (0)
  OPT_MV_SORT,           // matvec: lanes sorted by list length in windows (1)
  OPT_MV_VARIANT,        // matvec kernel variant for A/B measurements (0)
  OPT_SOLVE_GRAPH,       // single-rank solve as one CUDA graph (1) or host-driven loop (0)
  OPT_FUSED_ARNOLDI,     // single-rank fused cooperative Arnoldi kernel (1)
  OPT_MGS_PAIRS,         // fused MGS: two projections per grid barrier (1, reading Q28)
  OPT_ARNOLDI_PER_SM,    // fused Arnoldi: CTAs per SM (2)
  OPT_LOG_SLOW_ALLOC,    // diagnostics: log device allocations slower than this many ms (0 = off)
  OPT_MV_INDEX16,        // matvec: 16-bit neighbour-list entries when they fit (0: measured slower)
  OPT_SETUP_KERNEL,      // RASM setup kernel: 0 one factorisation per SM, 1 two per SM, 2 pipelined post phase
  OPT_COUNT
};
long long opt(Opt o);

// Raise kernel `fn`'s dynamic shared-memory limit on the current device to at least
// `bytes` (thread-safe, never lowers it): a per-device high-water mark under a mutex, so
// a launch that needs `bytes` cannot see another host thread lower the attribute
// between this call and the launch (concurrent contexts, RBF_COMM_THREADS).
int ensure_dyn_smem(const void *fn, size_t bytes);

#define RBF_TRY(call)          \
  do {                         \
    int s_ = (call);           \
    if (s_ < 0) return s_;     \
  } while (0)

// Kernel-side geometry (passed by value).  See rbf.h rbf_params and DESIGN.md Q1, Q5, Q9.
struct Geom {
  double x0, y0, x1, y1, cell;
  double rc2;          // rc*rc, computed once on the host (reading Q1)
  double neg_inv_2s2;  // -1 / (2 sigma^2)
  double esc;          // -log2(e) / (2 sigma^2): matvec exp argument in powers of 2
  double esc64;        // 64 * esc (table variant)
  double norm;         // 1 / (2 pi sigma^2), hoisted out of the pair sum (reading Q2)
  int ncx, ncy;
  int kh;              // matvec search rings = ceil(rc/c), bumped on near-integral rc/c
  int rings;           // RASM overlap rings
  double ovw;          // box overlap width delta (reading Q24); 0 = whole rings
  double tw;           // T-box truncation width tau (reading Q25); 0 = radial cutoff rc
  int asm_full;        // 1: additive Schwarz, Eq.(8) (full A_c^-1 per cell, reading Q26)
};

// Cell (cx, cy)'s box grown by w on every side, closed (readings Q24, Q25); the
// edges are x0 + cx*c rounded twice (no contraction), exactly as in the oracle.
struct CellBox {
  double lx, hx, ly, hy;
};
__device__ __forceinline__ CellBox cell_box(const Geom &g, int cx, int cy, double w) {
  CellBox b;
  b.lx = __dsub_rn(__dadd_rn(g.x0, __dmul_rn((double)cx, g.cell)), w);
  b.hx = __dadd_rn(__dadd_rn(g.x0, __dmul_rn((double)(cx + 1), g.cell)), w);
  b.ly = __dsub_rn(__dadd_rn(g.y0, __dmul_rn((double)cy, g.cell)), w);
  b.hy = __dadd_rn(__dadd_rn(g.y0, __dmul_rn((double)(cy + 1), g.cell)), w);
  return b;
}
__device__ __forceinline__ bool in_box(const CellBox &b, double x, double y) {
  return x >= b.lx && x <= b.hx && y >= b.ly && y <= b.hy;
}

// Per-cell overlap index lists of the box-overlap subdomains (ovw > 0): the global
// sorted indices of Omega_c in block order (idx[off[cl] ..]), own(c)'s position
// inside it (own[cl]).  idx == nullptr: Omega_c is the whole block.
struct OvList {
  const int *idx;
  const long long *off;
  const int *own;
};

// This rank's strip of cell rows and its position in the global sorted order.
struct Strip {
  int row_lo, row_hi;        // owned cell rows [row_lo, row_hi)
  int ext_row_lo, ext_row_hi;  // rows covered by the extended (halo) range
  long long ext_lo, own_lo, own_hi, ext_hi;  // global sorted positions
};

constexpr int kRedBlocks = 592;   // 4 x 148 SMs: fixed grid for deterministic reductions
constexpr int kRedThreads = 512;

struct ThreadGroup;  // RBF_COMM_THREADS rendezvous (comm.cu)

struct Halo {  // one direction of a halo exchange, in element offsets
  long long send_off, send_cnt;  // relative to the owned (local) vector
  long long recv_off, recv_cnt;  // relative to the ext vector
};


// exp(x) for x <= 0 on the FP64 pipe with a 64-entry table (reading Q15: <= 2 ulp;
// measured max 1 ulp against CUDA exp() over [-18.5, 0], tools/micro.cu):
//   k = round(64 x / ln2),  r = x - k ln2/64 (Cody-Waite, ln2/64 = L_HI + L_LO,
//   L_HI with 32 trailing zero bits so k*L_HI is exact),  |r| <= ln2/128,
//   exp(x) = 2^(k>>6) * T[k & 63] * (1 + r + r^2/2 + ... + r^5/120).
// 10 FP64 instructions + one cached table load, vs ~22 for exp().  x < -707 returns 0
// (the true value is below 1e-307).
static __device__ const double kExp2Tab64[64] = {
1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

__device__ __forceinline__ double exp_neg(double x) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer shifter
  const double kInvL = 92.33248261689366;    // 64 / ln2
  const double kLHi = 0.010830417275428772;  // ln2/64, high part (32 trailing zero bits)
  const double kLLo = 7.420820373486988e-09; // ln2/64 - kLHi
  if (x < -707.0) return 0.0;
  const double t = fma(x, kInvL, kMagic);
  const double kd = t - kMagic;
  const int k = __double2loint(t);
  double r = fma(kd, -kLHi, x);
  r = fma(kd, -kLLo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = r * p;
  const double T = __ldg(&kExp2Tab64[k & 63]);
  const double e = fma(T, p, T);
  return __hiloint2double(__double2hiint(e) + ((k >> 6) << 20), __double2loint(e));
}

// ---------------------------------------------------------------------------
// Table-free exp for the cutoff Gaussian (matvec, evaluation); reading Q15.
// ---------------------------------------------------------------------------
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-integer shifter
constexpr int kExpDeg = 9;  // polynomial degree of the default matvec / evaluation exp

// 2^f = 1 + f P(f) on [-1/2, 1/2]: minimax P (Remez on the relative error, DESIGN.md
// §6), highest coefficient first.  Degree 10: max error 1.5e-16; degree 9: 3.9e-16.
static __constant__ double kExp2P10[11] = {4.078071929588337e-10, 7.072570412814423e-09,
                                    1.0180647659234139e-07, 1.3215442675329823e-06,
                                    1.5252727385193868e-05, 0.0001540353044157213,
                                    0.0013333558153439966, 0.009618129107607003,
                                    0.05550410866479039, 0.24022650695910097,
                                    0.6931471805599457};
static __constant__ double kExp2P9[10] = {7.111758687557852e-09, 1.0210506458816145e-07,
                                   1.321523563477604e-06, 1.525264774769592e-05,
                                   0.00015403530800818256, 0.001333355824648072,
                                   0.009618129107380715, 0.05550410866434658,
                                   0.24022650695910472, 0.6931471805599516};

// exp(-r2/(2 sigma^2)) for 0 <= r2 < rc^2 (rc <= 37 sigma, so the result is a normal
// number > 2^-990 and no underflow guard is needed).  esc = -log2(e)/(2 sigma^2).
template <int DEG>
__device__ __forceinline__ double gauss_exp2(double r2, double esc) {
  const double t = fma(r2, esc, kMagic);
  const double kd = t - kMagic;
  const int k = __double2loint(t);
  const double f = fma(r2, esc, -kd);  // exact product, one rounding: |f| <= 1/2
  const double *P = DEG == 10 ? kExp2P10 : kExp2P9;
  double p = P[0];
#pragma unroll
  for (int i = 1; i <= DEG; ++i) p = fma(p, f, P[i]);
  const double q = fma(f, p, 1.0);
  return __hiloint2double(__double2hiint(q) + k * (1 << 20), __double2loint(q));
}

__device__ __forceinline__ double4 ld_rec(const double4 *p) {  // one 256-bit gather
  double4 v;
  asm volatile("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}

}  // namespace rbf

struct rbf_ctx {
  rbf_params p{};
  rbf::Geom g{};
  rbf::Strip s{};
  long long n = 0;
  int rank = 0, nranks = 1, comm_mode = RBF_COMM_NONE;
  ncclComm_t nccl = nullptr;
  rbf::ThreadGroup *tgroup = nullptr;  // RBF_COMM_THREADS (comm.cu)
  std::vector<long long> row_start;  // host: global sorted position of the first point of each cell row
  rbf::Halo halo_mv[2]{}, halo_pc[2]{};  // [0] = with rank-1 (below), [1] = with rank+1 (above)

  // device: cell list (global)
  int *cell_start = nullptr;   // ncx*ncy+1
  int *perm = nullptr;         // N: caller index of global sorted entry
  double2 *xy_ext = nullptr;   // positions of the ext range, sorted
  // RASM
  long long *x_off = nullptr;  // per owned cell (ncx * owned rows + 1), in doubles
  int *ov_idx = nullptr;       // box-overlap index lists (OvList), when g.ovw > 0
  long long *ov_off = nullptr;
  int *ov_own = nullptr;
  double *X = nullptr;         // rows of A_c^-1 for own(c), row-major, ld = n_ov rounded up to even
                               // (ASM: all n_ov rows of A_c^-1)
  long long *asm_toff = nullptr;  // ASM: offset of cell cl's local solution t_c (sum of n_ov)
  double *asm_t = nullptr;        // ASM: the local solutions t_c = A_c^-1 R_c u
  int *asm_map = nullptr;         // ASM: per point, the t entries that sum to z_i (cell order)
  long long *asm_poff = nullptr;  // ASM: CSR offsets of asm_map (n_loc + 1)
  long long asm_sb = 0;           // ASM across strips: asm_t = [t of the rings rows below the strip
                                  // (sb entries, from rank-1) | own cells' t | rows above (rank+1)]
  rbf::Halo halo_asm[2]{};        // ASM: exchange of the boundary rows' t with the neighbours
  long long x_count = 0;
  int max_ov = 0, max_own = 0, nsub = 0, n_lu = 0;
  int n_lu_pivot = 0;          // LU-path subdomains that needed row exchanges
  int max_cell = 0;            // largest cell population (all cells of the ext range)
  // matvec: packed source records {x, y, w, 0} (ext range) and the neighbour list
  // (ELL of 32-bit entries in groups of 4, chunks of 32 consecutive owned targets)
  double4 *rec = nullptr;
  int mv_var = 0;              // matvec kernel variant (A/B measurements only)
  int mv_g = 2;                // targets per lane (union lists with per-target mask bits)
  long long mv_lanes = 0;      // lanes (target pairs) of the owned range
  int4 *lane_tgt = nullptr;    // per lane: its G local targets (-1 = none), nearest-neighbour groups
  int nchunks = 0;
  int *chunk_len = nullptr;    // per chunk: list length (max over its lanes, multiple of 4)
  long long *chunk_off = nullptr;  // per chunk (+1): first entry
  void *nlist = nullptr;       // 32-bit: source index (ext-relative sorted order) | target mask bits;
                               // 16-bit (mv_w16): mask bits | row step | offset in the row's run
  int mv_w16 = 0;
  int4 *mv_win = nullptr;      // matvec variant 5: per CTA, the staged source window (bx0, bx1, by0, by1; x < 0: none)
  long long nlist_entries = 0;  // ELL entries including padding
  long long nlist_union = 0;    // sum over lanes of the union-list lengths
  // workspaces
  double *w_ext = nullptr;     // n_ext (multi-rank only)
  // multi-rank overlap of the halo exchange with the interior work
  int overlap = 0;             // 1 unless rbf_dist.flags has RBF_DIST_NO_OVERLAP
  long long mv_int_chunks = 0; // matvec: chunks [0, mv_int_chunks) need no halo
  cudaStream_t s_comm = nullptr;  // NCCL: high-priority stream of the halo exchange
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
  double *V = nullptr;         // (restart+1) x n_loc Krylov basis
  int V_m = 0;
  double *t1 = nullptr, *t2 = nullptr;
  double *red_part = nullptr;  // kRedBlocks
  unsigned *red_count = nullptr;
  double *dscal = nullptr;     // device scalars (see krylov.cu)
  double *hpin = nullptr;      // pinned, mapped host scalars: [0..2] GMRES mailbox, [8..] readbacks
  double *hpin_dev = nullptr;  // device alias of hpin
  int ar_grid = 0;             // CTAs of the fused single-rank Arnoldi kernel (0 = unused)
  double *ar_part = nullptr;   // its per-CTA partial sums
  unsigned *ar_bar = nullptr;  // its grid barrier (count, generation)
  int ar_m = 0;                // restart length ar_part is sized for
  int cg_grid = 0;             // CTAs of the fused CGS2 Arnoldi kernel (0 = unused)
  double *cg_blk = nullptr;    // multi-kernel CGS2 per-block partials (kRedBlocks x 32)
  double *dc_blk = nullptr;    // DCGS2 block-dot per-block partials (kRedBlocks x (2 m + 2))
  unsigned *cg_count = nullptr;
  int g_orth = -1;             // orthogonalisation the solve graph was built for
  // graph-driven solve (single rank): the whole restarted GMRES as one CUDA graph with
  // device-side while loops (conditional nodes), built per restart length
  cudaGraph_t g_graph = nullptr;
  cudaGraphExec_t g_exec = nullptr;
  int g_m = 0, g_hist_cap = 0;
  const double *g_V = nullptr;  // V the graph was built for
  void *g_state = nullptr;      // GState (krylov.cu)
  double *g_hist = nullptr;     // per-iteration residual estimates
  double *g_f = nullptr, *g_x = nullptr;  // the graph's right-hand side and iterate
  long long bytes = 0;
  double setup_ms[4] = {0, 0, 0, 0};
  cudaStream_t last_stream = nullptr;
};

namespace rbf {

long long n_loc(const rbf_ctx *c);
long long n_ext(const rbf_ctx *c);
int owned_cells(const rbf_ctx *c);

// device allocation helpers (stream-ordered pool allocator)
int dalloc(rbf_ctx *c, void **p, size_t bytes, cudaStream_t s);
void dfree(void *p, cudaStream_t s);

// Scratch buffers freed (stream-ordered) when the guard goes out of scope, so early
// error returns (RBF_TRY) do not leak them.
struct ScratchGuard {
  cudaStream_t s;
  std::vector<void *> ptrs;
  explicit ScratchGuard(cudaStream_t s_) : s(s_) {}
  template <class T> int alloc(rbf_ctx *c, T **p, size_t bytes) {
    int st = dalloc(c, (void **)p, bytes, s);
    if (st == RBF_OK) ptrs.push_back((void *)*p);
    return st;
  }
  ~ScratchGuard() {
    for (void *p : ptrs) dfree(p, s);
  }
};

// cells.cu
int build_cell_list(rbf_ctx *c, const double *xy_caller, cudaStream_t s);
int row_costs(rbf_ctx *c, cudaStream_t s, std::vector<long long> &out);  // strip cost per cell row
int count_pairs(rbf_ctx *c, long long *out, cudaStream_t s);
int launch_to_local(const rbf_ctx *c, const double *v_caller, double *v_loc, cudaStream_t s);
int launch_from_local(const rbf_ctx *c, const double *v_loc, double *v_caller, cudaStream_t s);
int launch_local_index(const rbf_ctx *c, int64_t *idx, cudaStream_t s);

// matvec.cu
int build_nlist(rbf_ctx *c, cudaStream_t s);
int launch_pack_range(const rbf_ctx *c, const double *src, long long cnt, long long off, cudaStream_t s);
// prepacked: w already in the records' w slot; part 0 = all targets, 1 = interior lanes,
// 2 = boundary lanes (multi-rank overlap: only the boundary lanes read the halo)
int launch_matvec(const rbf_ctx *c, const double *w_ext, double *y_loc, cudaStream_t s,
                  bool prepacked = false, int part = 0);
int launch_pack_w(const rbf_ctx *c, const double *w_ext, cudaStream_t s);

// evaluate.cu
// pairs_out: count the in-cutoff (query, source) pairs instead of evaluating
int evaluate(rbf_ctx *c, const double *q, long long m, const double *lam, double *out, cudaStream_t s,
             unsigned long long *pairs_out = nullptr);

// rasm.cu
int rasm_setup(rbf_ctx *c, cudaStream_t s);
int probe_read(long long *out);  // RBF_PROBE builds only
// part 0 = every cell, 1 = the interior cells, 2 = the cells within overlap_rings rows of
// a strip edge with a neighbour rank (only these read the halo)
int launch_asm_local(const rbf_ctx *c, const double *r_ext, cudaStream_t s);  // Eq.(8) t_c, own cells
int launch_asm_gather(const rbf_ctx *c, double *z_loc, cudaStream_t s);      // Eq.(8) sums
int launch_rasm_apply(const rbf_ctx *c, const double *r_ext, double *z_loc, cudaStream_t s, int part = 0);

// comm.cu
int comm_init(rbf_ctx *c, const rbf_dist *d);
void comm_destroy(rbf_ctx *c);
int halo_exchange(rbf_ctx *c, const double *v_loc, double *v_ext, bool matvec_depth, cudaStream_t s);
int allgather_scalars(rbf_ctx *c, const double *send, double *recv, int count, cudaStream_t s);
// v (count doubles, device) <- the sum of every rank's v, summed in rank order (THREADS)
// or by ncclAllReduce (callers use it only where at most one rank holds a nonzero per
// entry, so the sum is exact in any order)
int allreduce_vector(rbf_ctx *c, double *v, long long count, cudaStream_t s);
// The two operators across strips: halo exchange overlapped with the interior work
// (interior lanes / cells while the halo is in flight, then the boundary ones); without
// overlap (RBF_DIST_NO_OVERLAP) exchange first, then the whole operator.
int dist_matvec(rbf_ctx *c, const double *w_loc, double *y_loc, cudaStream_t s);
int dist_rasm_apply(rbf_ctx *c, const double *r_loc, double *z_loc, cudaStream_t s);

// krylov.cu
int solve_gmres(rbf_ctx *c, const double *f, const rbf_gmres_params *g, double *x,
                rbf_report *rep, cudaStream_t s);
int dot_host(rbf_ctx *c, const double *a, const double *b, double *out, cudaStream_t s);
int prebuild_solve(rbf_ctx *c, cudaStream_t s);  // GMRES workspace + solve graph (rbf_setup)

}  // namespace rbf
