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
  double norm;         // 1 / (2 pi sigma^2), hoisted out of the pair sum (reading Q2)
  int ncx, ncy;
  int kh;              // matvec search rings = ceil(rc/c), bumped on near-integral rc/c
  int rings;           // RASM overlap rings
};

// This rank's strip of cell rows and its position in the global sorted order.
struct Strip {
  int row_lo, row_hi;        // owned cell rows [row_lo, row_hi)
  int ext_row_lo, ext_row_hi;  // rows covered by the extended (halo) range
  long long ext_lo, own_lo, own_hi, ext_hi;  // global sorted positions
};

constexpr int kRedBlocks = 296;   // 2 x 148 SMs: fixed grid for deterministic reductions
constexpr int kRedThreads = 256;

struct Halo {  // one direction of a halo exchange, in element offsets
  long long send_off, send_cnt;  // relative to the owned (local) vector
  long long recv_off, recv_cnt;  // relative to the ext vector
};

}  // namespace rbf

struct rbf_ctx {
  rbf_params p{};
  rbf::Geom g{};
  rbf::Strip s{};
  long long n = 0;
  int rank = 0, nranks = 1, comm_mode = RBF_COMM_NONE;
  ncclComm_t nccl = nullptr;
  std::vector<long long> row_start;  // host: global sorted position of the first point of each cell row
  rbf::Halo halo_mv[2]{}, halo_pc[2]{};  // [0] = with rank-1 (below), [1] = with rank+1 (above)

  // device: cell list (global)
  int *cell_start = nullptr;   // ncx*ncy+1
  int *perm = nullptr;         // N: caller index of global sorted entry
  double2 *xy_ext = nullptr;   // positions of the ext range, sorted
  // RASM
  long long *x_off = nullptr;  // per owned cell (ncx * owned rows + 1), in doubles
  double *X = nullptr;         // rows of A_c^-1 for own(c), row-major, ld = n_ov rounded up to even
  long long x_count = 0;
  int max_ov = 0, max_own = 0, nsub = 0, n_lu = 0;
  // workspaces
  double *w_ext = nullptr;     // n_ext (multi-rank only)
  double *V = nullptr;         // (restart+1) x n_loc Krylov basis
  int V_m = 0;
  double *t1 = nullptr, *t2 = nullptr;
  double *red_part = nullptr;  // kRedBlocks
  unsigned *red_count = nullptr;
  double *dscal = nullptr;     // device scalars (see krylov.cu)
  double *hpin = nullptr;      // pinned host scalars
  long long bytes = 0;
  cudaStream_t last_stream = nullptr;
};

namespace rbf {

long long n_loc(const rbf_ctx *c);
long long n_ext(const rbf_ctx *c);
int owned_cells(const rbf_ctx *c);

// device allocation helpers (stream-ordered pool allocator)
int dalloc(rbf_ctx *c, void **p, size_t bytes, cudaStream_t s);
void dfree(void *p, cudaStream_t s);

// cells.cu
int build_cell_list(rbf_ctx *c, const double *xy_caller, cudaStream_t s);
int count_pairs(rbf_ctx *c, long long *out, cudaStream_t s);
int launch_to_local(const rbf_ctx *c, const double *v_caller, double *v_loc, cudaStream_t s);
int launch_from_local(const rbf_ctx *c, const double *v_loc, double *v_caller, cudaStream_t s);
int launch_local_index(const rbf_ctx *c, int64_t *idx, cudaStream_t s);

// matvec.cu
int launch_matvec(const rbf_ctx *c, const double *w_ext, double *y_loc, cudaStream_t s);

// rasm.cu
int rasm_setup(rbf_ctx *c, cudaStream_t s);
int launch_rasm_apply(const rbf_ctx *c, const double *r_ext, double *z_loc, cudaStream_t s);

// comm.cu
int comm_init(rbf_ctx *c, const rbf_dist *d);
void comm_destroy(rbf_ctx *c);
int halo_exchange(rbf_ctx *c, const double *v_loc, double *v_ext, bool matvec_depth, cudaStream_t s);
int allgather_scalars(rbf_ctx *c, const double *send, double *recv, int count, cudaStream_t s);

// krylov.cu
int solve_gmres(rbf_ctx *c, const double *f, const rbf_gmres_params *g, double *x,
                rbf_report *rep, cudaStream_t s);
int dot_host(rbf_ctx *c, const double *a, const double *b, double *out, cudaStream_t s);

}  // namespace rbf
