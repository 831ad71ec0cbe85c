// api.cu -- the C ABI of librbf.so (include/rbf.h): context lifecycle, validation,
// strip planning, and the thin wrappers around the kernels.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <string>

#include "common.cuh"

#include <map>
#include <mutex>
#include <unordered_map>

namespace rbf {

static thread_local std::string g_err;
static std::mutex g_alloc_mu;  // live device bytes per context (dalloc / dfree)
static std::unordered_map<void *, std::pair<rbf_ctx *, long long>> g_allocs;
static std::atomic<long long> g_launches{0};

void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

struct OptDef {
  const char *name;
  long long dflt, lo, hi;
};
static const OptDef kOptDefs[OPT_COUNT] = {
    {"poison", 0, 0, 1},         {"lu_nopiv", 1, 0, 1},    {"lu_smem_panel", 1, 0, 1},
    {"mv_targets_per_lane", 2, 1, 3}, {"mv_pair_targets", 1, 0, 1}, {"mv_sort_lanes", 1, 0, 1},
    {"mv_variant", 0, 0, 5},     {"solve_graph", 1, 0, 1}, {"fused_arnoldi", 1, 0, 1},
    {"mgs_pairs", 1, 0, 1},      {"arnoldi_ctas_per_sm", 2, 1, 4},
    {"log_slow_alloc", 0, 0, 1000000}, {"mv_index16", 0, 0, 1},
    {"setup_kernel", 0, 0, 2},
};
static std::atomic<long long> g_opt[OPT_COUNT] = {};
static std::once_flag g_opt_init;

static void opt_init() {
  std::call_once(g_opt_init, [] {
    for (int i = 0; i < OPT_COUNT; ++i) g_opt[i].store(kOptDefs[i].dflt);
  });
}

long long opt(Opt o) {
  opt_init();
  return g_opt[o].load(std::memory_order_relaxed);
}

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

long long n_loc(const rbf_ctx *c) { return c->s.own_hi - c->s.own_lo; }
long long n_ext(const rbf_ctx *c) { return c->s.ext_hi - c->s.ext_lo; }
int owned_cells(const rbf_ctx *c) { return (c->s.row_hi - c->s.row_lo) * c->g.ncx; }

// Stream-ordered allocations from the device's default memory pool.  The pool keeps
// freed memory (release threshold = max), so repeated setup/solve cycles do not
// return memory to the driver between steps.
//
// Buffers from 16 MB up (the X blocks, the neighbour list, the Krylov basis, ...) are
// recycled by the library itself: a freed big buffer is kept with an event recorded on
// the freeing stream, and a later request of the same size (within 1/8) takes it back
// after waiting on that event.  The pool alone picks blocks by its own fit rules, and a
// setup whose 19 GB neighbour list landed inside the previous context's 90 GB X block
// had to map fresh memory for the next X -- 0.1-1 s stalls in cudaMallocAsync on cfg4,
// at random steps (measured).  A failed allocation returns the cached
// buffers to the pool and retries once; rbf_trim_memory() releases everything.
constexpr size_t kCacheMin = 16ull << 20;
constexpr size_t kCacheCap = 140ull << 30;  // bytes kept for reuse at most
struct CachedBuf {
  void *p;
  size_t bytes;
  int dev;
  cudaEvent_t ev;
};
static std::mutex g_cache_mu;
static std::vector<CachedBuf> g_cache;               // oldest first
static std::unordered_map<void *, std::pair<size_t, int>> g_big;  // live big buffers

static void cache_release(CachedBuf &b, cudaStream_t s) {  // caller holds g_cache_mu
  cudaStreamWaitEvent(s, b.ev, 0);
  cudaEventDestroy(b.ev);
  cudaFreeAsync(b.p, s);
}

int dalloc(rbf_ctx *c, void **p, size_t bytes, cudaStream_t s) {
  static std::once_flag pool_configured;
  std::call_once(pool_configured, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  if (bytes == 0) bytes = 16;
  int dev = 0;
  cudaGetDevice(&dev);
  *p = nullptr;
  if (bytes >= kCacheMin) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int best = -1;
    for (int i = 0; i < (int)g_cache.size(); ++i) {
      const CachedBuf &b = g_cache[i];
      if (b.dev == dev && b.bytes >= bytes && b.bytes <= bytes + bytes / 8 &&
          (best < 0 || b.bytes < g_cache[best].bytes))
        best = i;
    }
    if (best >= 0) {
      CachedBuf b = g_cache[best];
      g_cache.erase(g_cache.begin() + best);
      cudaStreamWaitEvent(s, b.ev, 0);  // the previous owner's work on it is done
      cudaEventDestroy(b.ev);
      *p = b.p;
      g_big[b.p] = {b.bytes, dev};
    }
  }
  if (!*p) {
    const long long slow = opt(OPT_LOG_SLOW_ALLOC);
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e == cudaErrorMemoryAllocation) {  // hand the cached buffers back and retry
      (void)cudaGetLastError();
      {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto &b : g_cache) cache_release(b, s);
        g_cache.clear();
      }
      e = cudaMallocAsync(p, bytes, s);
    }
    if (slow > 0) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms >= (double)slow) fprintf(stderr, "librbf: cudaMallocAsync(%zu B) took %.1f ms\n", bytes, ms);
    }
    if (e != cudaSuccess) {
      *p = nullptr;
      set_error("device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? RBF_ENOMEM : RBF_ECUDA;
    }
    if (bytes >= kCacheMin) {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      g_big[*p] = {bytes, dev};
    }
  }
  // test hook: every new buffer filled with 0xFF bytes (a NaN in every double), so a
  // kernel reading scratch it never wrote shows up in the parity tests
  if (opt(OPT_POISON)) cudaMemsetAsync(*p, 0xFF, bytes, s);
  if (c) {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    c->bytes += (long long)bytes;
    g_allocs[*p] = {c, (long long)bytes};
  }
  return RBF_OK;
}

// c->bytes counts the bytes a context holds NOW: dfree subtracts what dalloc added
void dfree(void *p, cudaStream_t s) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_allocs.find(p);
    if (it != g_allocs.end()) {
      it->second.first->bytes -= it->second.second;
      g_allocs.erase(it);
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_big.find(p);
    if (it != g_big.end()) {
      CachedBuf b{p, it->second.first, it->second.second, nullptr};
      g_big.erase(it);
      if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(b.ev, s) == cudaSuccess) {
        g_cache.push_back(b);
        size_t tot = 0;
        for (auto &x : g_cache) tot += x.bytes;
        while (tot > kCacheCap && !g_cache.empty()) {  // oldest first
          tot -= g_cache.front().bytes;
          cache_release(g_cache.front(), s);
          g_cache.erase(g_cache.begin());
        }
        return;
      }
      if (b.ev) cudaEventDestroy(b.ev);
    }
  }
  cudaFreeAsync(p, s);
}

int trim_memory() {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (auto &b : g_cache) cache_release(b, nullptr);
    g_cache.clear();
  }
  RBF_CUDA_TRY(cudaDeviceSynchronize());
  int dev = 0;
  cudaMemPool_t pool;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  RBF_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  RBF_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
  return RBF_OK;
}

int ensure_dyn_smem(const void *fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> high;
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t &h = high[{dev, fn}];
  if (bytes > h) {
    RBF_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    h = bytes;
  }
  return RBF_OK;
}

int gather_positions(rbf_ctx *c, const double *xy, cudaStream_t s);  // cells.cu

static int plan_strips(const long long *counts, long long ncy, int P, long long min_rows,
                       long long *b) {
  long long N = 0;
  for (long long r = 0; r < ncy; ++r) N += counts[r];
  if (P < 1 || (long long)P * min_rows > ncy) {
    set_error("cannot cut %lld cell rows into %d strips of >= %lld rows", ncy, P, min_rows);
    return RBF_EINVAL;
  }
  b[0] = 0;
  b[P] = ncy;
  long long cum = 0, r = 0;
  for (int g = 1; g < P; ++g) {
    const long long target = (N * g + P / 2) / P;
    while (r < ncy && cum + counts[r] <= target) cum += counts[r++];
    // choose the closer of r and r+1
    if (r < ncy && (target - cum) > (cum + counts[r] - target)) cum += counts[r++];
    b[g] = r;
  }
  for (int g = 1; g < P; ++g)
    if (b[g] < b[g - 1] + min_rows) b[g] = b[g - 1] + min_rows;
  for (int g = P - 1; g >= 1; --g)
    if (b[g] > b[g + 1] - min_rows) b[g] = b[g + 1] - min_rows;
  for (int g = 0; g < P; ++g)
    if (b[g + 1] - b[g] < min_rows) {
      set_error("strip %d has fewer than %lld cell rows", g, min_rows);
      return RBF_EINVAL;
    }
  return RBF_OK;
}

// Strip `rank` of the cell-row partition `bounds` and its halos.  row_start[r] is
// the global sorted position of the first point of cell row r (ncy+1 entries).
// depth = rows of the extended range; kh / rings = matvec / RASM halo rows.
// Halo [0] is exchanged with rank-1 (below), [1] with rank+1 (above); send offsets
// are relative to the owned vector, receive offsets to the extended vector.
static void plan_strip(const long long *row_start, int ncy, const long long *bounds, int nranks,
                       int rank, int depth, int kh, int rings, Strip &S, Halo *hmv, Halo *hpc) {
  S.row_lo = (int)bounds[rank];
  S.row_hi = (int)bounds[rank + 1];
  S.ext_row_lo = S.row_lo - depth < 0 ? 0 : S.row_lo - depth;
  S.ext_row_hi = S.row_hi + depth > ncy ? ncy : S.row_hi + depth;
  S.own_lo = row_start[S.row_lo];
  S.own_hi = row_start[S.row_hi];
  S.ext_lo = row_start[S.ext_row_lo];
  S.ext_hi = row_start[S.ext_row_hi];
  auto halo = [&](int dd, Halo *h) {
    const bool below = rank > 0, above = rank < nranks - 1;
    const int lo = S.row_lo - dd < 0 ? 0 : S.row_lo - dd;
    const int hi = S.row_lo + dd > S.row_hi ? S.row_hi : S.row_lo + dd;
    h[0].recv_off = row_start[lo] - S.ext_lo;
    h[0].recv_cnt = below ? row_start[S.row_lo] - row_start[lo] : 0;
    h[0].send_off = 0;
    h[0].send_cnt = below ? row_start[hi] - row_start[S.row_lo] : 0;
    const int hi2 = S.row_hi + dd > ncy ? ncy : S.row_hi + dd;
    const int lo2 = S.row_hi - dd < S.row_lo ? S.row_lo : S.row_hi - dd;
    h[1].recv_off = row_start[S.row_hi] - S.ext_lo;
    h[1].recv_cnt = above ? row_start[hi2] - row_start[S.row_hi] : 0;
    h[1].send_off = row_start[lo2] - S.own_lo;
    h[1].send_cnt = above ? row_start[S.row_hi] - row_start[lo2] : 0;
  };
  halo(kh, hmv);
  halo(rings, hpc);
}

static int validate(const rbf_params *p, long long n) {
  if (!p) { set_error("params is NULL"); return RBF_EINVAL; }
  if (n < 1 || n > 0x7fffffffLL) { set_error("n = %lld outside [1, 2^31)", n); return RBF_EINVAL; }
  if (!(p->sigma > 0.0) || !std::isfinite(p->sigma)) { set_error("sigma must be > 0"); return RBF_EINVAL; }
  if (!(p->cell > 0.0) || !std::isfinite(p->cell)) { set_error("cell must be > 0"); return RBF_EINVAL; }
  if (!(p->rc > 0.0) || !std::isfinite(p->rc)) { set_error("rc must be > 0"); return RBF_EINVAL; }
  if (p->rc > 37.0 * p->sigma) {  // exp(-rc^2/2sigma^2) < 1e-297: the kernels assume this
    set_error("rc must be <= 37 sigma (entries beyond are below fp64 range)");
    return RBF_EINVAL;
  }
  if (p->overlap_rings < 0 || p->overlap_rings > 7) {
    set_error("overlap_rings must be in [0, 7]");
    return RBF_EINVAL;
  }
  if (!(p->overlap_width >= 0.0) || !std::isfinite(p->overlap_width)) {
    set_error("overlap_width must be >= 0 (finite)");
    return RBF_EINVAL;
  }
  if (p->schwarz != RBF_SCHWARZ_RASM && p->schwarz != RBF_SCHWARZ_ASM) {
    set_error("schwarz must be RBF_SCHWARZ_RASM (0) or RBF_SCHWARZ_ASM (1)");
    return RBF_EINVAL;
  }
  if (!(p->trunc_width >= 0.0) || !(p->trunc_width <= 8.0 * p->cell)) {
    set_error("trunc_width must be in [0, 8 cell] (finite)");
    return RBF_EINVAL;
  }
  if (!(p->x1 > p->x0) || !(p->y1 > p->y0) || !std::isfinite(p->x0) || !std::isfinite(p->x1) ||
      !std::isfinite(p->y0) || !std::isfinite(p->y1)) {
    set_error("box must satisfy x0 < x1, y0 < y1 (finite)");
    return RBF_EINVAL;
  }
  double ncx = std::ceil((p->x1 - p->x0) / p->cell), ncy = std::ceil((p->y1 - p->y0) / p->cell);
  if (ncx * ncy > 1.5e9) { set_error("too many cells (%g x %g)", ncx, ncy); return RBF_EINVAL; }
  return RBF_OK;
}

}  // namespace rbf

using namespace rbf;

extern "C" {

const char *rbf_last_error(void) { return g_err.c_str(); }

int64_t rbf_launch_count(void) { return g_launches.load(); }

/* debug: per-CTA clock64 phase stamps of the RASM setup kernel (RBF_PROBE builds) */
int rbf_debug_probe(int64_t *out) { return rbf::probe_read((long long *)out); }

namespace {
__global__ void k_poison_shared(int words) {
  extern __shared__ unsigned int sm_words[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm_words[i] = 0xFFFFFFFFu;
  __syncthreads();
  if (threadIdx.x == 0 && sm_words[words - 1] != 0xFFFFFFFFu) __trap();  // keep the stores
}
}  // namespace

int rbf_debug_poison_shared(void) {
  int dev = 0, sms = 0, optin = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  RBF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RBF_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  RBF_CUDA_TRY(cudaFuncSetAttribute(k_poison_shared, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  // one CTA with all the shared memory a block can hold per SM, several waves
  k_poison_shared<<<4 * sms, 1024, optin>>>(optin / 4);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  RBF_CUDA_TRY(cudaDeviceSynchronize());
  return RBF_OK;
}

int rbf_setup_times(const rbf_ctx *c, double out[4]) {
  if (!c || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  for (int i = 0; i < 4; ++i) out[i] = c->setup_ms[i];
  return RBF_OK;
}

int rbf_info(const rbf_ctx *c, int64_t out[8]) {
  if (!c || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  out[0] = c->x_count;
  out[1] = c->nsub;
  out[2] = c->max_ov;
  out[3] = c->max_own;
  out[4] = c->n_lu;
  out[5] = c->g.ncx;
  out[6] = c->g.ncy;
  out[7] = c->bytes;
  return RBF_OK;
}

int rbf_set_option(const char *name, int64_t value) {
  opt_init();
  if (!name) { set_error("rbf_set_option: NULL name"); return RBF_EINVAL; }
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!strcmp(name, kOptDefs[i].name)) {
      if (value < kOptDefs[i].lo || value > kOptDefs[i].hi) {
        set_error("rbf_set_option: %s must be in [%lld, %lld]", name, kOptDefs[i].lo, kOptDefs[i].hi);
        return RBF_EINVAL;
      }
      g_opt[i].store(value);
      return RBF_OK;
    }
  set_error("rbf_set_option: unknown option '%s'", name);
  return RBF_EINVAL;
}

int rbf_get_option(const char *name, int64_t *value) {
  opt_init();
  if (!name || !value) { set_error("rbf_get_option: NULL argument"); return RBF_EINVAL; }
  for (int i = 0; i < OPT_COUNT; ++i)
    if (!strcmp(name, kOptDefs[i].name)) {
      *value = g_opt[i].load();
      return RBF_OK;
    }
  set_error("rbf_get_option: unknown option '%s'", name);
  return RBF_EINVAL;
}

int rbf_trim_memory(void) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    set_error("rbf_trim_memory: no CUDA device (this library has no CPU fallback)");
    return RBF_ECUDA;
  }
  return trim_memory();
}

int rbf_lu_stats(const rbf_ctx *c, int64_t out[2]) {
  if (!c || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  out[0] = c->n_lu;
  out[1] = c->n_lu_pivot;
  return RBF_OK;
}

int rbf_debug_krylov_basis(const rbf_ctx *c, double *V_dev, int32_t nvec, void *stream) {
  if (!c || !V_dev) { set_error("NULL argument"); return RBF_EINVAL; }
  if (!c->V || nvec < 1 || nvec > c->V_m + 1) {
    set_error("rbf_debug_krylov_basis: %d vectors requested, %d held (solve first)", nvec,
              c->V ? c->V_m + 1 : 0);
    return RBF_EINVAL;
  }
  const size_t bytes = sizeof(double) * (size_t)nvec * (size_t)n_loc(c);
  RBF_CUDA_TRY(cudaMemcpyAsync(V_dev, c->V, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  RBF_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return RBF_OK;
}

int rbf_matvec_stats(const rbf_ctx *c, int64_t out[4]) {
  if (!c || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  out[0] = c->mv_lanes;
  out[1] = c->nchunks;
  out[2] = c->nlist_entries;
  out[3] = c->nlist_union;
  return RBF_OK;
}

int rbf_get_nccl_id(unsigned char out[128]) {
  if (!out) { set_error("out is NULL"); return RBF_EINVAL; }
  ncclUniqueId id;
  RBF_NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, id.internal, 128);
  return RBF_OK;
}

int rbf_plan_strips(const int64_t *row_counts, int64_t ncy, int32_t nranks, int64_t min_rows,
                    int64_t *row_bounds) {
  if (!row_counts || !row_bounds || ncy < 1) { set_error("bad arguments"); return RBF_EINVAL; }
  return plan_strips((const long long *)row_counts, ncy, nranks, min_rows, (long long *)row_bounds);
}

int rbf_plan_halo(const int64_t *row_start, int64_t ncy, const int64_t *row_bounds, int32_t nranks,
                  int32_t rank, int32_t kh, int32_t rings, int64_t out[12]) {
  if (!row_start || !row_bounds || !out || ncy < 1 || nranks < 1 || rank < 0 || rank >= nranks ||
      kh < 0 || rings < 0) {
    set_error("rbf_plan_halo: bad arguments");
    return RBF_EINVAL;
  }
  Strip S;
  Halo hmv[2], hpc[2];
  const int depth = kh > rings ? kh : rings;
  plan_strip((const long long *)row_start, (int)ncy, (const long long *)row_bounds, nranks, rank,
             depth, kh, rings, S, hmv, hpc);
  const long long v[12] = {S.ext_lo, S.own_lo, S.own_hi, S.ext_hi,
                           hmv[0].send_off, hmv[0].send_cnt, hmv[0].recv_off, hmv[0].recv_cnt,
                           hmv[1].send_off, hmv[1].send_cnt, hmv[1].recv_off, hmv[1].recv_cnt};
  for (int i = 0; i < 12; ++i) out[i] = v[i];
  return RBF_OK;
}

void rbf_destroy(rbf_ctx *c) {
  if (!c) return;
  cudaStream_t s = c->last_stream;
  dfree(c->cell_start, s);
  dfree(c->perm, s);
  dfree(c->xy_ext, s);
  dfree(c->x_off, s);
  dfree(c->ov_idx, s);
  dfree(c->ov_off, s);
  dfree(c->ov_own, s);
  dfree(c->rec, s);
  dfree(c->lane_tgt, s);
  dfree(c->chunk_len, s);
  dfree(c->chunk_off, s);
  dfree(c->nlist, s);
  dfree(c->mv_win, s);
  dfree(c->X, s);
  dfree(c->asm_toff, s);
  dfree(c->asm_t, s);
  dfree(c->asm_map, s);
  dfree(c->asm_poff, s);
  dfree(c->w_ext, s);
  dfree(c->V, s);
  dfree(c->t1, s);
  dfree(c->t2, s);
  dfree(c->red_part, s);
  dfree(c->red_count, s);
  dfree(c->dscal, s);
  dfree(c->ar_part, s);
  dfree(c->ar_bar, s);
  dfree(c->cg_blk, s);
  dfree(c->dc_blk, s);
  dfree(c->cg_count, s);
  if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
  if (c->g_graph) cudaGraphDestroy(c->g_graph);
  dfree(c->g_state, s);
  dfree(c->g_hist, s);
  dfree(c->g_f, s);
  dfree(c->g_x, s);
  if (c->hpin) cudaFreeHost(c->hpin);
  comm_destroy(c);
  delete c;
}

int rbf_setup(rbf_ctx **out, const double *xy, int64_t n, const rbf_params *p, const rbf_dist *d,
              void *stream) {
  if (!out || !xy) { set_error("rbf_setup: NULL argument"); return RBF_EINVAL; }
  *out = nullptr;
  RBF_TRY(validate(p, n));
  int ndev = 0;
  (void)cudaGetLastError();  // clear a stale non-sticky error from earlier calls
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    set_error("rbf_setup: no CUDA device (this library has no CPU fallback)");
    return RBF_ECUDA;
  }
  cudaStream_t s = (cudaStream_t)stream;
  rbf_ctx *c = new rbf_ctx();
  c->last_stream = s;
  c->p = *p;
  c->n = n;
  if (d) {
    if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks ||
        (d->comm != RBF_COMM_NONE && d->comm != RBF_COMM_NCCL && d->comm != RBF_COMM_THREADS)) {
      set_error("rbf_setup: bad rbf_dist (rank %d of %d, comm %d)", d->rank, d->nranks, d->comm);
      delete c;
      return RBF_EINVAL;
    }
    c->rank = d->rank;
    c->nranks = d->nranks;
    c->comm_mode = d->comm;
    c->overlap = !(d->flags & RBF_DIST_NO_OVERLAP) && d->comm != RBF_COMM_NONE;
  }
  Geom &g = c->g;
  g.x0 = p->x0; g.y0 = p->y0; g.x1 = p->x1; g.y1 = p->y1;
  g.cell = p->cell;
  g.rc2 = p->rc * p->rc;
  g.neg_inv_2s2 = -1.0 / (2.0 * p->sigma * p->sigma);
  g.esc = -1.0 / (2.0 * M_LN2 * p->sigma * p->sigma);
  g.esc64 = 64.0 * g.esc;
  g.norm = 1.0 / (2.0 * M_PI * p->sigma * p->sigma);
  g.ncx = (int)std::ceil((p->x1 - p->x0) / p->cell);
  g.ncy = (int)std::ceil((p->y1 - p->y0) / p->cell);
  if (g.ncx < 1) g.ncx = 1;
  if (g.ncy < 1) g.ncy = 1;
  g.kh = (int)std::ceil(p->rc / p->cell * (1.0 + 1e-12));
  g.tw = p->trunc_width;
  g.asm_full = p->schwarz == RBF_SCHWARZ_ASM;
  if (g.asm_full && c->nranks > 1 && p->overlap_width > 0.0) {
    set_error("rbf_setup: RBF_SCHWARZ_ASM across strips needs whole-ring overlap (overlap_width 0)");
    rbf_destroy(c);
    return RBF_EUNSUPPORTED;
  }
  // T-box (reading Q25): the box reaches floor(tw/c) + 1 cells beyond the target's cell
  if (g.tw > 0.0) g.kh = (int)std::floor(g.tw / p->cell * (1.0 + 1e-12)) + 1;
  g.rings = p->overlap_rings;
  g.ovw = p->overlap_width;
  cudaEvent_t ev[4];
  for (auto &e : ev) cudaEventCreate(&e);
  cudaEventRecord(ev[0], s);
  int st = build_cell_list(c, xy, s);
  cudaEventRecord(ev[1], s);
  if (st != RBF_OK) { rbf_destroy(c); return st; }
  // strips of cell rows balanced by a work model (matvec pairs + RASM apply entries per
  // row; on uniform data the same as balancing points); each strip >= halo
  // depth rows
  const int depth = g.kh > g.rings ? g.kh : g.rings;
  std::vector<long long> counts(g.ncy), bounds(c->nranks + 1);
  if (c->nranks > 1) {
    st = row_costs(c, s, counts);
    if (st != RBF_OK) { rbf_destroy(c); return st; }
  } else {
    for (int r = 0; r < g.ncy; ++r) counts[r] = c->row_start[r + 1] - c->row_start[r];
  }
  st = plan_strips(counts.data(), g.ncy, c->nranks, c->nranks > 1 ? depth : 1, bounds.data());
  if (st != RBF_OK) { rbf_destroy(c); return st; }
  plan_strip(c->row_start.data(), g.ncy, bounds.data(), c->nranks, c->rank, depth, g.kh, g.rings,
             c->s, c->halo_mv, c->halo_pc);
  st = gather_positions(c, xy, s);
  if (st == RBF_OK) st = build_nlist(c, s);
  cudaEventRecord(ev[2], s);
  if (st == RBF_OK && c->nranks > 1)
    st = dalloc(c, (void **)&c->w_ext, sizeof(double) * (size_t)(n_ext(c) > 0 ? n_ext(c) : 1), s);
  if (st == RBF_OK) st = comm_init(c, d);
  if (st == RBF_OK) st = rasm_setup(c, s);
  cudaEventRecord(ev[3], s);
  if (st == RBF_OK && cudaEventSynchronize(ev[3]) == cudaSuccess) {
    float a = 0, b = 0, d = 0, t = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&d, ev[2], ev[3]);
    cudaEventElapsedTime(&t, ev[0], ev[3]);
    c->setup_ms[0] = a;
    c->setup_ms[1] = b;
    c->setup_ms[2] = d;
    c->setup_ms[3] = t;
  }
  for (auto &e : ev) cudaEventDestroy(e);
  if (st != RBF_OK) { rbf_destroy(c); return st; }
  *out = c;
  return RBF_OK;
}

int64_t rbf_local_count(const rbf_ctx *c) { return c ? n_loc(c) : -1; }
int64_t rbf_ext_count(const rbf_ctx *c) { return c ? n_ext(c) : -1; }

int rbf_ranges(const rbf_ctx *c, int64_t o[4]) {
  if (!c || !o) { set_error("NULL argument"); return RBF_EINVAL; }
  o[0] = c->s.ext_lo; o[1] = c->s.own_lo; o[2] = c->s.own_hi; o[3] = c->s.ext_hi;
  return RBF_OK;
}

int rbf_local_index(const rbf_ctx *c, int64_t *idx, void *stream) {
  if (!c || !idx) { set_error("NULL argument"); return RBF_EINVAL; }
  return launch_local_index(c, idx, (cudaStream_t)stream);
}

__global__ void k_i32_to_i64(const int *a, long long n, int64_t *b) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < n) b[t] = a[t];
}

int rbf_cell_list(const rbf_ctx *c, int64_t *perm, int64_t *cs, int64_t dims[2], void *stream) {
  if (!c) { set_error("NULL ctx"); return RBF_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  long long nc = (long long)c->g.ncx * c->g.ncy + 1;
  if (perm) k_i32_to_i64<<<(int)((c->n + 255) / 256), 256, 0, s>>>(c->perm, c->n, perm); count_launch(1);
  if (cs) k_i32_to_i64<<<(int)((nc + 255) / 256), 256, 0, s>>>(c->cell_start, nc, cs); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  if (dims) { dims[0] = c->g.ncx; dims[1] = c->g.ncy; }
  return RBF_OK;
}

int rbf_to_local(const rbf_ctx *c, const double *vc, double *vl, void *stream) {
  if (!c || !vc || !vl) { set_error("NULL argument"); return RBF_EINVAL; }
  return launch_to_local(c, vc, vl, (cudaStream_t)stream);
}

int rbf_from_local(const rbf_ctx *c, const double *vl, double *vc, void *stream) {
  if (!c || !vc || !vl) { set_error("NULL argument"); return RBF_EINVAL; }
  return launch_from_local(c, vl, vc, (cudaStream_t)stream);
}

int rbf_matvec(rbf_ctx *c, const double *w, double *y, void *stream) {
  if (!c || !w || !y) { set_error("NULL argument"); return RBF_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (c->nranks > 1) return dist_matvec(c, w, y, s);
  return launch_matvec(c, w, y, s);
}

int rbf_rasm_apply(rbf_ctx *c, const double *r, double *z, void *stream) {
  if (!c || !r || !z) { set_error("NULL argument"); return RBF_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  if (c->nranks > 1) return dist_rasm_apply(c, r, z, s);
  return launch_rasm_apply(c, r, z, s);
}

int rbf_matvec_ext(rbf_ctx *c, const double *w_ext, double *y, void *stream) {
  if (!c || !w_ext || !y) { set_error("NULL argument"); return RBF_EINVAL; }
  return launch_matvec(c, w_ext, y, (cudaStream_t)stream);
}

int rbf_rasm_apply_ext(rbf_ctx *c, const double *r_ext, double *z, void *stream) {
  if (!c || !r_ext || !z) { set_error("NULL argument"); return RBF_EINVAL; }
  if (c->g.asm_full && c->nranks > 1) {  // the Eq.(8) sums need the neighbours' t (rbf_rasm_apply)
    set_error("rbf_rasm_apply_ext: RBF_SCHWARZ_ASM across strips needs rbf_rasm_apply (t exchange)");
    return RBF_EUNSUPPORTED;
  }
  return launch_rasm_apply(c, r_ext, z, (cudaStream_t)stream);
}

int rbf_solve(rbf_ctx *c, const double *f, const rbf_gmres_params *g, double *lam, rbf_report *rep,
              void *stream) {
  if (!c || !f || !g || !lam) { set_error("rbf_solve: NULL argument"); return RBF_EINVAL; }
  if (g->restart < 1 || g->max_iters < 1 || !(g->rtol >= 0.0) || !(g->atol >= 0.0)) {
    set_error("rbf_solve: restart >= 1, max_iters >= 1, rtol >= 0, atol >= 0 required");
    return RBF_EINVAL;
  }
  if (g->orth != RBF_ORTH_MGS && g->orth != RBF_ORTH_CGS2 && g->orth != RBF_ORTH_DCGS2) {
    set_error("rbf_solve: orth must be RBF_ORTH_MGS, RBF_ORTH_CGS2 or RBF_ORTH_DCGS2 (got %d)", g->orth);
    return RBF_EINVAL;
  }
  if (g->orth != RBF_ORTH_MGS && g->restart > RBF_CGS2_MAX_RESTART) {
    set_error("rbf_solve: CGS2/DCGS2 support restart <= %d (got %d)", RBF_CGS2_MAX_RESTART, g->restart);
    return RBF_EINVAL;
  }
  if (c->nranks > 1 && c->comm_mode == RBF_COMM_NONE) {
    set_error("rbf_solve: virtual strip contexts cannot solve (no communicator)");
    return RBF_EUNSUPPORTED;
  }
  c->last_stream = (cudaStream_t)stream;
  int st = solve_gmres(c, f, g, lam, rep, (cudaStream_t)stream);
  if (rep) {
    rep->n_cells = c->nsub;
    rep->bytes_device = c->bytes;
  }
  return st;
}

int rbf_evaluate(rbf_ctx *c, const double *q, int64_t m, const double *lam, double *s, void *stream) {
  if (!c || (m > 0 && (!q || !lam || !s))) { set_error("rbf_evaluate: NULL argument"); return RBF_EINVAL; }
  if (m < 0) { set_error("rbf_evaluate: m < 0"); return RBF_EINVAL; }
  return evaluate(c, q, m, lam, s, (cudaStream_t)stream);
}

int rbf_evaluate_count_pairs(rbf_ctx *c, const double *q, int64_t m, int64_t *n_pairs, void *stream) {
  if (!c || (!q && m > 0) || !n_pairs) { set_error("rbf_evaluate_count_pairs: NULL argument"); return RBF_EINVAL; }
  unsigned long long n = 0;
  RBF_TRY(evaluate(c, q, m, nullptr, nullptr, (cudaStream_t)stream, &n));
  *n_pairs = (int64_t)n;
  return RBF_OK;
}

int rbf_count_pairs(rbf_ctx *c, int64_t *np, void *stream) {
  if (!c || !np) { set_error("NULL argument"); return RBF_EINVAL; }
  long long v = 0;
  RBF_TRY(count_pairs(c, &v, (cudaStream_t)stream));
  *np = v;
  return RBF_OK;
}

int rbf_dot(rbf_ctx *c, const double *a, const double *b, double *out, void *stream) {
  if (!c || !a || !b || !out) { set_error("NULL argument"); return RBF_EINVAL; }
  return dot_host(c, a, b, out, (cudaStream_t)stream);
}

int rbf_interpolate_host(const double *xy_h, const double *f_h, int64_t n, const rbf_params *p,
                         const rbf_gmres_params *g, double *lam_h, rbf_report *rep, void *stream) {
  if (!xy_h || !f_h || !lam_h || !g) { set_error("rbf_interpolate_host: NULL argument"); return RBF_EINVAL; }
  RBF_TRY(validate(p, n));
  cudaStream_t s = (cudaStream_t)stream;
  double *xy = nullptr, *fc = nullptr, *fl = nullptr, *ll = nullptr;
  ScratchGuard sg(s);
  RBF_TRY(sg.alloc(nullptr, &xy, sizeof(double) * 2 * (size_t)n));
  RBF_TRY(sg.alloc(nullptr, &fc, sizeof(double) * (size_t)n));
  RBF_TRY(sg.alloc(nullptr, &fl, sizeof(double) * (size_t)n));
  RBF_TRY(sg.alloc(nullptr, &ll, sizeof(double) * (size_t)n));
  int st = RBF_OK;
  rbf_ctx *c = nullptr;
  do {
    if (cudaMemcpyAsync(xy, xy_h, sizeof(double) * 2 * (size_t)n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(fc, f_h, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      set_error("rbf_interpolate_host: host-to-device copy failed");
      st = RBF_ECUDA;
      break;
    }
    st = rbf_setup(&c, xy, n, p, nullptr, stream);
    if (st != RBF_OK) break;
    st = launch_to_local(c, fc, fl, s);
    if (st != RBF_OK) break;
    st = rbf_solve(c, fl, g, ll, rep, stream);
    if (st < 0) break;
    int st2 = launch_from_local(c, ll, fc, s);
    if (st2 != RBF_OK) { st = st2; break; }
    if (cudaMemcpyAsync(lam_h, fc, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      set_error("rbf_interpolate_host: device-to-host copy failed");
      st = RBF_ECUDA;
      break;
    }
  } while (0);
  if (c) rbf_destroy(c);
  return st;
}

}  // extern "C"
