// krylov.cu -- restarted GMRES(m), left preconditioned with RASM, modified
// Gram-Schmidt, Givens rotations (
// SPEC S:264-284; reading Q12).
//
// Vector work is fused into streaming kernels: MGS step j of iteration k is ONE
// pass  w <- w - h_{j-1,k} v_{j-1};  partial <w, v_j>  (the coefficient is read
// from device memory, no host round trip), the last step also forms ||w||^2.
// Reductions use a fixed grid and a fixed-shape tree, so the sums are
// deterministic; across ranks the per-rank partials are all-gathered and summed in
// rank order (reading Q14).  The Hessenberg column, Givens rotations and the
// residual estimate live on the device; the host reads back one scalar per
// iteration to decide convergence.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace rbf {

// Device scalar area layout (doubles), for restart m and P ranks.
struct Scal {
  int m, P;
  __host__ __device__ long long hloc() const { return 0; }                  // [m+2]
  __host__ __device__ long long hall() const { return m + 2; }              // [(m+2) P]
  __host__ __device__ long long H() const { return hall() + (long long)(m + 2) * P; }  // [(m+1) m]
  __host__ __device__ long long cs() const { return H() + (long long)(m + 1) * m; }
  __host__ __device__ long long sn() const { return cs() + m; }
  __host__ __device__ long long g() const { return sn() + m; }              // [m+1]
  __host__ __device__ long long y() const { return g() + m + 1; }           // [m]
  __host__ __device__ long long out() const { return y() + m; }             // [4]: |g|, hn, beta
  // CGS2 (reading Q23): this rank's pass-1 / pass-2 coefficients [m+2] and their
  // all-gathers [P (m+2)], rank-major with stride = the step's count k+1
  __host__ __device__ long long c1loc() const { return out() + 4; }
  __host__ __device__ long long c1all() const { return c1loc() + m + 2; }
  __host__ __device__ long long c2loc() const { return c1all() + (long long)(m + 2) * P; }
  __host__ __device__ long long c2all() const { return c2loc() + m + 2; }
  // DCGS2 (reading Q27): this step's block dots [<x_r, u>, <x_r, w>] (r = 0..k: v_0..v_{k-1},
  // u_k) and their all-gather (rank-major, stride 2(k+1)); unrotated Hessenberg; pending
  // first-pass coefficients; sweep coefficients {a_0..a_m, d_0..d_m, rho, e}
  __host__ __device__ long long dloc() const { return c2all() + (long long)(m + 2) * P; }
  __host__ __device__ long long dall() const { return dloc() + 2 * (m + 2); }
  __host__ __device__ long long Hraw() const { return dall() + (long long)2 * (m + 2) * P; }
  __host__ __device__ long long sp() const { return Hraw() + (long long)(m + 1) * m; }
  __host__ __device__ long long cf() const { return sp() + m + 2; }
  __host__ __device__ long long total() const { return cf() + 2 * (m + 2) + 2; }
};

// sum over ranks of entry j of a rank-major all-gather with `cnt` entries per rank
__device__ __forceinline__ double sum_ranks_rm(const double *all, int j, int cnt, int P) {
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += all[(long long)r * cnt + j];
  return s;
}

__device__ __forceinline__ double sum_ranks(const double *hall, int slot, int P) {
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += hall[(long long)slot * P + r];
  return s;
}

// Fixed-shape block reduction (deterministic).
__device__ __forceinline__ double block_sum(double v, double *sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

// Grid-level finish: every block writes its partial; the last block to arrive sums
// the partials in block order and writes *out.
__device__ __forceinline__ void grid_finish(double partial, double *blk, unsigned *count,
                                            double *out) {
  __shared__ bool last;
  __shared__ double sh[32];
  if (threadIdx.x == 0) {
    blk[blockIdx.x] = partial;
    __threadfence();
    unsigned t = atomicAdd(count, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += ((volatile double *)blk)[b];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    *out = v;
    *count = 0u;
  }
}

// w <- w - (sum_r coef[r]) x  (if coef != null);  out = <w, v>   (v may alias w)
__global__ __launch_bounds__(kRedThreads) void k_axpy_dot(const double *__restrict__ coef, int P,
                                                          double *w, const double *__restrict__ x,
                                                          const double *v, long long n,
                                                          double *__restrict__ blk,
                                                          unsigned *__restrict__ count,
                                                          double *__restrict__ out) {
  __shared__ double sh[32];
  double a = 0.0;
  if (coef) {
    for (int r = 0; r < P; ++r) a += coef[r];
  }
  const long long stride = (long long)gridDim.x * blockDim.x;
  // 4 elements in flight per thread (strided, coalesced), 4 partial sums combined in
  // a fixed order: deterministic for a fixed grid
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const bool alias = v == w;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double wv[4], vv[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      wv[u] = i < n ? w[i] : 0.0;
      vv[u] = i < n ? v[i] : 0.0;
      xv[u] = (coef && i < n) ? x[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (coef) {
        wv[u] = fma(-a, xv[u], wv[u]);
        if (i < n) w[i] = wv[u];
      }
      acc[u] = fma(wv[u], alias ? wv[u] : vv[u], acc[u]);  // v may alias w (norm of the update)
    }
  }
  double bs = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), sh);
  grid_finish(bs, blk, count, out);
}

__global__ void k_scale_by_norm(double *__restrict__ w, long long n, const double *__restrict__ nrm2,
                                int P, double4 *__restrict__ rec) {
  double h = sqrt(sum_ranks(nrm2, 0, P));
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = (h == 0.0) ? w[i] : w[i] / h;
    w[i] = v;
    if (rec) reinterpret_cast<double *>(rec + i)[2] = v;  // single rank: pre-pack the matvec input
  }
}

__global__ void k_sub(const double *__restrict__ f, double *__restrict__ t, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    t[i] = f[i] - t[i];
}

// Start of a cycle: g = (beta, 0, ...), beta = sqrt(sum_r nrm2[r]).
__global__ void k_cycle_init(double *S, Scal L, const double *nrm2) {  // nrm2 = slot 0
  double beta = sqrt(sum_ranks(nrm2, 0, L.P));
  for (int i = 0; i <= L.m; ++i) S[L.g() + i] = 0.0;
  S[L.g()] = beta;
  S[L.out() + 2] = beta;
}

// Column k of H from the all-gathered MGS results, previous rotations, new rotation,
// g update (Saad's GMRES with Givens; oracle orc_gmres follows the same steps).
// CGS2 (c1 != null): H(j,k) = pass-1 + pass-2 coefficients (rank-major all-gathers
// with k+1 entries per rank); ||w||^2 still comes from hall slot k+1.
__device__ void givens_step(double *S, const Scal &L, const double *hall, int k,
                            const double *c1 = nullptr, const double *c2 = nullptr) {
  const int m = L.m;
  double *H = S + L.H();
  double *cs = S + L.cs(), *sn = S + L.sn(), *g = S + L.g();
  for (int j = 0; j <= k; ++j)
    H[(long long)j * m + k] = c1 ? sum_ranks_rm(c1, j, k + 1, L.P) + sum_ranks_rm(c2, j, k + 1, L.P)
                                 : sum_ranks(hall, j, L.P);
  const double hn = sqrt(sum_ranks(hall, k + 1, L.P));
  H[(long long)(k + 1) * m + k] = hn;
  for (int j = 0; j < k; ++j) {
    double a = H[(long long)j * m + k], c = H[(long long)(j + 1) * m + k];
    H[(long long)j * m + k] = cs[j] * a + sn[j] * c;
    H[(long long)(j + 1) * m + k] = -sn[j] * a + cs[j] * c;
  }
  double a = H[(long long)k * m + k], c = H[(long long)(k + 1) * m + k];
  double den = hypot(a, c);
  cs[k] = a / den;
  sn[k] = c / den;
  H[(long long)k * m + k] = den;
  H[(long long)(k + 1) * m + k] = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  S[L.out() + 0] = fabs(g[k + 1]);
  S[L.out() + 1] = hn;
}

// Host-mapped mailbox ring: each Arnoldi step posts its residual estimate and its
// sequence number to slot seq % kMbSlots; the host polls that slot without any CUDA
// call (no stream synchronisation per iteration).  A ring, not a single slot: with
// the one-step lookahead, step k+1 may post before the host has read step k.
struct Mailbox {
  double gabs, hn;
  long long seq;
};
constexpr int kMbSlots = 4;
constexpr int kHpinScal = 16;  // hpin[kHpinScal...] : scalar read-backs (after the ring)
static_assert(sizeof(Mailbox) * kMbSlots <= sizeof(double) * kHpinScal, "mailbox ring overlaps");
constexpr int kDcMaxOut = 2 * (RBF_CGS2_MAX_RESTART + 1);  // DCGS2 block-dot outputs per step

__device__ __forceinline__ void post_mailbox(Mailbox *ring, const double *S, const Scal &L, long long seq) {
  volatile Mailbox *v = ring + (seq % kMbSlots);
  v->gabs = S[L.out() + 0];
  v->hn = S[L.out() + 1];
  __threadfence_system();
  v->seq = seq;
}

__global__ void k_givens(double *S, Scal L, const double *hall, int k, Mailbox *mb, long long seq,
                         const double *c1, const double *c2) {
  givens_step(S, L, hall, k, c1, c2);
  post_mailbox(mb, S, L, seq);
}

// ---------------------------------------------------------------------------
// Single-rank Arnoldi step in ONE cooperative launch: w = V[k+1] stays in
// registers while all k+1 MGS projections, the norm, the scaling and the Givens
// update run, separated by a software grid barrier (all CTAs co-resident by the
// cooperative launch).  Each projection reads only v_j (8 B/element) instead of
// w, v_{j-1}, v_j and a write of w.  Per-CTA partial sums are combined by every
// CTA in CTA order: deterministic.
// ---------------------------------------------------------------------------
constexpr int kArThreads = 1024;
constexpr int kArE = 8;  // elements per thread held in registers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp 0 only: arrive at the grid barrier (count, generation) after this CTA's
// partial is globally visible, and wait for the last CTA.
__device__ __forceinline__ void grid_arrive_wait(unsigned *bar, unsigned nb, int lane) {
  if (lane == 0) {
    volatile unsigned *vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncwarp();
}

// Each step j: the dot <w, v_j> (or ||w||^2 for j = k+1) is reduced in a fixed
// order (lanes, warps, then the CTAs' partials in CTA order by warp 0 of every CTA),
// with two __syncthreads and one grid barrier per step; v_j stays in registers for
// the update and v_{j+1} is loaded before the barrier, so the HBM latency of the
// next projection overlaps the reduction.
// Device-side loop state of the graph-driven solve (single rank).
struct GState {
  int k, it, conv, nan, kend, restarts, max_iters, pad;
  double rtol, atol, tol_abs, beta0, beta_last;
  double fsq, rsq;  // ||f||^2 and ||f - A x||^2 of the final iterate (report)
};

// After Arnoldi step k (block 0, thread 0): Givens, history, loop control.
__device__ __forceinline__ void graph_step_end(double *S, const Scal &L, int k, GState *st,
                                               double *hist, cudaGraphConditionalHandle inner) {
  givens_step(S, L, S + L.hloc(), k);
  const double gabs = S[L.out() + 0], hn = S[L.out() + 1];
  const int it = st->it;
  hist[it] = gabs / st->beta0;
  st->it = it + 1;
  st->k = k + 1;
  st->kend = k + 1;
  const bool bad = !isfinite(gabs) || !isfinite(hn);
  const bool conv = !bad && (gabs <= st->tol_abs || hn == 0.0);
  st->conv = conv;
  st->nan |= bad;
  const bool stop = conv || bad || k + 1 >= L.m || it + 1 >= st->max_iters;
  cudaGraphSetConditional(inner, stop ? 0u : 1u);
}

__global__ __launch_bounds__(kArThreads, 1) void k_arnoldi_fused(double *V, long long ldv, long long n,
                                                              int k, double *S, Scal L,
                                                              double *part, unsigned *bar,
                                                              Mailbox *mb, long long seq,
                                                              double4 *rec, const double *w_in,
                                                              GState *st, double *hist,
                                                              cudaGraphConditionalHandle inner) {
  if (st) k = st->k;  // graph mode: the step index lives on the device
  __shared__ double sh_w[kArThreads / 32];
  __shared__ double sh_h;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  const long long chunk = (n + G - 1) / G;
  const long long base = (long long)blockIdx.x * chunk;
  const long long end = base + chunk < n ? base + chunk : n;
  double *wv = V + (long long)(k + 1) * ldv;
  const double *win = w_in ? w_in : wv;
  double w[kArE], vc[kArE], vn[kArE];
#pragma unroll
  for (int e = 0; e < kArE; ++e) {
    const long long i = base + threadIdx.x + (long long)e * kArThreads;
    w[e] = i < end ? win[i] : 0.0;
    vc[e] = i < end ? V[i] : 0.0;  // v_0
  }
  for (int j = 0; j <= k + 1; ++j) {
    double acc = 0.0;
    if (j <= k) {
#pragma unroll
      for (int e = 0; e < kArE; ++e) acc = fma(w[e], vc[e], acc);
      if (j + 1 <= k && threadIdx.x != 0) {  // prefetch v_{j+1} (not by thread 0: its fence
        const double *vj1 = V + (long long)(j + 1) * ldv;  // in the grid barrier would wait for them)
#pragma unroll
        for (int e = 0; e < kArE; ++e) {
          const long long i = base + threadIdx.x + (long long)e * kArThreads;
          vn[e] = i < end ? vj1[i] : 0.0;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < kArE; ++e) acc = fma(w[e], w[e], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) sh_w[warp] = acc;
    __syncthreads();
    if (warp == 0) {
      double t = (lane < kArThreads / 32) ? sh_w[lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) part[(long long)j * G + blockIdx.x] = t;
    }
    cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0 && j + 1 <= k) {
      const double *vj1 = V + (long long)(j + 1) * ldv;
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        const long long i = base + (long long)e * kArThreads;
        vn[e] = i < end ? vj1[i] : 0.0;
      }
    }
    if (warp == 0) {
      double hs = 0.0;
      for (unsigned b = lane; b < G; b += 32) hs += ((volatile double *)part)[(long long)j * G + b];
      hs = warp_sum(hs);
      if (lane == 0) {
        sh_h = hs;
        if (blockIdx.x == 0) S[L.hloc() + j] = hs;
      }
    }
    __syncthreads();
    const double h = sh_h;
    if (j <= k) {
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        w[e] = fma(-h, vc[e], w[e]);
        vc[e] = vn[e];
      }
    } else {
      const double hn = sqrt(h);
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        const long long i = base + threadIdx.x + (long long)e * kArThreads;
        if (i < end) {
          const double v = (hn != 0.0) ? w[e] / hn : w[e];
          wv[i] = v;
          reinterpret_cast<double *>(rec + i)[2] = v;  // the next matvec's input, pre-packed
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (st) {
      graph_step_end(S, L, k, st, hist, inner);
    } else {
      givens_step(S, L, S + L.hloc(), k);
      post_mailbox(mb, S, L, seq);
    }
  }
}

// ---------------------------------------------------------------------------
// The same MGS step with TWO projections per grid barrier (reading Q28): for the pair
// (v_j, v_{j+1}) one reduction gives D1 = <w, v_j>, D2 = <w, v_{j+1}>, D3 = <v_j, v_{j+1}>;
// then h_j = D1 and h_{j+1} = <w - h_j v_j, v_{j+1}> = D2 - h_j D3 (MGS's coefficient,
// the inner product of the updated vector, expanded), and w -= h_j v_j, then
// w -= h_{j+1} v_{j+1} in MGS's order.  ceil((k+1)/2) + 1 barriers instead of k + 2.
// The pair's vectors are loaded after the barrier (the next pair is prefetched into L2
// during it); part slots: D1, D2 at j, j+1 and D3 at (m + 2) + j.
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(kArThreads, 1) void k_arnoldi_mgs2(double *V, long long ldv, long long n,
                                                             int k, double *S, Scal L,
                                                             double *part, unsigned *bar,
                                                             Mailbox *mb, long long seq,
                                                             double4 *rec, const double *w_in,
                                                             GState *st, double *hist,
                                                             cudaGraphConditionalHandle inner) {
  if (st) k = st->k;
  __shared__ double sh_w[3][kArThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  const long long chunk = (n + G - 1) / G;
  const long long base = (long long)blockIdx.x * chunk;
  const long long end = base + chunk < n ? base + chunk : n;
  const long long d3 = (long long)(L.m + 2) * G;
  double *wv = V + (long long)(k + 1) * ldv;
  const double *win = w_in ? w_in : wv;
  double w[kArE], va[kArE], vb[kArE];
#pragma unroll
  for (int e = 0; e < kArE; ++e) {
    const long long i = base + threadIdx.x + (long long)e * kArThreads;
    w[e] = i < end ? win[i] : 0.0;
  }
  for (int j = 0; j <= k + 1; j += 2) {
    const bool norm = j == k + 1;           // the last step: ||w||^2 only
    const bool pair = !norm && j + 1 <= k;  // two projections in this step
    double a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (norm) {
#pragma unroll
      for (int e = 0; e < kArE; ++e) a1 = fma(w[e], w[e], a1);
    } else {
      const double *vj = V + (long long)j * ldv, *vj1 = V + (long long)(j + 1) * ldv;
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        const long long i = base + threadIdx.x + (long long)e * kArThreads;
        va[e] = i < end ? vj[i] : 0.0;
        vb[e] = (pair && i < end) ? vj1[i] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        a1 = fma(w[e], va[e], a1);
        a2 = fma(w[e], vb[e], a2);
        a3 = fma(va[e], vb[e], a3);
      }
    }
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    a3 = warp_sum(a3);
    if (lane == 0) {
      sh_w[0][warp] = a1;
      sh_w[1][warp] = a2;
      sh_w[2][warp] = a3;
    }
    __syncthreads();
    if (warp < 3) {
      double t = (lane < kArThreads / 32) ? sh_w[warp][lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) part[(warp == 2 ? d3 + (long long)j * G : (long long)(j + warp) * G) + blockIdx.x] = t;
    }
    if (!norm && j + 2 <= k) {  // the next pair into L2 while the barrier runs
      const long long i = base + threadIdx.x;
      if (i < end) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(V + (long long)(j + 2) * ldv + i));
        if (j + 3 <= k) asm volatile("prefetch.global.L2 [%0];" ::"l"(V + (long long)(j + 3) * ldv + i));
      }
    }
    cooperative_groups::this_grid().sync();
    if (warp < 3) {
      double hs = 0.0;
      const long long off = warp == 2 ? d3 + (long long)j * G : (long long)(j + warp) * G;
      if (warp == 0 || pair)
        for (unsigned b = lane; b < G; b += 32) hs += ((volatile double *)part)[off + b];
      hs = warp_sum(hs);
      if (lane == 0) sh_w[warp][0] = hs;  // sh_w is free again after the barrier
    }
    __syncthreads();
    if (norm) {
      const double hn = sqrt(sh_w[0][0]);
      if (blockIdx.x == 0 && threadIdx.x == 0) S[L.hloc() + j] = sh_w[0][0];
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        const long long i = base + threadIdx.x + (long long)e * kArThreads;
        if (i < end) {
          const double v = (hn != 0.0) ? w[e] / hn : w[e];
          wv[i] = v;
          reinterpret_cast<double *>(rec + i)[2] = v;  // the next matvec's input, pre-packed
        }
      }
    } else {
      const double h1 = sh_w[0][0];
      const double h2 = pair ? sh_w[1][0] - h1 * sh_w[2][0] : 0.0;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        S[L.hloc() + j] = h1;
        if (pair) S[L.hloc() + j + 1] = h2;
      }
#pragma unroll
      for (int e = 0; e < kArE; ++e) {
        w[e] = fma(-h1, va[e], w[e]);
        if (pair) w[e] = fma(-h2, vb[e], w[e]);
      }
      if (!pair) j -= 1;  // odd count: the norm step follows directly (j + 2 - 1 = k + 1)
    }
    __syncthreads();  // sh_w reused by the next step's partials
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (st) {
      graph_step_end(S, L, k, st, hist, inner);
    } else {
      givens_step(S, L, S + L.hloc(), k);
      post_mailbox(mb, S, L, seq);
    }
  }
}

// ---------------------------------------------------------------------------
// CGS2 Arnoldi step (reading Q23), single rank, ONE cooperative launch with three
// grid barriers instead of k+2: pass 1 h1 = V^T w; pass 2 w -= V h1, then
// h2 = V^T w; pass 3 w -= V h2 and ||w||^2.  Same layout as k_arnoldi_fused (w in
// registers, kArE elements per thread); every pass loops over the basis vectors
// with kArE independent loads per thread per vector, one warp reduction per vector
// into shared memory, and one CTA-level reduction + grid barrier per pass.
// Fixed-order reductions: deterministic.
// ---------------------------------------------------------------------------
constexpr int kCgMaxM = RBF_CGS2_MAX_RESTART;
constexpr int kArWarps = kArThreads / 32;
static_assert(kCgMaxM <= kArWarps, "one warp per coefficient in the CTA reductions");

// CTA partials sh_red[j][warp] (j < cnt) -> part[j*G + cta]; grid barrier; CTA-order
// sums of the partials -> sh_out[j].
__device__ __forceinline__ void cg_reduce(double (*sh_red)[kArWarps], int cnt, double *part,
                                          double *sh_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  __syncthreads();
  if (warp < cnt) {
    const double t = warp_sum(sh_red[warp][lane]);
    if (lane == 0) part[(long long)warp * G + blockIdx.x] = t;
  }
  cooperative_groups::this_grid().sync();
  if (warp < cnt) {
    double hs = 0.0;
    for (unsigned b = lane; b < G; b += 32) hs += ((volatile double *)part)[(long long)warp * G + b];
    hs = warp_sum(hs);
    if (lane == 0) sh_out[warp] = hs;
  }
  __syncthreads();
}

__global__ __launch_bounds__(kArThreads, 1) void k_arnoldi_cgs2(double *V, long long ldv, long long n,
                                                             int k, double *S, Scal L,
                                                             double *part, unsigned *bar,
                                                             Mailbox *mb, long long seq,
                                                             double4 *rec, const double *w_in,
                                                             GState *st, double *hist,
                                                             cudaGraphConditionalHandle inner) {
  (void)bar;
  if (st) k = st->k;
  __shared__ double sh_red[kCgMaxM][kArWarps];
  __shared__ double sh_h1[kCgMaxM + 1], sh_h2[kCgMaxM + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  const long long chunk = (n + G - 1) / G;
  const long long base = (long long)blockIdx.x * chunk;
  const long long end = base + chunk < n ? base + chunk : n;
  const int cnt = k + 1;
  double *wv = V + (long long)(k + 1) * ldv;
  const double *win = w_in ? w_in : wv;
  double *part1 = part, *part2 = part + (long long)(kCgMaxM + 1) * G,
         *part3 = part + 2LL * (kCgMaxM + 1) * G;
  long long idx[kArE];
  bool ok[kArE];
  double w[kArE];
#pragma unroll
  for (int e = 0; e < kArE; ++e) {
    idx[e] = base + threadIdx.x + (long long)e * kArThreads;
    ok[e] = idx[e] < end;
    w[e] = ok[e] ? win[idx[e]] : 0.0;
  }
  // <w, v_j> for all j < cnt -> sh_red[j][warp]
  auto dots = [&]() {
    for (int j = 0; j < cnt; ++j) {
      const double *vj = V + (long long)j * ldv;
      double vv[kArE];
#pragma unroll
      for (int e = 0; e < kArE; ++e) vv[e] = ok[e] ? __ldcg(vj + idx[e]) : 0.0;
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < kArE; ++e) acc = fma(w[e], vv[e], acc);
      acc = warp_sum(acc);
      if (lane == 0) sh_red[j][warp] = acc;
    }
  };
  // w -= sum_j h[j] v_j
  auto update = [&](const double *h) {
    for (int j = 0; j < cnt; ++j) {
      const double *vj = V + (long long)j * ldv;
      const double hj = h[j];
      double vv[kArE];
#pragma unroll
      for (int e = 0; e < kArE; ++e) vv[e] = ok[e] ? __ldcg(vj + idx[e]) : 0.0;
#pragma unroll
      for (int e = 0; e < kArE; ++e) w[e] = fma(-hj, vv[e], w[e]);
    }
  };
  dots();  // pass 1
  cg_reduce(sh_red, cnt, part1, sh_h1);
  update(sh_h1);  // pass 2
  dots();
  cg_reduce(sh_red, cnt, part2, sh_h2);
  if (blockIdx.x == 0 && threadIdx.x < cnt) S[L.hloc() + threadIdx.x] = sh_h1[threadIdx.x] + sh_h2[threadIdx.x];
  update(sh_h2);  // pass 3
  double nrm = 0.0;
#pragma unroll
  for (int e = 0; e < kArE; ++e) nrm = fma(w[e], w[e], nrm);
  nrm = warp_sum(nrm);
  if (lane == 0) sh_red[0][warp] = nrm;
  cg_reduce(sh_red, 1, part3, sh_h1);
  const double nsq = sh_h1[0];
  if (blockIdx.x == 0 && threadIdx.x == 0) S[L.hloc() + cnt] = nsq;
  // v_{k+1} = w / ||w||, also into the next matvec's records
  const double hn = sqrt(nsq);
#pragma unroll
  for (int e = 0; e < kArE; ++e) {
    if (ok[e]) {
      const double v = (hn != 0.0) ? w[e] / hn : w[e];
      wv[idx[e]] = v;
      reinterpret_cast<double *>(rec + idx[e])[2] = v;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (st) {
      graph_step_end(S, L, k, st, hist, inner);
    } else {
      givens_step(S, L, S + L.hloc(), k);
      post_mailbox(mb, S, L, seq);
    }
  }
}

// CGS2 pass for the multi-kernel path (several ranks, or n beyond the cooperative
// kernel's reach).  MODE 0: out[j] = <w, v_j>;  MODE 1: w -= V c, out[j] = <w, v_j>;
// MODE 2: w -= V c, out[0] = ||w||^2;  c_j = sum over ranks of the previous pass's
// all-gather (rank-major, cnt per rank).  Each thread holds kCpE elements of w in
// registers per chunk and loops over the basis vectors (kCpE independent loads per
// vector); per-warp partials accumulate in shared memory in chunk order, blocks'
// partials blk[j * gridDim + b] are summed in block order by the last block:
// deterministic for a fixed grid.
constexpr int kCpE = 4;
template <int MODE>
__global__ __launch_bounds__(kRedThreads) void k_cgs_pass(double *w, const double *__restrict__ V,
                                                          long long ldv, int cnt, long long n,
                                                          const double *__restrict__ call, int P,
                                                          double *__restrict__ blk,
                                                          unsigned *__restrict__ count,
                                                          double *__restrict__ out) {
  constexpr int W_ = kRedThreads / 32;
  __shared__ double sh_c[kCgMaxM];
  __shared__ double sh_acc[kCgMaxM][W_];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nout = MODE == 2 ? 1 : cnt;
  if (MODE > 0 && threadIdx.x < cnt) sh_c[threadIdx.x] = sum_ranks_rm(call, threadIdx.x, cnt, P);
  for (int t = threadIdx.x; t < kCgMaxM * W_; t += blockDim.x) (&sh_acc[0][0])[t] = 0.0;
  __syncthreads();
  const long long cstride = (long long)gridDim.x * blockDim.x * kCpE;
  for (long long c0 = (long long)blockIdx.x * blockDim.x * kCpE; c0 < n; c0 += cstride) {
    long long idx[kCpE];
    bool ok[kCpE];
    double wv[kCpE];
#pragma unroll
    for (int e = 0; e < kCpE; ++e) {
      idx[e] = c0 + threadIdx.x + (long long)e * blockDim.x;
      ok[e] = idx[e] < n;
      wv[e] = ok[e] ? w[idx[e]] : 0.0;
    }
    if (MODE > 0) {
      for (int j = 0; j < cnt; ++j) {
        const double *vj = V + (long long)j * ldv;
        const double cj = sh_c[j];
        double vv[kCpE];
#pragma unroll
        for (int e = 0; e < kCpE; ++e) vv[e] = ok[e] ? vj[idx[e]] : 0.0;
#pragma unroll
        for (int e = 0; e < kCpE; ++e) wv[e] = fma(-cj, vv[e], wv[e]);
      }
#pragma unroll
      for (int e = 0; e < kCpE; ++e)
        if (ok[e]) w[idx[e]] = wv[e];
    }
    if (MODE == 2) {
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < kCpE; ++e) acc = fma(wv[e], wv[e], acc);
      acc = warp_sum(acc);
      if (lane == 0) sh_acc[0][warp] += acc;
    } else {
      for (int j = 0; j < cnt; ++j) {
        const double *vj = V + (long long)j * ldv;
        double vv[kCpE];
#pragma unroll
        for (int e = 0; e < kCpE; ++e) vv[e] = ok[e] ? vj[idx[e]] : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < kCpE; ++e) acc = fma(wv[e], vv[e], acc);
        acc = warp_sum(acc);
        if (lane == 0) sh_acc[j][warp] += acc;
      }
    }
  }
  __syncthreads();
  for (int j = warp; j < nout; j += W_) {
    double t = lane < W_ ? sh_acc[j][lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) blk[(long long)j * gridDim.x + blockIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = warp; j < nout; j += W_) {
    double t = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) t += ((volatile double *)blk)[(long long)j * gridDim.x + b];
    t = warp_sum(t);
    if (lane == 0) out[j] = t;
  }
  if (threadIdx.x == 0) *count = 0u;
}

// ---------------------------------------------------------------------------
// DCGS2 (reading Q27; oracle gmres_dcgs2): per Arnoldi step k ONE block reduction,
//   k_dcgs_dots:   x_r = <v_r, u_k>, y_r = <v_r, w> for r < k, and <u_k, u_k>, <u_k, w>
//                  (w = B u_k; absent at the cycle's last step) -- one pass over
//                  V_0..V_{k-1}, u_k, w with fixed-order sums;
//   all-gather of the 2(k+1) partials (several ranks);
//   k_dcgs_scalar: rho = sqrt(alpha - |a|^2), column k-1 of H (= pending first pass + a,
//                  rho), its Givens rotation and residual estimate (mailbox), the next
//                  first-pass coefficients s = (c - H a) / rho and the sweep coefficients;
//   k_dcgs_update: v_k = (u_k - V a) / rho,  u_{k+1} = (w - V d - e u_k) / rho  (one pass).
// ---------------------------------------------------------------------------
__global__ __launch_bounds__(kRedThreads) void k_dcgs_dots(const double *__restrict__ V, long long ldv,
                                                           int k, long long n,
                                                           const double *__restrict__ w,
                                                           double *__restrict__ blk,
                                                           unsigned *__restrict__ count,
                                                           double *__restrict__ out) {
  constexpr int W_ = kRedThreads / 32;
  __shared__ double sh_acc[kDcMaxOut][W_];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = k + 1, nout = 2 * cnt;
  const double *u = V + (long long)k * ldv;
  for (int t = threadIdx.x; t < kDcMaxOut * W_; t += blockDim.x) (&sh_acc[0][0])[t] = 0.0;
  __syncthreads();
  const long long cstride = (long long)gridDim.x * blockDim.x * kCpE;
  for (long long c0 = (long long)blockIdx.x * blockDim.x * kCpE; c0 < n; c0 += cstride) {
    long long idx[kCpE];
    bool ok[kCpE];
    double uv[kCpE], wv[kCpE];
#pragma unroll
    for (int e = 0; e < kCpE; ++e) {
      idx[e] = c0 + threadIdx.x + (long long)e * blockDim.x;
      ok[e] = idx[e] < n;
      uv[e] = ok[e] ? u[idx[e]] : 0.0;
      wv[e] = (ok[e] && w) ? w[idx[e]] : 0.0;
    }
    for (int j = 0; j < cnt; ++j) {
      double vv[kCpE];
      if (j < k) {
        const double *vj = V + (long long)j * ldv;
#pragma unroll
        for (int e = 0; e < kCpE; ++e) vv[e] = ok[e] ? vj[idx[e]] : 0.0;
      } else {
#pragma unroll
        for (int e = 0; e < kCpE; ++e) vv[e] = uv[e];
      }
      double au = 0.0, aw = 0.0;
#pragma unroll
      for (int e = 0; e < kCpE; ++e) {
        au = fma(vv[e], uv[e], au);
        aw = fma(vv[e], wv[e], aw);
      }
      au = warp_sum(au);
      aw = warp_sum(aw);
      if (lane == 0) {
        sh_acc[j][warp] += au;
        sh_acc[cnt + j][warp] += aw;
      }
    }
  }
  __syncthreads();
  for (int j = warp; j < nout; j += W_) {
    double t = lane < W_ ? sh_acc[j][lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) blk[(long long)j * gridDim.x + blockIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = warp; j < nout; j += W_) {
    double t = 0.0;
    for (unsigned b = lane; b < gridDim.x; b += 32) t += ((volatile double *)blk)[(long long)j * gridDim.x + b];
    t = warp_sum(t);
    if (lane == 0) out[j] = t;
  }
  if (threadIdx.x == 0) *count = 0u;
}

// One thread.  all = rank-major all-gather of the step's 2(k+1) partials.
__global__ void k_dcgs_scalar(double *S, Scal L, const double *all, int k, Mailbox *mb, long long seq) {
  const int m = L.m, P = L.P, cnt = k + 1, stride = 2 * cnt;
  double *Hr = S + L.Hraw(), *H = S + L.H(), *sp = S + L.sp(), *cf = S + L.cf();
  double *cs = S + L.cs(), *sn = S + L.sn(), *g = S + L.g();
  double *a = cf, *d = cf + (m + 2);
  double asq = 0.0;
  for (int j = 0; j < k; ++j) {
    a[j] = sum_ranks_rm(all, j, stride, P);
    asq += a[j] * a[j];
  }
  const double alpha = sum_ranks_rm(all, k, stride, P);
  const double rho2 = alpha - asq;
  const double rho = rho2 > 0.0 ? sqrt(rho2) : (rho2 == rho2 ? 0.0 : rho2);  // NaN stays NaN
  if (k == 0) {  // cycle start: beta = ||u_0||, g = beta e_1
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = rho;
    S[L.out() + 2] = rho;
  } else {  // finish column k-1 of the Arnoldi relation, then Givens (as givens_step)
    const int kc = k - 1;
    for (int j = 0; j < k; ++j) Hr[(long long)j * m + kc] = sp[j] + a[j];
    Hr[(long long)k * m + kc] = rho;
    for (int j = 0; j <= k; ++j) H[(long long)j * m + kc] = Hr[(long long)j * m + kc];
    for (int j = 0; j < kc; ++j) {
      const double p = H[(long long)j * m + kc], q = H[(long long)(j + 1) * m + kc];
      H[(long long)j * m + kc] = cs[j] * p + sn[j] * q;
      H[(long long)(j + 1) * m + kc] = -sn[j] * p + cs[j] * q;
    }
    const double p = H[(long long)kc * m + kc], q = H[(long long)k * m + kc];
    const double den = hypot(p, q);
    cs[kc] = p / den;
    sn[kc] = q / den;
    H[(long long)kc * m + kc] = den;
    H[(long long)k * m + kc] = 0.0;
    g[k] = -sn[kc] * g[kc];
    g[kc] = cs[kc] * g[kc];
    S[L.out() + 0] = fabs(g[k]);
    S[L.out() + 1] = rho;
    post_mailbox(mb, S, L, seq);
  }
  if (k < m) {  // the next direction's first pass (w = B u_k present)
    double ab = 0.0;
    for (int j = 0; j < k; ++j) ab += a[j] * sum_ranks_rm(all, cnt + j, stride, P);
    const double gamma = sum_ranks_rm(all, cnt + k, stride, P);
    const double ck = (gamma - ab) / rho, e = ck / rho;
    for (int j = 0; j <= k; ++j) {
      const double cj = j < k ? sum_ranks_rm(all, cnt + j, stride, P) : ck;
      double ha = 0.0;
      for (int i = 0; i < k; ++i) ha += Hr[(long long)j * m + i] * a[i];
      sp[j] = (cj - ha) / rho;
      if (j < k) d[j] = cj - e * a[j];
    }
    cf[2 * (m + 2)] = rho;
    cf[2 * (m + 2) + 1] = e;
  }
}

// v_k = (u_k - sum_j a_j v_j) / rho  -> slot k;  u_{k+1} = (w - sum_j d_j v_j - e u_k) / rho
// -> slot k+1 (w is read from there); rec (single rank): u_{k+1} packed for the next matvec.
constexpr int kDuE = 4;
__global__ __launch_bounds__(kRedThreads) void k_dcgs_update(double *V, long long ldv, int k, long long n,
                                                             const double *__restrict__ S, Scal L,
                                                             double4 *__restrict__ rec) {
  __shared__ double sa[kCgMaxM + 2], sd[kCgMaxM + 2];
  const double *cf = S + L.cf();
  if (threadIdx.x < k) {
    sa[threadIdx.x] = cf[threadIdx.x];
    sd[threadIdx.x] = cf[(L.m + 2) + threadIdx.x];
  }
  __syncthreads();
  const double rho = cf[2 * (L.m + 2)], e = cf[2 * (L.m + 2) + 1];
  double *u = V + (long long)k * ldv, *w = V + (long long)(k + 1) * ldv;
  const long long cstride = (long long)gridDim.x * blockDim.x * kDuE;
  for (long long c0 = (long long)blockIdx.x * blockDim.x * kDuE; c0 < n; c0 += cstride) {
    long long idx[kDuE];
    bool ok[kDuE];
    double uv[kDuE], vk[kDuE], nx[kDuE];
#pragma unroll
    for (int q = 0; q < kDuE; ++q) {
      idx[q] = c0 + threadIdx.x + (long long)q * blockDim.x;
      ok[q] = idx[q] < n;
      uv[q] = ok[q] ? u[idx[q]] : 0.0;
      vk[q] = uv[q];
      nx[q] = ok[q] ? fma(-e, uv[q], w[idx[q]]) : 0.0;
    }
    for (int j = 0; j < k; ++j) {
      const double *vj = V + (long long)j * ldv;
      const double aj = sa[j], dj = sd[j];
#pragma unroll
      for (int q = 0; q < kDuE; ++q) {
        const double v = ok[q] ? vj[idx[q]] : 0.0;
        vk[q] = fma(-aj, v, vk[q]);
        nx[q] = fma(-dj, v, nx[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < kDuE; ++q)
      if (ok[q]) {
        u[idx[q]] = vk[q] / rho;
        const double un = nx[q] / rho;
        w[idx[q]] = un;
        if (rec) reinterpret_cast<double *>(rec + idx[q])[2] = un;
      }
  }
}

// ---- graph-mode control kernels (one thread)
__global__ void k_g_begin(const double *nrm2, GState *st, cudaGraphConditionalHandle outer) {
  const double beta0 = sqrt(*nrm2);
  st->beta0 = beta0;
  st->tol_abs = fmax(st->rtol * beta0, st->atol);
  st->it = 0;
  st->k = 0;
  st->kend = 0;
  st->restarts = 0;
  st->nan = !isfinite(beta0);
  st->conv = beta0 == 0.0;
  st->beta_last = beta0;
  cudaGraphSetConditional(outer, (!st->conv && !st->nan && st->max_iters > 0) ? 1u : 0u);
}

__global__ void k_g_cycle(double *S, Scal L, const double *nrm2, GState *st,
                          cudaGraphConditionalHandle inner) {
  const double beta = sqrt(*nrm2);
  for (int i = 0; i <= L.m; ++i) S[L.g() + i] = 0.0;
  S[L.g()] = beta;
  S[L.out() + 2] = beta;
  st->k = 0;
  st->kend = 0;
  cudaGraphSetConditional(inner, (!st->conv && !st->nan && st->it < st->max_iters) ? 1u : 0u);
}

// End of a cycle: explicit preconditioned residual norm^2 in nrm2 (reading Q12).
__global__ void k_g_end_cycle(const double *nrm2, GState *st, cudaGraphConditionalHandle outer) {
  const double beta = sqrt(*nrm2);
  st->beta_last = beta;
  bool more = !st->conv && !st->nan && st->it < st->max_iters;
  if (more) {
    st->restarts += 1;
    if (beta <= st->tol_abs) {
      st->conv = 1;
      more = false;
    }
  }
  cudaGraphSetConditional(outer, more ? 1u : 0u);
}

__global__ void k_backsolve_g(double *S, Scal L, const GState *st) {
  const int kend = st->kend, m = L.m;
  const double *H = S + L.H(), *g = S + L.g();
  double *y = S + L.y();
  for (int i = kend - 1; i >= 0; --i) {
    double sacc = g[i];
    for (int j = i + 1; j < kend; ++j) sacc -= H[(long long)i * m + j] * y[j];
    y[i] = sacc / H[(long long)i * m + i];
  }
}

__global__ void k_update_x_g(double *__restrict__ x, const double *__restrict__ V, long long ldv,
                             const double *__restrict__ S, Scal L, const GState *st, long long n) {
  const int kend = st->kend;
  const double *y = S + L.y();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double xi = x[i];
    for (int j = 0; j < kend; ++j) xi += y[j] * V[j * ldv + i];
    x[i] = xi;
  }
}

// y = H(0:kend, 0:kend)^-1 g(0:kend)
__global__ void k_backsolve(double *S, Scal L, int kend) {
  const int m = L.m;
  const double *H = S + L.H(), *g = S + L.g();
  double *y = S + L.y();
  for (int i = kend - 1; i >= 0; --i) {
    double s = g[i];
    for (int j = i + 1; j < kend; ++j) s -= H[(long long)i * m + j] * y[j];
    y[i] = s / H[(long long)i * m + i];
  }
}

// x += sum_{j < kend} y_j V_j   (one streaming pass)
__global__ void k_update_x(double *__restrict__ x, const double *__restrict__ V, long long ldv,
                           const double *__restrict__ S, Scal L, int kend, long long n) {
  const double *y = S + L.y();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double xi = x[i];
    for (int j = 0; j < kend; ++j) xi += y[j] * V[j * ldv + i];
    x[i] = xi;
  }
}

// ---------------------------------------------------------------------------

struct Op {
  rbf_ctx *c;
  cudaStream_t s;
  // y = A w (halo of w first)
  int matvec(const double *w, double *y, bool prepacked = false) {
    if (c->nranks > 1) return dist_matvec(c, w, y, s);
    return launch_matvec(c, w, y, s, prepacked);
  }
  int pc(const double *r, double *z) {
    if (c->nranks > 1) return dist_rasm_apply(c, r, z, s);
    return launch_rasm_apply(c, r, z, s);
  }
};

// per-CTA partial sums of the fused Arnoldi kernels: MGS (m+2) slots, CGS2 3 passes
static size_t part_doubles(const rbf_ctx *c, int m) {
  const size_t a = (size_t)2 * (m + 2) * (size_t)c->ar_grid;  // MGS pairs: D3 after the m+2 slots
  const size_t b = (size_t)3 * (kCgMaxM + 1) * (size_t)c->cg_grid;
  return (a > b ? a : b) + 1;
}

static int ensure_workspace(rbf_ctx *c, int m, cudaStream_t s) {
  const long long n = n_loc(c);
  if (c->V && c->V_m >= m) return RBF_OK;
  if (c->V) dfree(c->V, s);
  if (c->dscal) dfree(c->dscal, s);
  c->V = nullptr;
  c->dscal = nullptr;
  RBF_TRY(dalloc(c, (void **)&c->V, sizeof(double) * (size_t)(m + 1) * (size_t)(n > 0 ? n : 1), s));
  Scal L{m, c->nranks};
  RBF_TRY(dalloc(c, (void **)&c->dscal, sizeof(double) * (size_t)L.total(), s));
  RBF_CUDA_TRY(cudaMemsetAsync(c->dscal, 0, sizeof(double) * (size_t)L.total(), s));
  c->V_m = m;
  if (!c->t1) RBF_TRY(dalloc(c, (void **)&c->t1, sizeof(double) * (size_t)(n > 0 ? n : 1), s));
  if (!c->t2) RBF_TRY(dalloc(c, (void **)&c->t2, sizeof(double) * (size_t)(n > 0 ? n : 1), s));
  if (!c->red_part) RBF_TRY(dalloc(c, (void **)&c->red_part, sizeof(double) * kRedBlocks, s));
  if (!c->red_count) {
    RBF_TRY(dalloc(c, (void **)&c->red_count, sizeof(unsigned), s));
    RBF_CUDA_TRY(cudaMemsetAsync(c->red_count, 0, sizeof(unsigned), s));
  }
  if (!c->hpin) {
    RBF_CUDA_TRY(cudaHostAlloc((void **)&c->hpin, sizeof(double) * (kHpinScal + 8 + c->nranks), cudaHostAllocMapped));
    RBF_CUDA_TRY(cudaHostGetDevicePointer((void **)&c->hpin_dev, c->hpin, 0));
  }
  if (!c->dc_blk) RBF_TRY(dalloc(c, (void **)&c->dc_blk, sizeof(double) * (size_t)kRedBlocks * kDcMaxOut, s));
  if (!c->cg_blk) {
    RBF_TRY(dalloc(c, (void **)&c->cg_blk, sizeof(double) * (size_t)kRedBlocks * kCgMaxM, s));
    RBF_TRY(dalloc(c, (void **)&c->cg_count, sizeof(unsigned), s));
    RBF_CUDA_TRY(cudaMemsetAsync(c->cg_count, 0, sizeof(unsigned), s));
  }
  if (c->nranks == 1 && c->ar_part && c->ar_m < m) {  // per-step partials sized by m
    dfree(c->ar_part, s);
    c->ar_part = nullptr;
    RBF_TRY(dalloc(c, (void **)&c->ar_part, sizeof(double) * part_doubles(c, m), s));
    c->ar_m = m;
  }
  if (c->nranks == 1 && !c->ar_part && c->ar_m == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    RBF_CUDA_TRY(cudaGetDevice(&dev));
    RBF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // the grid must fit both MGS kernels (launch_fused_step picks one of them)
    int per_sm2 = 0;
    RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_arnoldi_fused, kArThreads, 0));
    RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_arnoldi_mgs2, kArThreads, 0));
    per_sm = per_sm < per_sm2 ? per_sm : per_sm2;
    int coop = 0;
    RBF_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    const int ar_per_sm = (int)opt(OPT_ARNOLDI_PER_SM);
    c->ar_grid = (coop && per_sm > 0) ? sms * (per_sm < ar_per_sm ? per_sm : ar_per_sm) : 0;
    if (!opt(OPT_FUSED_ARNOLDI)) c->ar_grid = 0;
    if (c->ar_grid > 0 && (long long)c->ar_grid * kArThreads * kArE < n) c->ar_grid = 0;
    // fused CGS2: same layout as the MGS kernel (w in registers, kArE per thread)
    int cg_per_sm = 0;
    RBF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cg_per_sm, k_arnoldi_cgs2, kArThreads, 0));
    c->cg_grid = (coop && cg_per_sm > 0) ? sms * (cg_per_sm < ar_per_sm ? cg_per_sm : ar_per_sm) : 0;
    if (!opt(OPT_FUSED_ARNOLDI)) c->cg_grid = 0;
    if (c->cg_grid > 0 && (long long)c->cg_grid * kArThreads * kArE < n) c->cg_grid = 0;
    c->ar_m = m;
    if (c->ar_grid > 0 || c->cg_grid > 0) {
      RBF_TRY(dalloc(c, (void **)&c->ar_part, sizeof(double) * part_doubles(c, m), s));
      RBF_TRY(dalloc(c, (void **)&c->ar_bar, sizeof(unsigned) * 2, s));
      RBF_CUDA_TRY(cudaMemsetAsync(c->ar_bar, 0, sizeof(unsigned) * 2, s));
    }
  }
  return RBF_OK;
}

static int grid_for(long long n) {
  long long b = (n + kRedThreads - 1) / kRedThreads;
  return (int)(b < kRedBlocks ? (b > 0 ? b : 1) : kRedBlocks);
}

// out_dev = this rank's partial <a, b> (optionally after w -= coef*x)
static int axpy_dot(rbf_ctx *c, const double *coef, double *w, const double *x, const double *v,
                    double *out_dev, cudaStream_t s) {
  const long long n = n_loc(c);
  k_axpy_dot<<<grid_for(n), kRedThreads, 0, s>>>(coef, c->nranks, w, x, v, n, c->red_part,
                                                  c->red_count, out_dev); count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

// Reduce a scalar slot across ranks: hloc[slot] -> hall[slot*P ...]
static int reduce_slot(rbf_ctx *c, const Scal &L, int slot, cudaStream_t s) {
  if (c->nranks <= 1) return RBF_OK;
  return allgather_scalars(c, c->dscal + L.hloc() + slot, c->dscal + L.hall() + (long long)slot * L.P,
                           1, s);
}

static const double *hall_slot(rbf_ctx *c, const Scal &L, int slot) {
  return c->nranks <= 1 ? c->dscal + L.hloc() + slot : c->dscal + L.hall() + (long long)slot * L.P;
}

static int read_scalars(rbf_ctx *c, const double *src, int count, cudaStream_t s) {
  RBF_CUDA_TRY(cudaMemcpyAsync(c->hpin + kHpinScal, src, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  return RBF_OK;
}

// Global <a, b> (summed over ranks in rank order) to the host.
static int global_dot(rbf_ctx *c, const Scal &L, const double *a, const double *b, double *out,
                      cudaStream_t s) {
  RBF_TRY(axpy_dot(c, nullptr, const_cast<double *>(a), nullptr, b, c->dscal + L.hloc(), s));
  RBF_TRY(reduce_slot(c, L, 0, s));
  RBF_TRY(read_scalars(c, hall_slot(c, L, 0), c->nranks, s));
  double t = 0.0;
  for (int r = 0; r < c->nranks; ++r) t += c->hpin[kHpinScal + r];
  *out = t;
  return RBF_OK;
}

int dot_host(rbf_ctx *c, const double *a, const double *b, double *out, cudaStream_t s) {
  RBF_TRY(ensure_workspace(c, c->V_m > 0 ? c->V_m : 1, s));
  Scal L{c->V_m, c->nranks};
  return global_dot(c, L, a, b, out, s);
}

struct PhaseTimer {  // rotating event sets; a set is read only when it is surely complete
  static constexpr int kSets = 4;
  bool on = false;
  cudaEvent_t e[kSets][4]{};
  double mv = 0, pc = 0, orth = 0;
  int init(bool enable) {
    on = enable;
    if (!on) return RBF_OK;
    for (auto &set : e)
      for (auto &x : set) RBF_CUDA_TRY(cudaEventCreate(&x));
    return RBF_OK;
  }
  void rec(long long seq, int i, cudaStream_t s) {
    if (on) cudaEventRecord(e[seq % kSets][i], s);
  }
  // add the phase times of Arnoldi step `seq` (its events must be complete or
  // `wait` must be set)
  void accumulate(long long seq, bool wait) {
    if (!on || seq < 1) return;
    auto &set = e[seq % kSets];
    if (wait) cudaEventSynchronize(set[3]);
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, set[0], set[1]);
    cudaEventElapsedTime(&b, set[1], set[2]);
    cudaEventElapsedTime(&d, set[2], set[3]);
    mv += a;
    pc += b;
    orth += d;
  }
  ~PhaseTimer() {
    if (on)
      for (auto &set : e)
        for (auto &x : set) cudaEventDestroy(x);
  }
};

// Spin on the mailbox until iteration `seq` has posted (no CUDA API call in the
// fast path; the stream is queried now and then to surface errors).
static int wait_mailbox(rbf_ctx *c, long long seq, cudaStream_t s, double *gabs, double *hn) {
  volatile Mailbox *mb = reinterpret_cast<volatile Mailbox *>(c->hpin) + (seq % kMbSlots);
  for (long long spin = 0; mb->seq != seq; ++spin) {
    if ((spin & 0xfff) == 0xfff) {
      cudaError_t e = cudaStreamQuery(s);
      if (e != cudaSuccess && e != cudaErrorNotReady) {
        set_error("GMRES iteration failed: %s", cudaGetErrorString(e));
        return RBF_ECUDA;
      }
      if (e == cudaSuccess && mb->seq != seq) {  // stream drained but no post: cannot happen
        set_error("GMRES mailbox: iteration %lld never posted", seq);
        return RBF_ECUDA;
      }
    }
  }
  *gabs = mb->gabs;
  *hn = mb->hn;
  return RBF_OK;
}

// ---------------------------------------------------------------------------
// Graph-driven solve (single rank with the fused Arnoldi kernel): the whole
// restarted GMRES is ONE CUDA graph -- an outer while node over restart cycles and
// an inner while node over Arnoldi steps, both driven by cudaGraphSetConditional
// from the kernels that compute the residual estimates -- so no host round trip or
// launch latency sits between iterations and host jitter cannot stall the GPU.
// ---------------------------------------------------------------------------
// the single-rank cooperative Arnoldi kernel for this orthogonalisation is usable
static bool fused_ok(const rbf_ctx *c, int orth) {
  if (orth == RBF_ORTH_DCGS2) return false;  // multi-kernel path (one reduction per step)
  return c->nranks == 1 && c->rec && (orth == RBF_ORTH_CGS2 ? c->cg_grid : c->ar_grid) > 0;
}

static bool graph_path(const rbf_ctx *c, const rbf_gmres_params *gp) {
  return fused_ok(c, gp->orth) && !gp->timing && opt(OPT_SOLVE_GRAPH);
}

// one fused Arnoldi step (cooperative launch); graph mode passes st/hist/inner
static int launch_fused_step(rbf_ctx *c, int orth, double *V, long long n, int k, Scal L,
                             Mailbox *mb, long long seq, const double *w_in, GState *st,
                             double *hist, cudaGraphConditionalHandle inner, cudaStream_t s) {
  double *Sp = c->dscal, *part = c->ar_part;
  unsigned *bar = c->ar_bar;
  long long ldv_ = n, n_ = n, seq_ = seq;
  int k_ = k;
  double4 *rec = c->rec;
  void *args[] = {&V, &ldv_, &n_, &k_, &Sp, &L, &part, &bar, &mb, &seq_, &rec, &w_in, &st, &hist, &inner};
  const bool mgs_pair = opt(OPT_MGS_PAIRS) != 0;  // two MGS projections per grid barrier (reading Q28)
  if (orth == RBF_ORTH_CGS2)
    RBF_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_arnoldi_cgs2, c->cg_grid, kArThreads, args,
                                             0, s));
  else
    RBF_CUDA_TRY(cudaLaunchCooperativeKernel(
        mgs_pair ? (const void *)k_arnoldi_mgs2 : (const void *)k_arnoldi_fused, c->ar_grid, kArThreads,
        args, 0, s));
  count_launch(1);
  return RBF_OK;
}

static int capture_leaf(cudaStream_t s, cudaGraphNode_t *leaf) {
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t *deps = nullptr;
  size_t nd = 0;
  RBF_CUDA_TRY(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd));
  if (nd != 1) {
    set_error("graph capture: expected one leaf node, got %zu", nd);
    return RBF_ECUDA;
  }
  *leaf = deps[0];
  return RBF_OK;
}

static int build_solve_graph_on(rbf_ctx *c, int m, int orth, cudaStream_t s);

static int build_solve_graph(rbf_ctx *c, int m, int orth, cudaStream_t user) {
  // capture on a private stream (the legacy default stream cannot be captured);
  // nothing is executed, so the user stream may still be busy (rbf_setup builds the
  // graph while the RASM setup kernel runs)
  (void)user;
  cudaStream_t cs;
  RBF_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const int st = build_solve_graph_on(c, m, orth, cs);
  cudaStreamDestroy(cs);
  return st;
}

static int build_solve_graph_on(rbf_ctx *c, int m, int orth, cudaStream_t s) {
  const long long n = n_loc(c);
  Scal L{m, 1};
  double *V = c->V, *S = c->dscal, *slot0 = c->dscal + L.hloc();
  GState *st = reinterpret_cast<GState *>(c->g_state);
  const int blocks = grid_for(n);
  if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
  if (c->g_graph) cudaGraphDestroy(c->g_graph);
  c->g_exec = nullptr;
  c->g_graph = nullptr;
  cudaGraph_t G;
  RBF_CUDA_TRY(cudaGraphCreate(&G, 0));
  c->g_graph = G;
  cudaGraphConditionalHandle h_outer, h_inner;
  RBF_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_outer, G, 0, cudaGraphCondAssignDefault));
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  // -- prologue: x = 0, z0 = M^-1 f, ||z0||^2, tolerance, outer condition
  cudaGraphNode_t leaf;
  RBF_CUDA_TRY(cudaStreamBeginCaptureToGraph(s, G, nullptr, nullptr, 0, mode));
  RBF_CUDA_TRY(cudaMemsetAsync(c->g_x, 0, sizeof(double) * (size_t)n, s));
  RBF_TRY(axpy_dot(c, nullptr, c->g_f, nullptr, c->g_f, &st->fsq, s));
  RBF_TRY(launch_rasm_apply(c, c->g_f, V, s));
  RBF_TRY(axpy_dot(c, nullptr, V, nullptr, V, slot0, s));
  k_g_begin<<<1, 1, 0, s>>>(slot0, st, h_outer);
  count_launch(1);
  RBF_TRY(capture_leaf(s, &leaf));
  RBF_CUDA_TRY(cudaStreamEndCapture(s, &G));
  // -- outer while: one restart cycle per iteration
  cudaGraphNodeParams op = {};
  op.type = cudaGraphNodeTypeConditional;
  op.conditional.handle = h_outer;
  op.conditional.type = cudaGraphCondTypeWhile;
  op.conditional.size = 1;
  cudaGraphNode_t outer_node;
  RBF_CUDA_TRY(cudaGraphAddNode(&outer_node, G, &leaf, 1, &op));
  cudaGraph_t B = op.conditional.phGraph_out[0];
  RBF_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_inner, B, 0, cudaGraphCondAssignDefault));
  RBF_CUDA_TRY(cudaStreamBeginCaptureToGraph(s, B, nullptr, nullptr, 0, mode));
  k_g_cycle<<<1, 1, 0, s>>>(S, L, slot0, st, h_inner);
  k_scale_by_norm<<<blocks, kRedThreads, 0, s>>>(V, n, slot0, 1, c->rec);  // v0, pre-packed
  count_launch(2);
  RBF_TRY(capture_leaf(s, &leaf));
  RBF_CUDA_TRY(cudaStreamEndCapture(s, &B));
  // -- inner while: one Arnoldi step per iteration (matvec, RASM apply, fused MGS+Givens)
  cudaGraphNodeParams ip = {};
  ip.type = cudaGraphNodeTypeConditional;
  ip.conditional.handle = h_inner;
  ip.conditional.type = cudaGraphCondTypeWhile;
  ip.conditional.size = 1;
  cudaGraphNode_t inner_node;
  RBF_CUDA_TRY(cudaGraphAddNode(&inner_node, B, &leaf, 1, &ip));
  cudaGraph_t I = ip.conditional.phGraph_out[0];
  RBF_CUDA_TRY(cudaStreamBeginCaptureToGraph(s, I, nullptr, nullptr, 0, mode));
  RBF_TRY(launch_matvec(c, V, c->t1, s, true));
  RBF_TRY(launch_rasm_apply(c, c->t1, c->t2, s));
  RBF_TRY(launch_fused_step(c, orth, V, n, 0, L, nullptr, 0, c->t2, st, c->g_hist, h_inner, s));
  RBF_CUDA_TRY(cudaStreamEndCapture(s, &I));
  // -- end of cycle: x += V y, explicit residual f - A x, z = M^-1 (f - A x), ||z||^2
  RBF_CUDA_TRY(cudaStreamBeginCaptureToGraph(s, B, &inner_node, nullptr, 1, mode));
  k_backsolve_g<<<1, 1, 0, s>>>(S, L, st);
  k_update_x_g<<<blocks, kRedThreads, 0, s>>>(c->g_x, V, n, S, L, st, n);
  count_launch(2);
  RBF_TRY(launch_matvec(c, c->g_x, c->t1, s, false));
  k_sub<<<blocks, kRedThreads, 0, s>>>(c->g_f, c->t1, n);
  count_launch(1);
  RBF_TRY(axpy_dot(c, nullptr, c->t1, nullptr, c->t1, &st->rsq, s));
  RBF_TRY(launch_rasm_apply(c, c->t1, V, s));
  RBF_TRY(axpy_dot(c, nullptr, V, nullptr, V, slot0, s));
  k_g_end_cycle<<<1, 1, 0, s>>>(slot0, st, h_outer);
  count_launch(1);
  RBF_CUDA_TRY(cudaStreamEndCapture(s, &B));
  RBF_CUDA_TRY(cudaGraphInstantiate(&c->g_exec, G, 0));
  c->g_m = m;
  c->g_V = V;
  c->g_orth = orth;
  return RBF_OK;
}

static int prepare_solve_graph(rbf_ctx *c, int m, int max_iters, int orth, cudaStream_t s) {
  const long long n = n_loc(c);
  if (!c->g_state) RBF_TRY(dalloc(c, &c->g_state, sizeof(GState), s));
  if (!c->g_f) RBF_TRY(dalloc(c, (void **)&c->g_f, sizeof(double) * (size_t)(n > 0 ? n : 1), s));
  if (!c->g_x) RBF_TRY(dalloc(c, (void **)&c->g_x, sizeof(double) * (size_t)(n > 0 ? n : 1), s));
  bool rebuild = c->g_exec == nullptr || c->g_m != m || c->g_V != c->V || c->g_orth != orth;
  if (c->g_hist_cap < max_iters) {
    dfree(c->g_hist, s);
    c->g_hist_cap = max_iters > 1024 ? max_iters : 1024;
    RBF_TRY(dalloc(c, (void **)&c->g_hist, sizeof(double) * (size_t)c->g_hist_cap, s));
    rebuild = true;
  }
  if (rebuild) RBF_TRY(build_solve_graph(c, m, orth, s));
  return RBF_OK;
}


// rbf_setup hook: allocate the default GMRES workspace and build the solve graph while
// the RASM setup kernel occupies the GPU (the capture and instantiation are host work).
int prebuild_solve(rbf_ctx *c, cudaStream_t s) {
  rbf_gmres_params gp{};
  gp.restart = 30;
  gp.max_iters = 1000;
  RBF_TRY(ensure_workspace(c, gp.restart, s));
  if (!graph_path(c, &gp)) return RBF_OK;
  return prepare_solve_graph(c, gp.restart, gp.max_iters, gp.orth, s);
}

static int solve_gmres_graph(rbf_ctx *c, const double *f, const rbf_gmres_params *gp, double *x,
                             rbf_report *rep, cudaStream_t s) {
  const int m = gp->restart;
  const long long n = n_loc(c);
  RBF_TRY(prepare_solve_graph(c, m, gp->max_iters, gp->orth, s));
  GState hs{};
  hs.max_iters = gp->max_iters;
  hs.rtol = gp->rtol;
  hs.atol = gp->atol;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  RBF_CUDA_TRY(cudaEventCreate(&t0));
  RBF_CUDA_TRY(cudaEventCreate(&t1));
  RBF_CUDA_TRY(cudaMemcpyAsync(c->g_state, &hs, sizeof(GState), cudaMemcpyHostToDevice, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(c->g_f, f, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s));
  RBF_CUDA_TRY(cudaEventRecord(t0, s));
  RBF_CUDA_TRY(cudaGraphLaunch(c->g_exec, s));
  RBF_CUDA_TRY(cudaEventRecord(t1, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(x, c->g_x, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&hs, c->g_state, sizeof(GState), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  // launches executed by the graph: prologue 3 (+ matvec/apply), per cycle 12, per step 4
  const int cycles = hs.it > 0 ? hs.restarts + 1 : 0;
  count_launch(4 + 12 * cycles + 4 * hs.it);
  const bool converged = hs.conv != 0;
  int status = RBF_OK;
  if (hs.nan) status = RBF_ENUMERIC;
  else if (!converged) status = RBF_NOT_CONVERGED;
  if (rep) {
    int hl = 0;
    if (rep->history && rep->history_cap > 0 && hs.it > 0) {
      hl = hs.it < rep->history_cap ? hs.it : rep->history_cap;
      RBF_CUDA_TRY(cudaMemcpy(rep->history, c->g_hist, sizeof(double) * hl, cudaMemcpyDeviceToHost));
    }
    // the graph's last cycle left ||f - A x||^2 and ||M^-1 (f - A x)|| in the state
    const double fsq = hs.fsq, rsq = hs.it > 0 ? hs.rsq : 0.0;
    const double psq = hs.it > 0 ? hs.beta_last * hs.beta_last : 0.0;
    double last = 0.0;
    if (hs.it > 0) RBF_CUDA_TRY(cudaMemcpy(&last, c->g_hist + hs.it - 1, sizeof(double), cudaMemcpyDeviceToHost));
    rep->iterations = hs.it;
    rep->converged = converged;
    rep->restarts = hs.restarts;
    rep->beta0 = hs.beta0;
    rep->resid_est = hs.it > 0 ? last : 0.0;
    rep->resid_true = fsq > 0 ? std::sqrt(rsq / fsq) : 0.0;
    rep->resid_precond = hs.beta0 > 0 ? std::sqrt(psq) / hs.beta0 : 0.0;
    rep->history_len = hl;
    rep->ms_matmult = rep->ms_pcapply = rep->ms_orth = 0.0;
    rep->ms_total = ms;
    rep->status = status;
  }
  return status;
}

int solve_gmres(rbf_ctx *c, const double *f, const rbf_gmres_params *gp, double *x,
                rbf_report *rep, cudaStream_t s) {
  const int m = gp->restart;
  const long long n = n_loc(c);
  RBF_TRY(ensure_workspace(c, m, s));
  if (graph_path(c, gp)) return solve_gmres_graph(c, f, gp, x, rep, s);
  Scal L{m, c->nranks};
  Op op{c, s};
  double *V = c->V;
  const long long ldv = n;
  PhaseTimer pt;
  RBF_TRY(pt.init(gp->timing != 0));
  cudaEvent_t t_begin = nullptr, t_end = nullptr;  // ms_total (always recorded)
  RBF_CUDA_TRY(cudaEventCreate(&t_begin));
  RBF_CUDA_TRY(cudaEventCreate(&t_end));
  RBF_CUDA_TRY(cudaEventRecord(t_begin, s));
  const int blocks = grid_for(n);
  const int orth = gp->orth;
  const bool fused = fused_ok(c, orth);
  const bool prepack = fused;  // the fused kernels write v_{k+1} into the matvec records

  RBF_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, s));
  // beta0 = ||M^-1 f||  (x0 = 0)
  RBF_TRY(op.pc(f, V));
  double beta0sq = 0.0;
  RBF_TRY(global_dot(c, L, V, V, &beta0sq, s));
  const double beta0 = std::sqrt(beta0sq);
  int it = 0, restarts = 0, converged = 0, status = RBF_OK, hist_len = 0;
  double resid_est = 0.0;
  if (beta0 == 0.0) {
    converged = 1;
  } else {
    const double tol = std::fmax(gp->rtol * beta0, gp->atol);
    long long seq_enq = 0, seq_base = 0;  // Arnoldi steps enqueued; steps before this cycle
    for (int i = 0; i < kMbSlots; ++i) reinterpret_cast<volatile Mailbox *>(c->hpin)[i].seq = -1;
    for (;;) {
      int kend = 0;
      bool done = false;
      if (orth == RBF_ORTH_DCGS2) {
        // ---- delayed CGS2, one reduction per step (reading Q27): V0 holds u_0 (the
        // unscaled preconditioned residual); step k (0..m) applies the operator to u_k,
        // reduces [V_{<k}, u_k]^T [u_k, w] once, finishes column k-1 (mailbox) and
        // forms v_k and u_{k+1}.  The host waits for column kc at step kc+1 while step
        // kc+2 is already enqueued (one-step lookahead, as for MGS).
        const int P = c->nranks;
        const bool pk = P == 1 && c->rec != nullptr;  // u_{k+1} packed by the sweep
        double *S = c->dscal;
        double *dl = S + L.dloc(), *da = P > 1 ? S + L.dall() : dl;
        Mailbox *mb = reinterpret_cast<Mailbox *>(c->hpin_dev);
        auto enqueue_d = [&](int k) -> int {
          const long long seq = ++seq_enq;
          double *u = V + (long long)k * ldv;
          double *w = V + (long long)(k + 1) * ldv;
          pt.rec(seq, 0, s);
          if (k < m) RBF_TRY(op.matvec(u, c->t1, pk && k > 0));
          pt.rec(seq, 1, s);
          if (k < m) RBF_TRY(op.pc(c->t1, w));
          pt.rec(seq, 2, s);
          k_dcgs_dots<<<grid_for(n), kRedThreads, 0, s>>>(V, ldv, k, n, k < m ? w : nullptr, c->dc_blk,
                                                          c->cg_count, dl);
          count_launch(1);
          if (P > 1) RBF_TRY(allgather_scalars(c, dl, da, 2 * (k + 1), s));
          k_dcgs_scalar<<<1, 1, 0, s>>>(S, L, da, k, mb, seq);
          count_launch(1);
          if (k < m) {
            k_dcgs_update<<<blocks, kRedThreads, 0, s>>>(V, ldv, k, n, S, L, pk ? c->rec : nullptr);
            count_launch(1);
          }
          RBF_CUDA_TRY(cudaGetLastError());
          pt.rec(seq, 3, s);
          return RBF_OK;
        };
        RBF_TRY(enqueue_d(0));
        RBF_TRY(enqueue_d(1));
        for (int kc = 0; kc < m; ++kc) {
          if (kc + 2 <= m && it + 1 < gp->max_iters) RBF_TRY(enqueue_d(kc + 2));
          double gabs = 0.0, hn = 0.0;
          RBF_TRY(wait_mailbox(c, seq_base + kc + 2, s, &gabs, &hn));  // step kc+1
          pt.accumulate(seq_base + kc + 1, false);                     // step kc: complete
          ++it;
          resid_est = gabs / beta0;
          if (rep && rep->history && hist_len < rep->history_cap) rep->history[hist_len++] = resid_est;
          kend = kc + 1;
          if (!std::isfinite(gabs) || !std::isfinite(hn)) {
            status = RBF_ENUMERIC;
            done = true;
            break;
          }
          if (gabs <= tol || hn == 0.0) {
            converged = 1;
            done = true;
            break;
          }
          if (it >= gp->max_iters) {
            done = true;
            break;
          }
        }
        if (kend >= 1) pt.accumulate(seq_base + kend + 1, true);
      } else {
      // V0 holds the unscaled preconditioned residual; its ||.||^2 is in slot 0
      k_cycle_init<<<1, 1, 0, s>>>(c->dscal, L, hall_slot(c, L, 0)); count_launch(1);
      k_scale_by_norm<<<blocks, kRedThreads, 0, s>>>(V, n, hall_slot(c, L, 0), L.P, prepack ? c->rec : nullptr);
      count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
      // enqueue Arnoldi step k (matvec, preconditioner, orthogonalisation, Givens)
      auto enqueue = [&](int k) -> int {
        double *vk = V + (long long)k * ldv;
        double *w = V + (long long)(k + 1) * ldv;
        const long long seq = ++seq_enq;
        pt.rec(seq, 0, s);
        // single rank: the basis vector v_k was written into the matvec records by the
        // kernel that produced it (cycle start or the previous Arnoldi step)
        RBF_TRY(op.matvec(vk, c->t1, prepack));
        pt.rec(seq, 1, s);
        RBF_TRY(op.pc(c->t1, w));
        pt.rec(seq, 2, s);
        Mailbox *mb = reinterpret_cast<Mailbox *>(c->hpin_dev);
        if (fused) {
          // single rank: orthogonalisation + norm + scale + Givens in one cooperative launch
          RBF_TRY(launch_fused_step(c, orth, V, n, k, L, mb, seq, nullptr, nullptr, nullptr, 0, s));
        } else if (orth == RBF_ORTH_CGS2) {
          // classical Gram-Schmidt twice: three passes, one all-gather each (reading Q23)
          const int cnt = k + 1, P = c->nranks, gb = grid_for(n);
          double *S = c->dscal;
          double *c1l = S + L.c1loc(), *c2l = S + L.c2loc();
          double *c1a = P > 1 ? S + L.c1all() : c1l, *c2a = P > 1 ? S + L.c2all() : c2l;
          k_cgs_pass<0><<<gb, kRedThreads, 0, s>>>(w, V, ldv, cnt, n, nullptr, P, c->cg_blk,
                                                   c->cg_count, c1l);
          count_launch(1);
          if (P > 1) RBF_TRY(allgather_scalars(c, c1l, c1a, cnt, s));
          k_cgs_pass<1><<<gb, kRedThreads, 0, s>>>(w, V, ldv, cnt, n, c1a, P, c->cg_blk, c->cg_count,
                                                   c2l);
          count_launch(1);
          if (P > 1) RBF_TRY(allgather_scalars(c, c2l, c2a, cnt, s));
          k_cgs_pass<2><<<gb, kRedThreads, 0, s>>>(w, V, ldv, cnt, n, c2a, P, c->cg_blk, c->cg_count,
                                                   S + L.hloc() + k + 1);
          count_launch(1);
          RBF_TRY(reduce_slot(c, L, k + 1, s));
          k_givens<<<1, 1, 0, s>>>(S, L, hall_slot(c, L, 0), k, mb, seq, c1a, c2a);
          count_launch(1);
          k_scale_by_norm<<<blocks, kRedThreads, 0, s>>>(w, n, hall_slot(c, L, k + 1), L.P, nullptr);
          count_launch(1);
        } else {
          for (int j = 0; j <= k; ++j) {  // modified Gram-Schmidt, fused axpy + dot
            const double *coef = (j > 0) ? hall_slot(c, L, j - 1) : nullptr;
            const double *xprev = (j > 0) ? V + (long long)(j - 1) * ldv : nullptr;
            RBF_TRY(axpy_dot(c, coef, w, xprev, V + (long long)j * ldv, c->dscal + L.hloc() + j, s));
            RBF_TRY(reduce_slot(c, L, j, s));
          }
          RBF_TRY(axpy_dot(c, hall_slot(c, L, k), w, vk, w, c->dscal + L.hloc() + k + 1, s));
          RBF_TRY(reduce_slot(c, L, k + 1, s));
          k_givens<<<1, 1, 0, s>>>(c->dscal, L, hall_slot(c, L, 0), k, mb, seq, nullptr, nullptr);
          count_launch(1);
          k_scale_by_norm<<<blocks, kRedThreads, 0, s>>>(w, n, hall_slot(c, L, k + 1), L.P, nullptr);
          count_launch(1);
        }
        RBF_CUDA_TRY(cudaGetLastError());
        pt.rec(seq, 3, s);
        return RBF_OK;
      };
      // One-iteration lookahead: step k+1 is enqueued before the host waits for
      // step k's residual.  If step k converges, step k+1's writes (V[k+2], H column
      // k+1, g[k+1..k+2]) are outside what the solution update reads.
      RBF_TRY(enqueue(0));
      for (int k = 0; k < m; ++k) {
        if (k + 1 < m && it + 1 < gp->max_iters) RBF_TRY(enqueue(k + 1));
        double gabs = 0.0, hn = 0.0;
        RBF_TRY(wait_mailbox(c, seq_base + k + 1, s, &gabs, &hn));
        if (k >= 1) pt.accumulate(seq_base + k, false);  // previous step: events complete
        ++it;
        resid_est = gabs / beta0;
        if (rep && rep->history && hist_len < rep->history_cap) rep->history[hist_len++] = resid_est;
        kend = k + 1;
        if (!std::isfinite(gabs) || !std::isfinite(hn)) {
          status = RBF_ENUMERIC;
          done = true;
          break;
        }
        if (gabs <= tol || hn == 0.0) {
          converged = 1;
          done = true;
          break;
        }
        if (it >= gp->max_iters) {
          done = true;
          break;
        }
      }
      if (kend >= 1) pt.accumulate(seq_base + kend, true);  // last step of the cycle
      }  // MGS / CGS2
      seq_base = seq_enq;
      k_backsolve<<<1, 1, 0, s>>>(c->dscal, L, kend); count_launch(1);
      k_update_x<<<blocks, kRedThreads, 0, s>>>(x, V, ldv, c->dscal, L, kend, n); count_launch(1);
      RBF_CUDA_TRY(cudaGetLastError());
      if (done) break;
      // restart: V0 = M^-1 (f - A x), explicitly
      RBF_TRY(op.matvec(x, c->t1));
      k_sub<<<blocks, kRedThreads, 0, s>>>(f, c->t1, n); count_launch(1);
      RBF_TRY(op.pc(c->t1, V));
      double bsq = 0.0;
      RBF_TRY(global_dot(c, L, V, V, &bsq, s));
      ++restarts;
      const double beta = std::sqrt(bsq);
      if (beta <= tol) {
        converged = 1;
        resid_est = beta / beta0;
        break;
      }
    }
  }
  double ms_total = 0.0;
  {
    RBF_CUDA_TRY(cudaEventRecord(t_end, s));
    RBF_CUDA_TRY(cudaEventSynchronize(t_end));
    float ms = 0;
    cudaEventElapsedTime(&ms, t_begin, t_end);
    ms_total = ms;
    cudaEventDestroy(t_begin);
    cudaEventDestroy(t_end);
  }
  if (rep) {
    // explicit residuals (not part of the timed solve)
    double fsq = 0.0, rsq = 0.0, psq = 0.0;
    RBF_TRY(global_dot(c, L, f, f, &fsq, s));
    RBF_TRY(op.matvec(x, c->t1));
    k_sub<<<blocks, kRedThreads, 0, s>>>(f, c->t1, n); count_launch(1);
    RBF_TRY(global_dot(c, L, c->t1, c->t1, &rsq, s));
    RBF_TRY(op.pc(c->t1, c->t2));
    RBF_TRY(global_dot(c, L, c->t2, c->t2, &psq, s));
    rep->iterations = it;
    rep->converged = converged;
    rep->restarts = restarts;
    rep->beta0 = beta0;
    rep->resid_est = resid_est;
    rep->resid_true = fsq > 0 ? std::sqrt(rsq / fsq) : 0.0;
    rep->resid_precond = beta0 > 0 ? std::sqrt(psq) / beta0 : 0.0;
    rep->history_len = hist_len;
    rep->ms_matmult = pt.mv;
    rep->ms_pcapply = pt.pc;
    rep->ms_orth = pt.orth;
    rep->ms_total = ms_total;
  }
  if (status == RBF_OK && !converged) status = RBF_NOT_CONVERGED;
  if (rep) rep->status = status;
  return status;
}

}  // namespace rbf
