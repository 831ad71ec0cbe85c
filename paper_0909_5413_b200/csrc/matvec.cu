// matvec.cu -- fp64 cutoff-Gaussian matvec (Eq.(12)).
//
//   y_i = norm * sum_{j : fma(dx,dx,dy*dy) < rc^2} w_j exp(-r2_ij / (2 sigma^2))
//
// over the (2kh+1)^2 cell stencil around the target's cell (row-major keys make it
// 2kh+1 contiguous runs of the sorted arrays).
//
// The truncated operator is applied matrix-free in its VALUES (every entry is
// recomputed, "without actually storing the matrix"), but its sparsity
// pattern -- which of the stencil's sources lie within rc of each target -- is
// found once in rbf_setup (the exact fp64 test of reading Q1) and kept as an
// ELLPACK-style list of 32-bit source indices, 4 bytes per in-cutoff pair (O(N)
// storage).  A matvec then spends its FP64 pipe only on in-cutoff pairs.
//
// Layout (B200): one warp per chunk of 32 CONSECUTIVE targets (sorted order; chunks
// ignore cell boundaries, so all 32 lanes carry work), lanes walk their own lists in
// lock step, 4 entries per coalesced 16-byte load.  The sources are gathered from a
// packed record array {x, y, w, 0} -- ONE 256-bit load (LDG.E.ENL2.256) per pair --
// whose w slot is refreshed by k_pack_w before each matvec.  The L1 data pipe, not
// the FP64 pipe, is what a gather-based matvec saturates first (ncu, profiles/), so
// every byte through L1 counts: 32 B per pair for the record, 4 B for the index.
//
// exp() runs on the FP64 pipe with no table: k = round(-r2 log2e/(2s^2)),
// f = -r2 log2e/(2 s^2) - k in [-1/2, 1/2] (one fma from the exact product), 2^f =
// 1 + f P(f) with P a minimax polynomial of degree DEG (default 9: max relative
// error 3.9e-16 ~ 3.5 ulp; 10: 1.5e-16; reading Q15), 2^k by an integer add to the
// exponent field.  (A 64-entry table
// variant, replicated per lane in shared memory, was measured slower: the table
// loads compete with the gathers for the L1 data pipe; profiles/.)
//
// Padding entries point at the target itself (a finite term) and are masked by a
// predicated accumulate, so the per-target sum is exactly the sum over its list in
// stencil order (rows, then sorted order): deterministic and bitwise identical for
// any strip decomposition (reading Q20).
#include <cub/cub.cuh>

#include <cstdlib>

#include "common.cuh"

namespace rbf {

constexpr int kMvWarps = 8;  // target chunks per CTA
constexpr int kMvThreads = 32 * kMvWarps;


__device__ __forceinline__ int target_cell(const Geom &g, double2 p, int &cx, int &cy) {
  double tx = floor(__ddiv_rn(__dsub_rn(p.x, g.x0), g.cell));
  double ty = floor(__ddiv_rn(__dsub_rn(p.y, g.y0), g.cell));
  cx = (int)fmin(fmax(tx, 0.0), (double)(g.ncx - 1));
  cy = (int)fmin(fmax(ty, 0.0), (double)(g.ncy - 1));
  return cy * g.ncx + cx;
}

// ---------------------------------------------------------------------------
// Neighbour-list build (setup).  Each lane owns G consecutive targets (sorted
// order) and walks the UNION of their in-cutoff lists: one record load then serves
// G pairs, dividing the L1 bytes per pair by ~G (at ~88% slot efficiency for G = 2
// on lattices; the masked-off slots are computed and discarded).  Entry =
// source index (ext-relative) | bit (31 - j) set iff the source is within rc of
// target j.  The union is enumerated in stencil order over the bounding box of the
// G stencils, so each target sees exactly its own list in its own stencil order:
// sums are bitwise independent of G and of the strip decomposition (reading Q20).
// One thread per lane; a warp = a chunk of 32 G targets.
// MODE 0: union length per chunk (max over lanes, rounded up to 4).
// MODE 1: write the entries (ELL, groups of 4 per lane) and the padding (mask 0).
// ---------------------------------------------------------------------------
template <int G>
struct MvIdx {
  static constexpr unsigned kIdxMask = (1u << (32 - G)) - 1u;
  static __device__ __forceinline__ unsigned bit(int j) { return 1u << (31 - j); }
};

// The G local targets of lane lt: tgt[lt] (pairs chosen at setup, -1 = none) when
// given, else G consecutive targets.
template <int G>
__device__ __forceinline__ void lane_targets(const int4 *__restrict__ tgt, long long lt, long long nloc,
                                             long long nlanes, int *t) {
  if (G >= 2 && tgt) {
    const int4 v = lt < nlanes ? tgt[lt] : make_int4(-1, -1, -1, -1);
    t[0] = v.x;
    if (G > 1) t[1] = v.y;
    if (G > 2) t[G - 1] = v.z;
  } else {
#pragma unroll
    for (int j = 0; j < G; ++j) t[j] = lt * G + j < nloc ? (int)(lt * G + j) : -1;
  }
}

// 16-bit entries (W16, G = 2 only): [15:14] the two targets' mask bits, [13:11] the rows
// the lane's box walk advanced since its previous entry, [10:0] the offset from the start
// of the current row's run (cell_start[(by0 + row) ncx + bx0]); the lane's box corner key
// by0 ncx + bx0 is kept in its lane_tgt .w.  MODE 0 reports the largest offset and row
// step (fmt[0], fmt[1]) so the host picks 16-bit entries only when they fit.
template <int MODE, int G, bool W16 = false, bool ST = false>
__global__ __launch_bounds__(kMvThreads) void k_nlist(Geom g, Strip st, const double2 *__restrict__ xy,
                                                      const int *__restrict__ cell_start, long long nloc,
                                                      int4 *__restrict__ tgt, long long nlanes,
                                                      int *__restrict__ chunk_len,
                                                      const long long *__restrict__ chunk_off,
                                                      void *__restrict__ list_v,
                                                      unsigned long long *__restrict__ n_union,
                                                      int *__restrict__ lane_len, int *__restrict__ fmt,
                                                      const int4 *__restrict__ win = nullptr) {
  unsigned *list = reinterpret_cast<unsigned *>(list_v);
  unsigned short *list16 = reinterpret_cast<unsigned short *>(list_v);
  const long long lt = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // lane-group
  int t[G];
  lane_targets<G>(tgt, lt, nloc, nlanes, t);
  const int lane = threadIdx.x & 31;
  const long long ch = lt >> 5;
  const bool in_chunk = (ch << 5) < nlanes;  // lanes past the end of a ragged last chunk
  const long long own_off = st.own_lo - st.ext_lo;
  int cnt = 0;
  long long base = 0;
  if (MODE == 1 && in_chunk) base = chunk_off[ch];
  double2 p[G];
  bool act[G];
  CellBox tb[G];  // T-box of each target's cell (reading Q25; used when g.tw > 0)
  const bool tbox = g.tw > 0.0;
  int bx0 = g.ncx, bx1 = -1, by0 = g.ncy, by1 = -1;
#pragma unroll
  for (int j = 0; j < G; ++j) {
    act[j] = t[j] >= 0;
    p[j] = xy[own_off + (act[j] ? t[j] : 0)];
    int cx = 0, cy = 0;
    if (act[j]) target_cell(g, p[j], cx, cy);
    tb[j] = cell_box(g, cx, cy, g.tw);
    if (act[j]) {
      bx0 = min(bx0, max(cx - g.kh, 0));
      bx1 = max(bx1, min(cx + g.kh, g.ncx - 1));
      by0 = min(by0, max(cy - g.kh, 0));
      by1 = max(by1, min(cy + g.kh, g.ncy - 1));
    }
  }
  int prev_row = 0, max_off = 0, max_step = 0;
  uint4 grp = make_uint4(0, 0, 0, 0);  // MODE 1, 32-bit: the lane's current group of four
  // matvec variant 5: entries are slots of the CTA's staged window (its rows' runs
  // [cell_start(by, wbx0), cell_start(by, wbx1 + 1)) back to back) instead of indices
  int4 wv = make_int4(-1, -1, 0, -1);
  if (ST && MODE == 1 && in_chunk) wv = win[lt / kMvThreads];
  const bool staged = ST && wv.x >= 0;
  long long wslot = 0;  // slot of the first source of row wv.z + r, advanced row by row
  if (staged)
    for (int by = wv.z; by < by0; ++by)
      wslot += cell_start[by * g.ncx + wv.y + 1] - cell_start[by * g.ncx + wv.x];
  const double mg = 1e-9 * g.cell;
  for (int by = by0; by <= by1; ++by) {
    const int s0 = cell_start[by * g.ncx + bx0];
    const long long rs = staged ? wslot + (s0 - cell_start[by * g.ncx + wv.x]) : 0;
    if (staged) wslot += cell_start[by * g.ncx + wv.y + 1] - cell_start[by * g.ncx + wv.x];
    // radial cutoff: only the cells of this row that the targets' discs reach in x (the
    // row's distance from a target, less a margin, bounds |dy| from below); the skipped
    // sources carry no mask bit, so the list (entries, order, offsets from s0) is unchanged
    int xa = bx0, xb = bx1;
    if (!tbox) {
      const double lo = g.y0 + by * g.cell, hi = lo + g.cell;
      double wl = 1e300, wh = -1e300;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const double dy = fmax(fmax(fmax(lo - p[j].y, p[j].y - hi), 0.0) - mg, 0.0);
        const double w2 = g.rc2 - dy * dy;
        if (act[j] && w2 > 0.0) {
          const double wx = sqrt(w2) + mg;
          wl = fmin(wl, p[j].x - wx);
          wh = fmax(wh, p[j].x + wx);
        }
      }
      if (wl <= wh) {
        xa = max(bx0, (int)floor((wl - g.x0) / g.cell));
        xb = min(bx1, (int)floor((wh - g.x0) / g.cell));
      } else {
        xb = xa - 1;
      }
    }
    const int s_lo = xa <= xb ? cell_start[by * g.ncx + xa] : 0;
    const int s1 = xa <= xb ? cell_start[by * g.ncx + xb + 1] : 0;
    for (int s = s_lo; s < s1; ++s) {
      const double2 o = xy[s - st.ext_lo];
      unsigned m = 0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const double dx = p[j].x - o.x, dy = p[j].y - o.y;
        const bool in = tbox ? in_box(tb[j], o.x, o.y) : fma(dx, dx, dy * dy) < g.rc2;
        if (act[j] && in) m |= MvIdx<G>::bit(j);
      }
      if (m) {
        const int row = by - by0, step = row - prev_row, off = s - s0;
        prev_row = row;
        max_off = max(max_off, off);
        max_step = max(max_step, step);
        const long long at = base + ((long long)(cnt >> 2) * 32 + lane) * 4 + (cnt & 3);
        if (MODE == 1 && W16) {
          list16[at] = (unsigned short)((m >> 16) | ((unsigned)step << 11) | (unsigned)off);
        } else if (MODE == 1) {  // four entries per 16-byte store (full sectors)
          const unsigned v = (unsigned)(staged ? rs + (s - s0) : s - st.ext_lo) | m;
          const int q = cnt & 3;
          if (q == 0) grp.x = v;
          else if (q == 1) grp.y = v;
          else if (q == 2) grp.z = v;
          else {
            grp.w = v;
            *reinterpret_cast<uint4 *>(list + (at - 3)) = grp;
          }
        }
        ++cnt;
      }
    }
  }
  if (MODE == 0) {
    max_off = __reduce_max_sync(0xffffffffu, max_off);
    max_step = __reduce_max_sync(0xffffffffu, max_step);
    if (lane == 0 && fmt) {
      atomicMax(&fmt[0], max_off);
      atomicMax(&fmt[1], max_step);
    }
    if (tgt && lt < nlanes) tgt[lt].w = bx1 >= bx0 ? by0 * g.ncx + bx0 : -1;  // the lane's box corner
  }
  const int kmax = (__reduce_max_sync(0xffffffffu, cnt) + 3) & ~3;  // groups of 4
  if (MODE == 0) {
    if (lane == 0 && in_chunk) chunk_len[ch] = kmax;
    if (lane_len && lt < nlanes) lane_len[lt] = cnt;
    const int csum = __reduce_add_sync(0xffffffffu, cnt);  // union entries (statistics)
    if (lane == 0 && csum) atomicAdd(n_union, (unsigned long long)csum);
  } else if (in_chunk) {  // padding: no mask bit (32-bit: the lane's first target; 16-bit:
                          // offset 0 of the current row, clamped into the ext range)
    const unsigned self = staged ? 0u : (unsigned)(own_off + (act[0] ? t[0] : 0));
    if (W16) {
      for (int k = cnt; k < kmax; ++k) list16[base + ((long long)(k >> 2) * 32 + lane) * 4 + (k & 3)] = 0;
    } else {
      for (int k = cnt; k < kmax; ++k) {
        const int q = k & 3;
        if (q == 0) grp.x = self;
        else if (q == 1) grp.y = self;
        else if (q == 2) grp.z = self;
        else {
          grp.w = self;
          *reinterpret_cast<uint4 *>(list + base + ((long long)(k >> 2) * 32 + lane) * 4) = grp;
        }
      }
    }
  }
}

__global__ void k_len_to_entries(const int *__restrict__ len, long long n, long long *__restrict__ out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = 32LL * len[i];
}

__global__ void k_init_rec(const double2 *__restrict__ xy, long long n, double4 *__restrict__ rec) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) rec[i] = make_double4(xy[i].x, xy[i].y, 0.0, 0.0);
}

// w slot of the records (ext range); one streaming pass, 8 B in / 8 B out per point.
__global__ void k_pack_w(const double *__restrict__ w, long long n, double4 *__restrict__ rec) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) reinterpret_cast<double *>(rec + i)[2] = w[i];
}

// ---------------------------------------------------------------------------
// Matvec variant 5 (A/B measurement of the staged design, SURVEY §8.a2 / DESIGN.md §6):
// each CTA's sources -- the union box of its lanes' stencils, 2kh+1 (or 2kh+2) cell
// rows, each one contiguous run of the sorted records -- are copied into shared memory
// by one 1-D bulk copy per row (cp.async.bulk, mbarrier completion) and the lanes gather
// from there; list entries are window slots.  CTAs whose window exceeds kMvStageMax
// records (targets spanning two cell rows, the cells' leftover singles) keep the global
// gathers.
// ---------------------------------------------------------------------------
constexpr int kMvStageMax = 3400;  // records per CTA window (106 KB: two CTAs per SM)

__global__ __launch_bounds__(kMvThreads) void k_mv_windows(Geom g, Strip st, const double2 *__restrict__ xy,
                                                           const int *__restrict__ cell_start, long long nloc,
                                                           const int4 *__restrict__ tgt, long long nlanes,
                                                           int4 *__restrict__ win) {
  __shared__ int sb[4];
  if (threadIdx.x == 0) { sb[0] = g.ncx; sb[1] = -1; sb[2] = g.ncy; sb[3] = -1; }
  __syncthreads();
  const long long lt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int t[2];
  lane_targets<2>(tgt, lt, nloc, nlanes, t);
  const long long own_off = st.own_lo - st.ext_lo;
  for (int j = 0; j < 2; ++j) {
    if (t[j] < 0) continue;
    int cx = 0, cy = 0;
    target_cell(g, xy[own_off + t[j]], cx, cy);
    atomicMin(&sb[0], max(cx - g.kh, 0));
    atomicMax(&sb[1], min(cx + g.kh, g.ncx - 1));
    atomicMin(&sb[2], max(cy - g.kh, 0));
    atomicMax(&sb[3], min(cy + g.kh, g.ncy - 1));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int by = sb[2]; by <= sb[3]; ++by)
      tot += cell_start[by * g.ncx + sb[1] + 1] - cell_start[by * g.ncx + sb[0]];
    win[blockIdx.x] = (sb[1] >= sb[0] && tot <= kMvStageMax) ? make_int4(sb[0], sb[1], sb[2], sb[3])
                                                             : make_int4(-1, -1, 0, -1);
  }
}

__device__ __forceinline__ void mbar_init(unsigned long long *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *m, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(m);
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(a), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(m))
               : "memory");
}

template <int DEG, int MINB>
__global__ __launch_bounds__(kMvThreads, MINB) void k_matvec_st(
    Geom g, Strip st, long long nloc, long long own_off, const double4 *__restrict__ rec,
    const int *__restrict__ cell_start, const int4 *__restrict__ win, const int4 *__restrict__ tgt,
    long long nlanes, const int *__restrict__ chunk_len, const long long *__restrict__ chunk_off,
    const unsigned *__restrict__ list, double *__restrict__ y) {
  extern __shared__ __align__(16) double4 srec[];
  __shared__ __align__(8) unsigned long long mbar;
  const int lane = threadIdx.x & 31;
  const int4 wv = win[blockIdx.x];
  const bool staged = wv.x >= 0;  // uniform per CTA
  if (staged && threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    long long tot = 0;
    for (int by = wv.z; by <= wv.w; ++by)
      tot += cell_start[by * g.ncx + wv.y + 1] - cell_start[by * g.ncx + wv.x];
    mbar_expect_tx(&mbar, (unsigned)(tot * sizeof(double4)));
    long long slot = 0;
    for (int by = wv.z; by <= wv.w; ++by) {
      const int s0 = cell_start[by * g.ncx + wv.x], s1 = cell_start[by * g.ncx + wv.y + 1];
      if (s1 > s0) bulk_g2s(srec + slot, rec + (s0 - st.ext_lo), (unsigned)((s1 - s0) * sizeof(double4)), &mbar);
      slot += s1 - s0;
    }
  }
  __syncthreads();
  const long long lt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ch = lt >> 5;
  int t[2];
  lane_targets<2>(tgt, lt, nloc, nlanes, t);
  double2 me[2];
  double acc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double4 r = rec[own_off + (t[j] >= 0 ? t[j] : 0)];
    me[j] = make_double2(r.x, r.y);
    acc[j] = 0.0;
  }
  if (staged) mbar_wait(&mbar, 0);
  if ((ch << 5) < nlanes) {
    const int K = chunk_len[ch];
    const uint4 *lp = reinterpret_cast<const uint4 *>(list + chunk_off[ch]) + lane;
    const double esc = g.esc;
    uint4 nxt = (K > 0) ? __ldcs(lp) : make_uint4(0, 0, 0, 0);
    for (int k = 0; k < K; k += 4) {
      const uint4 ev = nxt;
      if (k + 4 < K) nxt = __ldcs(lp + ((k >> 2) + 1) * 32);
      const unsigned es[4] = {ev.x, ev.y, ev.z, ev.w};
      double4 o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned idx = es[u] & MvIdx<2>::kIdxMask;
        o[u] = staged ? srec[idx] : ld_rec(rec + idx);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double dx = me[j].x - o[u].x, dy = me[j].y - o[u].y;
          const double e = gauss_exp2<DEG>(fma(dx, dx, dy * dy), esc);
          if (es[u] & MvIdx<2>::bit(j)) acc[j] = fma(o[u].z, e, acc[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (t[j] >= 0) y[t[j]] = acc[j] * g.norm;
  }
}

// ---------------------------------------------------------------------------
// The matvec: one warp per chunk of 32 G consecutive targets, G per lane; U list
// entries (U record gathers) in flight per lane.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int G, int DEG, int U, int MINB, bool PF = false>
__global__ __launch_bounds__(kMvThreads, MINB) void k_matvec(
    Geom g, long long nloc, long long own_off, const double4 *__restrict__ rec,
    const int4 *__restrict__ tgt, long long nlanes,
    const int *__restrict__ chunk_len, const long long *__restrict__ chunk_off,
    const unsigned *__restrict__ list, double *__restrict__ y, long long lane0) {
  const int lane = threadIdx.x & 31;
  const long long lt = lane0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ch = lt >> 5;
  if ((ch << 5) >= nlanes) return;  // whole warp beyond the last chunk
  int t[G];
  lane_targets<G>(tgt, lt, nloc, nlanes, t);
  double2 me[G];
  double acc[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const double4 r = rec[own_off + (t[j] >= 0 ? t[j] : 0)];
    me[j] = make_double2(r.x, r.y);
    acc[j] = 0.0;
  }
  const int K = chunk_len[ch];  // multiple of 4
  const uint4 *lp = reinterpret_cast<const uint4 *>(list + chunk_off[ch]) + lane;
  const double esc = g.esc;
  uint4 nxt = (K > 0) ? __ldcs(lp) : make_uint4(0, 0, 0, 0);
  for (int k = 0; k < K; k += 4) {
    const uint4 ev = nxt;
    if (k + 4 < K) nxt = __ldcs(lp + ((k >> 2) + 1) * 32);
    const unsigned es[4] = {ev.x, ev.y, ev.z, ev.w};
    if (PF && k + 4 < K) {  // the next group's records into L1 while this group computes
      prefetch_l1(rec + (nxt.x & MvIdx<G>::kIdxMask));
      prefetch_l1(rec + (nxt.y & MvIdx<G>::kIdxMask));
      prefetch_l1(rec + (nxt.z & MvIdx<G>::kIdxMask));
      prefetch_l1(rec + (nxt.w & MvIdx<G>::kIdxMask));
    }
#pragma unroll
    for (int u0 = 0; u0 < 4; u0 += U) {
      double4 o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) o[u] = ld_rec(rec + (es[u0 + u] & MvIdx<G>::kIdxMask));
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const double dx = me[j].x - o[u].x, dy = me[j].y - o[u].y;
          const double e = gauss_exp2<DEG>(fma(dx, dx, dy * dy), esc);
          if (es[u0 + u] & MvIdx<G>::bit(j)) acc[j] = fma(o[u].z, e, acc[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j)
    if (t[j] >= 0) y[t[j]] = acc[j] * g.norm;
}

// The same matvec over 16-bit entries (two targets per lane): the source index is
// the current row's run start + the entry's offset; a lane moves to its next box row
// (one cell_start load) when an entry says so.  Half the list bytes of k_matvec.
template <int DEG, int MINB>
__global__ __launch_bounds__(kMvThreads, MINB) void k_matvec16(
    Geom g, long long own_off, long long ext_lo, long long n_ext, const int *__restrict__ cell_start,
    const double4 *__restrict__ rec, const int4 *__restrict__ tgt, long long nlanes,
    const int *__restrict__ chunk_len, const long long *__restrict__ chunk_off,
    const unsigned short *__restrict__ list, double *__restrict__ y, long long lane0) {
  const int lane = threadIdx.x & 31;
  const long long lt = lane0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ch = lt >> 5;
  if ((ch << 5) >= nlanes) return;  // whole warp beyond the last chunk
  const int4 tv = lt < nlanes ? tgt[lt] : make_int4(-1, -1, -1, -1);
  const int t[2] = {tv.x, tv.y};
  double2 me[2];
  double acc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double4 r = rec[own_off + (t[j] >= 0 ? t[j] : 0)];
    me[j] = make_double2(r.x, r.y);
    acc[j] = 0.0;
  }
  int row_key = tv.w;
  long long rbase = row_key >= 0 ? (long long)cell_start[row_key] - ext_lo : own_off;
  const long long last = n_ext - 1;
  const int K = chunk_len[ch];  // multiple of 4
  const uint2 *lp = reinterpret_cast<const uint2 *>(list + chunk_off[ch]) + lane;
  const double esc = g.esc;
  uint2 nxt = (K > 0) ? __ldcs(lp) : make_uint2(0, 0);
  for (int k = 0; k < K; k += 4) {
    const uint2 ev = nxt;
    if (k + 4 < K) nxt = __ldcs(lp + ((k >> 2) + 1) * 32);
    const unsigned es[4] = {ev.x & 0xffffu, ev.x >> 16, ev.y & 0xffffu, ev.y >> 16};
    double4 o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned step = (es[u] >> 11) & 7u;
      if (step) {
        row_key += (int)step * g.ncx;
        rbase = (long long)cell_start[row_key] - ext_lo;
      }
      long long idx = rbase + (long long)(es[u] & 0x7ffu);
      idx = idx < last ? idx : last;
      o[u] = ld_rec(rec + idx);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double dx = me[j].x - o[u].x, dy = me[j].y - o[u].y;
        const double e = gauss_exp2<DEG>(fma(dx, dx, dy * dy), esc);
        if (es[u] & (0x8000u >> j)) acc[j] = fma(o[u].z, e, acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
    if (t[j] >= 0) y[t[j]] = acc[j] * g.norm;
}

// ---------------------------------------------------------------------------
// Target pairing (setup): within each owned cell, greedy nearest-neighbour matching
// in sorted order (each unpaired point takes its nearest unpaired successor), then
// the cells' leftover singles paired in cell order.  Close pairs have nearly the
// same in-cutoff set, so fewer of the union's slots are masked (0.88 -> 0.91 useful
// on cfg2-like lattices, tools/: pairing study in DESIGN.md).  The pairing changes
// only which lane computes a target, never the sums (ascending-source union lists).
// ---------------------------------------------------------------------------
__global__ void k_pair_counts(Geom g, Strip st, const int *__restrict__ cell_start, int ncl, int gs,
                              long long *__restrict__ ngroups, long long *__restrict__ nsingle) {
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl > ncl) return;
  if (cl == ncl) {
    ngroups[cl] = 0;
    nsingle[cl] = 0;
    return;
  }
  const int key = (st.row_lo + cl / g.ncx) * g.ncx + cl % g.ncx;
  const int nc = cell_start[key + 1] - cell_start[key];
  ngroups[cl] = nc / gs;
  nsingle[cl] = nc % gs;
}

constexpr int kPairMax = 256;  // greedy grouping up to this cell population (else consecutive)

// Groups of gs (2 or 3) targets: each unused point in sorted order takes its gs-1
// nearest unused successors in the cell; the remaining n_c mod gs points go to the
// singles list (grouped in cell order afterwards).
__global__ void k_pair_cells(Geom g, Strip st, const int *__restrict__ cell_start, int ncl, int gs,
                             const double2 *__restrict__ xy, const long long *__restrict__ poff,
                             const long long *__restrict__ soff, int4 *__restrict__ tgt,
                             int *__restrict__ singles) {
  const int cl = blockIdx.x * blockDim.x + threadIdx.x;
  if (cl >= ncl) return;
  const int key = (st.row_lo + cl / g.ncx) * g.ncx + cl % g.ncx;
  const int s0 = cell_start[key], nc = cell_start[key + 1] - s0;
  const long long loc0 = s0 - st.own_lo, own_off = st.own_lo - st.ext_lo;
  long long q = poff[cl], sq = soff[cl];
  const int ngr = nc / gs;
  if (nc > kPairMax) {
    for (int gi = 0; gi < ngr; ++gi) {
      const int i = gi * gs;
      tgt[q++] = make_int4((int)(loc0 + i), (int)(loc0 + i + 1), gs > 2 ? (int)(loc0 + i + 2) : -1, -1);
    }
    for (int i = ngr * gs; i < nc; ++i) singles[sq++] = (int)(loc0 + i);
    return;
  }
  unsigned used[kPairMax / 32];
  for (int w = 0; w < kPairMax / 32; ++w) used[w] = 0u;
  int made = 0;
  for (int i = 0; i < nc && made < ngr; ++i) {
    if (used[i >> 5] >> (i & 31) & 1u) continue;
    used[i >> 5] |= 1u << (i & 31);
    const double2 pi = xy[own_off + loc0 + i];
    int b1 = -1, b2 = -1;
    double d1 = 0.0, d2 = 0.0;
    for (int j = i + 1; j < nc; ++j) {
      if (used[j >> 5] >> (j & 31) & 1u) continue;
      const double2 pj = xy[own_off + loc0 + j];
      const double dx = pi.x - pj.x, dy = pi.y - pj.y;
      const double d = fma(dx, dx, dy * dy);
      if (b1 < 0 || d < d1) {
        b2 = b1; d2 = d1;
        b1 = j; d1 = d;
      } else if (gs > 2 && (b2 < 0 || d < d2)) {
        b2 = j; d2 = d;
      }
    }
    used[b1 >> 5] |= 1u << (b1 & 31);
    if (gs > 2) used[b2 >> 5] |= 1u << (b2 & 31);
    tgt[q++] = make_int4((int)(loc0 + i), (int)(loc0 + b1), gs > 2 ? (int)(loc0 + b2) : -1, -1);
    ++made;
  }
  for (int i = 0; i < nc; ++i)
    if (!(used[i >> 5] >> (i & 31) & 1u)) singles[sq++] = (int)(loc0 + i);
}

__global__ void k_pair_singles(const int *__restrict__ singles, long long ns, int gs, long long first,
                               int4 *__restrict__ tgt) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gs * i >= ns) return;
  const long long b = gs * i;
  tgt[first + i] = make_int4(singles[b], b + 1 < ns ? singles[b + 1] : -1,
                             (gs > 2 && b + 2 < ns) ? singles[b + 2] : -1, -1);
}

static int pair_targets(rbf_ctx *c, int gs, cudaStream_t s, long long *lanes_out) {
  const int ncl = owned_cells(c);
  long long *np = nullptr, *ns = nullptr, *poff = nullptr, *soff = nullptr;
  RBF_TRY(dalloc(c, (void **)&np, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&ns, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&poff, sizeof(long long) * (ncl + 1), s));
  RBF_TRY(dalloc(c, (void **)&soff, sizeof(long long) * (ncl + 1), s));
  k_pair_counts<<<(ncl + 1 + 255) / 256, 256, 0, s>>>(c->g, c->s, c->cell_start, ncl, gs, np, ns);
  count_launch(1);
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, np, poff, ncl + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tb, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, np, poff, ncl + 1, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, ns, soff, ncl + 1, s));
  count_launch(4);
  long long tot[2] = {0, 0};
  RBF_CUDA_TRY(cudaMemcpyAsync(&tot[0], poff + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&tot[1], soff + ncl, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  const long long P = tot[0], S = tot[1], lanes = P + (S + gs - 1) / gs;
  int *singles = nullptr;
  RBF_TRY(dalloc(c, (void **)&c->lane_tgt, sizeof(int4) * (size_t)(lanes > 0 ? lanes : 1), s));
  RBF_TRY(dalloc(c, (void **)&singles, sizeof(int) * (size_t)(S > 0 ? S : 1), s));
  if (ncl > 0) {
    k_pair_cells<<<(ncl + 127) / 128, 128, 0, s>>>(c->g, c->s, c->cell_start, ncl, gs, c->xy_ext, poff,
                                                  soff, c->lane_tgt, singles);
    count_launch(1);
  }
  if (S > 0) {
    k_pair_singles<<<(int)(((S + gs - 1) / gs + 255) / 256), 256, 0, s>>>(singles, S, gs, P, c->lane_tgt);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  dfree(tmp, s);
  dfree(np, s);
  dfree(ns, s);
  dfree(poff, s);
  dfree(soff, s);
  dfree(singles, s);
  *lanes_out = lanes;
  return RBF_OK;
}

// Lanes sorted by union-list length (descending) inside windows of kSortWin lanes, so
// the 32 lanes of a chunk have similar lengths and the ELL padding (chunk length =
// its longest lane) shrinks; windows keep the chunks spatially compact.  Ties keep
// the original order (deterministic).  Also writes the chunk lengths.
constexpr int kSortWin = 256;
__global__ __launch_bounds__(kSortWin) void k_sort_lanes(const int *__restrict__ len,
                                                         const int4 *__restrict__ tgt_in,
                                                         long long nlanes, int4 *__restrict__ tgt_out,
                                                         int *__restrict__ chunk_len) {
  __shared__ int key[kSortWin];
  __shared__ int idx[kSortWin];
  const int t = threadIdx.x;
  const long long base = (long long)blockIdx.x * kSortWin, l = base + t;
  key[t] = l < nlanes ? len[l] : -1;
  idx[t] = t;
  __syncthreads();
  for (int size = 2; size <= kSortWin; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int p = t ^ stride;
      if (p > t) {
        // descending by key, ascending by idx on ties, within bitonic sequences
        const bool up = (t & size) == 0;
        const bool before = key[t] > key[p] || (key[t] == key[p] && idx[t] < idx[p]);
        if (before != up) {
          const int k0 = key[t], i0 = idx[t];
          key[t] = key[p];
          idx[t] = idx[p];
          key[p] = k0;
          idx[p] = i0;
        }
      }
      __syncthreads();
    }
  }
  if (l < nlanes) tgt_out[l] = tgt_in[base + idx[t]];
  if ((t & 31) == 0 && l < nlanes) chunk_len[l >> 5] = (key[t] + 3) & ~3;
}

// Interior / boundary split of the lanes (multi-rank overlap): a lane is a
// boundary lane if one of its targets lies in the kh cell rows next to a strip edge that
// has a neighbour rank (its stencil reaches the halo).  Interior lanes first (stable),
// padded with empty lanes to a multiple of the sort window, then the boundary lanes:
// chunks never mix the two, so the interior chunks can run while the halo is in flight.
// Which lane computes a target never changes its sum (union lists in stencil order).
__global__ void k_lane_class(Geom g, Strip st, int nranks, int rank, const double2 *__restrict__ xy,
                             const int4 *__restrict__ tgt, long long nlanes, int *__restrict__ inner,
                             int *__restrict__ outer) {
  const long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (l >= nlanes) return;
  const int4 v = tgt[l];
  const int t[3] = {v.x, v.y, v.z};
  const long long own_off = st.own_lo - st.ext_lo;
  bool bnd = false;
  for (int j = 0; j < 3; ++j) {
    if (t[j] < 0) continue;
    int cx = 0, cy = 0;
    target_cell(g, xy[own_off + t[j]], cx, cy);
    bnd |= (rank > 0 && cy < st.row_lo + g.kh) || (rank < nranks - 1 && cy >= st.row_hi - g.kh);
  }
  inner[l] = !bnd;
  outer[l] = bnd;
}

__global__ void k_fill_int4(int4 *__restrict__ p, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = make_int4(-1, -1, -1, -1);
}

static int split_lanes(rbf_ctx *c, cudaStream_t s, long long *lanes_io) {
  const long long L = *lanes_io;
  if (c->nranks <= 1 || L <= 0) return RBF_OK;
  ScratchGuard sg(s);
  int *fi = nullptr, *fo = nullptr, *cnt = nullptr;
  RBF_TRY(sg.alloc(c, &fi, sizeof(int) * L));
  RBF_TRY(sg.alloc(c, &fo, sizeof(int) * L));
  RBF_TRY(sg.alloc(c, &cnt, sizeof(int) * 2));
  k_lane_class<<<(int)((L + 255) / 256), 256, 0, s>>>(c->g, c->s, c->nranks, c->rank, c->xy_ext, c->lane_tgt,
                                                      L, fi, fo);
  count_launch(1);
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tb, c->lane_tgt, fi, c->lane_tgt, cnt, (int)L, s));
  void *tmp = nullptr;
  RBF_TRY(sg.alloc(c, &tmp, tb));
  // count the interior lanes first (to place the boundary block after the padding)
  int4 *scratch = nullptr;
  RBF_TRY(sg.alloc(c, &scratch, sizeof(int4) * (size_t)L));
  RBF_CUDA_TRY(cub::DeviceSelect::Flagged(tmp, tb, c->lane_tgt, fi, scratch, cnt, (int)L, s));
  int h_in = 0;
  RBF_CUDA_TRY(cudaMemcpyAsync(&h_in, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  const long long pad = (h_in + kSortWin - 1) / kSortWin * kSortWin;
  const long long L2 = pad + (L - h_in);
  int4 *out = nullptr;
  RBF_TRY(dalloc(c, (void **)&out, sizeof(int4) * (size_t)L2, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(out, scratch, sizeof(int4) * (size_t)h_in, cudaMemcpyDeviceToDevice, s));
  if (pad > h_in) {
    k_fill_int4<<<(int)((pad - h_in + 255) / 256), 256, 0, s>>>(out + h_in, pad - h_in);
    count_launch(1);
  }
  RBF_CUDA_TRY(cub::DeviceSelect::Flagged(tmp, tb, c->lane_tgt, fo, out + pad, cnt + 1, (int)L, s));
  count_launch(4);
  RBF_CUDA_TRY(cudaGetLastError());
  dfree(c->lane_tgt, s);
  c->lane_tgt = out;
  c->mv_int_chunks = pad / 32;
  *lanes_io = L2;
  return RBF_OK;
}

int build_nlist(rbf_ctx *c, cudaStream_t s) {
  const long long nl = n_loc(c), ne = n_ext(c);
  c->mv_var = (int)opt(OPT_MV_VARIANT);  // A/B switch; 0 = default
  c->mv_g = (int)opt(OPT_MV_G);
  if (c->mv_g < 1 || c->mv_g > 3) c->mv_g = 2;
  if (ne >= (1LL << (32 - c->mv_g))) c->mv_g = 1;  // source index must fit beside the mask bits
  if (ne >= (1LL << 31)) {
    set_error("rbf_setup: %lld points in one strip exceed the 31-bit neighbour-list index", ne);
    return RBF_EINVAL;
  }
  const int G = c->mv_g;
  RBF_TRY(dalloc(c, (void **)&c->rec, sizeof(double4) * (size_t)(ne > 0 ? ne : 1), s));
  if (ne > 0) {
    k_init_rec<<<(int)((ne + 255) / 256), 256, 0, s>>>(c->xy_ext, ne, c->rec);
    count_launch(1);
  }
  if (nl <= 0) return RBF_OK;
  long long lanes = (nl + G - 1) / G;
  if (G >= 2 && opt(OPT_MV_PAIR)) RBF_TRY(pair_targets(c, G, s, &lanes));
  c->mv_int_chunks = 0;
  if (c->overlap && c->lane_tgt) RBF_TRY(split_lanes(c, s, &lanes));
  c->mv_lanes = lanes;
  c->nchunks = (int)((lanes + 31) / 32);
  const int nch = c->nchunks;
  RBF_TRY(dalloc(c, (void **)&c->chunk_len, sizeof(int) * nch, s));
  RBF_TRY(dalloc(c, (void **)&c->chunk_off, sizeof(long long) * (nch + 1), s));
  const int blocks = (int)((lanes + kMvThreads - 1) / kMvThreads);
#define RBF_NLIST(MODE, W16, off, lst)                                                              \
  switch (G) {                                                                                      \
    case 1: k_nlist<MODE, 1><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, nl, \
                                                            nullptr, lanes, c->chunk_len, off, lst, nu, ll, fmt); break; \
    case 3: k_nlist<MODE, 3><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, nl, \
                                                            c->lane_tgt, lanes, c->chunk_len, off, lst, nu, ll, fmt); break; \
    default: k_nlist<MODE, 2, W16><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, nl, \
                                                             c->lane_tgt, lanes, c->chunk_len, off, lst, nu, ll, fmt); break; \
  }
  int *fmt = nullptr;  // largest row offset and row step of any entry (16-bit format check)
  RBF_TRY(dalloc(c, (void **)&fmt, sizeof(int) * 2, s));
  RBF_CUDA_TRY(cudaMemsetAsync(fmt, 0, sizeof(int) * 2, s));
  unsigned long long *nu = nullptr;
  RBF_TRY(dalloc(c, (void **)&nu, sizeof(unsigned long long), s));
  RBF_CUDA_TRY(cudaMemsetAsync(nu, 0, sizeof(unsigned long long), s));
  int *ll = nullptr;
  const bool sort_lanes = G >= 2 && c->lane_tgt && opt(OPT_MV_SORT);
  if (sort_lanes) RBF_TRY(dalloc(c, (void **)&ll, sizeof(int) * (size_t)lanes, s));
  RBF_NLIST(0, false, nullptr, nullptr);
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  if (sort_lanes) {
    int4 *sorted = nullptr;
    RBF_TRY(dalloc(c, (void **)&sorted, sizeof(int4) * (size_t)lanes, s));
    k_sort_lanes<<<(int)((lanes + kSortWin - 1) / kSortWin), kSortWin, 0, s>>>(ll, c->lane_tgt, lanes,
                                                                             sorted, c->chunk_len);
    count_launch(1);
    RBF_CUDA_TRY(cudaGetLastError());
    dfree(c->lane_tgt, s);
    c->lane_tgt = sorted;
    dfree(ll, s);
    ll = nullptr;
  }
  // offsets (in entries) = exclusive scan of 32 * len
  long long *w64 = nullptr;
  RBF_TRY(dalloc(c, (void **)&w64, sizeof(long long) * (nch + 1), s));
  RBF_CUDA_TRY(cudaMemsetAsync(w64 + nch, 0, sizeof(long long), s));
  k_len_to_entries<<<(nch + 255) / 256, 256, 0, s>>>(c->chunk_len, nch, w64);
  count_launch(1);
  size_t tb = 0;
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, w64, c->chunk_off, nch + 1, s));
  void *tmp = nullptr;
  RBF_TRY(dalloc(c, &tmp, tb, s));
  RBF_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, w64, c->chunk_off, nch + 1, s));
  count_launch(2);
  long long total = 0;
  unsigned long long hnu = 0;
  int hfmt[2] = {0, 0};
  RBF_CUDA_TRY(cudaMemcpyAsync(&total, c->chunk_off + nch, sizeof(long long), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(&hnu, nu, sizeof(hnu), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaMemcpyAsync(hfmt, fmt, sizeof(hfmt), cudaMemcpyDeviceToHost, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(fmt, s);
  fmt = nullptr;
  // 16-bit entries when every row offset fits 11 bits and every row step 3 bits
  c->mv_w16 = G == 2 && c->lane_tgt && opt(OPT_MV_INDEX16) && hfmt[0] < 2048 && hfmt[1] < 8 &&
              c->mv_var == 0;
  dfree(tmp, s);
  dfree(w64, s);
  c->nlist_entries = total;
  c->nlist_union = (long long)hnu;
  dfree(nu, s);
  RBF_TRY(dalloc(c, (void **)&c->nlist, (c->mv_w16 ? 2 : 4) * (size_t)(total > 0 ? total : 1), s));
  // variant 5 (staged sources, A/B only): one window per matvec CTA, single strip
  const bool stage = c->mv_var == 5 && G == 2 && c->lane_tgt && c->mv_int_chunks == 0 && !c->mv_w16;
  if (stage) {
    RBF_TRY(dalloc(c, (void **)&c->mv_win, sizeof(int4) * (size_t)blocks, s));
    k_mv_windows<<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, nl, c->lane_tgt, lanes,
                                               c->mv_win);
    count_launch(1);
    RBF_CUDA_TRY(cudaGetLastError());
  }
  if (c->mv_w16) {
    RBF_NLIST(1, true, c->chunk_off, c->nlist);
  } else if (stage) {
    k_nlist<1, 2, false, true><<<blocks, kMvThreads, 0, s>>>(c->g, c->s, c->xy_ext, c->cell_start, nl, c->lane_tgt, lanes,
                                               c->chunk_len, c->chunk_off, c->nlist, nu, ll, fmt, c->mv_win);
  } else {
    RBF_NLIST(1, false, c->chunk_off, c->nlist);
  }
#undef RBF_NLIST
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_pack_w(const rbf_ctx *c, const double *w_ext, cudaStream_t s) {
  return launch_pack_range(c, w_ext, n_ext(c), 0, s);
}

// w slot of records [off, off + cnt) of the ext range from src[0 .. cnt)
int launch_pack_range(const rbf_ctx *c, const double *src, long long cnt, long long off, cudaStream_t s) {
  if (cnt > 0) {
    k_pack_w<<<(int)((cnt + 255) / 256), 256, 0, s>>>(src, cnt, c->rec + off);
    count_launch(1);
  }
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

int launch_matvec(const rbf_ctx *c, const double *w_ext, double *y_loc, cudaStream_t s, bool prepacked,
                  int part) {
  const long long nl = n_loc(c);
  if (nl <= 0) return RBF_OK;
  if (!prepacked) RBF_TRY(launch_pack_w(c, w_ext, s));
  const int G = c->mv_g;
  // part 0: every lane; 1: the interior chunks; 2: the boundary chunks (split_lanes)
  const long long split = 32LL * c->mv_int_chunks < c->mv_lanes ? 32LL * c->mv_int_chunks : c->mv_lanes;
  const long long lane0 = part == 2 ? split : 0;
  const long long lane1 = part == 1 ? split : c->mv_lanes;
  const long long lanes = c->mv_lanes;
  if (lane1 <= lane0) return RBF_OK;
  const int blocks = (int)((lane1 - lane0 + kMvThreads - 1) / kMvThreads);
  const long long own_off = c->s.own_lo - c->s.ext_lo;
#define RBF_MV(GG, DEG, U, MB, ...)                                                            \
  k_matvec<GG, DEG, U, MB, ##__VA_ARGS__><<<blocks, kMvThreads, 0, s>>>(c->g, nl, own_off, c->rec, \
                                                     GG >= 2 ? c->lane_tgt : nullptr, lane1, c->chunk_len,  \
                                                     c->chunk_off, reinterpret_cast<const unsigned *>(c->nlist), y_loc, lane0)
  // Measured alternatives: profiles/r01_matvec_variants_cfg2.txt (2 gathers in flight,
  // 2/4/5 CTAs per SM, L1 prefetch of the next group's records, G = 1 or 3, the
  // degree-10 exp: none faster than the default).
  (void)lanes;
  if (c->mv_win) {
    const size_t dyn = sizeof(double4) * kMvStageMax;
    RBF_TRY(ensure_dyn_smem((const void *)k_matvec_st<kExpDeg, 2>, dyn));
    k_matvec_st<kExpDeg, 2><<<blocks, kMvThreads, dyn, s>>>(c->g, c->s, nl, own_off, c->rec, c->cell_start,
                                                           c->mv_win, c->lane_tgt, lane1, c->chunk_len,
                                                           c->chunk_off, reinterpret_cast<const unsigned *>(c->nlist),
                                                           y_loc);
  } else if (c->mv_w16) {
    k_matvec16<kExpDeg, 3><<<blocks, kMvThreads, 0, s>>>(
        c->g, own_off, c->s.ext_lo, n_ext(c), c->cell_start, c->rec, c->lane_tgt, lane1, c->chunk_len,
        c->chunk_off, reinterpret_cast<const unsigned short *>(c->nlist), y_loc, lane0);
  } else if (G == 1) RBF_MV(1, kExpDeg, 4, 1);
  else if (G == 3) RBF_MV(3, kExpDeg, 4, 1);
  else if (c->mv_var == 1) RBF_MV(2, 9, 4, 1);
  else if (c->mv_var == 2) RBF_MV(2, 10, 4, 3);  // degree-10 exp (1.5e-16), 3 CTAs/SM
  else if (c->mv_var == 3) RBF_MV(2, 10, 4, 4);  // 62 registers, 4 CTAs/SM
  else if (c->mv_var == 4) RBF_MV(2, 10, 4, 1);  // 84 registers, 2 CTAs/SM
  else RBF_MV(2, kExpDeg, 4, 3);  // default: degree-9 exp (3.9e-16 = 3.5 ulp), 3 CTAs/SM (fastest)
#undef RBF_MV
  count_launch(1);
  RBF_CUDA_TRY(cudaGetLastError());
  return RBF_OK;
}

}  // namespace rbf
