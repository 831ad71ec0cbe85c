// Microbenchmark of the two 8x8 diagonal-tile factorizations of k_rasm_setup_tc
// (extracted from paper_0909_5413_b200/csrc/rasm.cu by a script); design evidence only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int toff(int it, int jt) { return ((it * (it + 1)) / 2 + jt) * 64; }
__device__ __forceinline__ int swz(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) << 2)); }

// 8x8 Cholesky of the diagonal tile j in place (lanes 0..7 = rows) plus its inverse:
// lower part = L_d, upper part (r < c) = Linv[c][r], rdiag = 1 / diag(L_d).
__device__ __forceinline__ bool diag_factor(double *sm, double *rdiag, int j, int lane) {
  double *D = sm + toff(j, j);
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = (lane < 8) ? D[swz(lane, c)] : 1.0;
  bool bad = false;
  double rinv = 1.0;  // 1 / L[lane][lane]
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double akk = __shfl_sync(0xffffffffu, a[k], k);
    bad |= !(akk > 0.0);
    const double il = rsqrt(akk);  // 1 / l_kk
    const double lik = (lane == k) ? akk * il : a[k] * il;
    if (lane == k) rinv = il;
    a[k] = (lane >= k) ? lik : 0.0;
#pragma unroll
    for (int jj = k + 1; jj < 8; ++jj) {
      const double ljk = __shfl_sync(0xffffffffu, lik, jj);
      if (lane >= jj) a[jj] = fma(-lik, ljk, a[jj]);
    }
  }
  // Linv column `lane`: x = L^-1 e_lane by forward substitution
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double sacc = (lane == i) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) sacc = fma(-__shfl_sync(0xffffffffu, a[k], i), x[k], sacc);
    x[i] = sacc * __shfl_sync(0xffffffffu, rinv, i);
  }
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) D[swz(lane, c)] = (c <= lane) ? a[c] : x[c];
    rdiag[j * 8 + lane] = rinv;
  }
  return bad;
}

__device__ __forceinline__ bool diag_factor_fast(double *sm, double *rdiag, int j, int lane) {
  double *D = sm + toff(j, j);
  double a[36];  // packed lower triangle, a[r(r+1)/2 + c]
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) a[r * (r + 1) / 2 + c] = D[swz(r, c)];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double akk = a[k * (k + 1) / 2 + k];
    bad |= !(akk > 0.0);
    const double il = rsqrt(akk);
    if (lane == 0) rdiag[j * 8 + k] = il;
    a[k * (k + 1) / 2 + k] = akk * il;
#pragma unroll
    for (int i = k + 1; i < 8; ++i) a[i * (i + 1) / 2 + k] *= il;
#pragma unroll
    for (int jj = k + 1; jj < 8; ++jj)
#pragma unroll
      for (int i = jj; i < 8; ++i)
        a[i * (i + 1) / 2 + jj] = fma(-a[i * (i + 1) / 2 + k], a[jj * (jj + 1) / 2 + k], a[i * (i + 1) / 2 + jj]);
  }
  __syncwarp();  // every lane has read the tile before it is overwritten
#pragma unroll
  for (int r = 0; r < 8; ++r)  // lower part = L, row r written by lane r
    if (lane == r) {
#pragma unroll
      for (int c = 0; c <= r; ++c) D[swz(r, c)] = a[r * (r + 1) / 2 + c];
    }
  __syncwarp();
  // column `lane` of L^-1 by forward substitution (L read back, broadcast), stored
  // transposed in the upper part: D[lane][i] = Linv[i][lane], i > lane
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double sacc = (lane == i) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < i; ++m) sacc = fma(-D[swz(i, m)], x[m], sacc);
    x[i] = sacc * rdiag[j * 8 + i];
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i > lane) D[swz(lane, i)] = x[i];
  }
  return bad;
}


template <int V>
__global__ void k(double *out, long long *cyc, int reps) {
  __shared__ double sm[64 * 2];
  __shared__ double rdiag[16];
  const int lane = threadIdx.x & 31;
  long long tot = 0;
  bool bad = false;
  for (int r = 0; r < reps; ++r) {
    // SPD tile: diag dominant
    for (int e = lane; e < 64; e += 32) { int i = e / 8, c = e % 8; sm[swz(i, c)] = (i == c) ? 10.0 + r : 1.0 / (1 + i + c); }
    __syncwarp();
    long long t0 = clock64();
    bad |= V == 0 ? diag_factor(sm, rdiag, 0, lane) : diag_factor_fast(sm, rdiag, 0, lane);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
  }
  if (lane == 0) { cyc[V] = tot / reps; out[V] = sm[swz(7, 7)] + sm[swz(1, 6)] + rdiag[3] + bad; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 16); cudaMalloc(&c, 16);
  k<0><<<1, 32>>>(o, c, 100); k<1><<<1, 32>>>(o, c, 100);
  long long h[2]; double ho[2];
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 16, cudaMemcpyDeviceToHost);
  printf("diag_factor %lld cyc (check %.15g), diag_factor_fast %lld cyc (check %.15g)\n", h[0], ho[0], h[1], ho[1]);
}
