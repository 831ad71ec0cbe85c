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


__device__ __forceinline__ double rsqrt_fast(double a) {
  // fp32 hardware estimate, then two Newton steps in fp64: y <- y (3 - a y^2) / 2
  double y = (double)rsqrtf((float)a);
  double h = a * y;
  double r = fma(-h, y, 1.0);
  y = fma(0.5 * y, r, y);
  h = a * y;
  r = fma(-h, y, 1.0);
  return fma(0.5 * y, r, y);
}

// Restructured: the next pivot row updates its diagonal lane-locally (the pivot
// chain is shfl + rsqrt + mul + fma per step), off-diagonal updates in parallel.
__device__ long long g_stamp[4];
__device__ __forceinline__ bool diag_factor2(double *sm, double *rdiag, int j, int lane) {
  long long t0 = clock64();
  double *D = sm + toff(j, j);
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = (lane < 8) ? D[swz(lane, c)] : (c == 0 ? 1.0 : 0.0);
  bool bad = false;
  double rinv = 1.0;
  double dcur = a[0];  // this lane's running diagonal candidate (meaningful for lane = next pivot)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double akk = __shfl_sync(0xffffffffu, (lane == k) ? dcur : a[k], k);
    bad |= !(akk > 0.0);
    const double il = rsqrt(akk);
    const double lik = (lane == k) ? akk * il : a[k] * il;  // row `lane`, column k of L
    if (lane == k) rinv = il;
    a[k] = (lane >= k) ? lik : 0.0;
    if (k + 1 < 8) dcur = fma(-lik, lik, a[k + 1]);  // next pivot (lane k+1), lane-local
#pragma unroll
    for (int jj = k + 1; jj < 8; ++jj) {
      const double ljk = __shfl_sync(0xffffffffu, lik, jj);
      if (lane >= jj) a[jj] = fma(-lik, ljk, a[jj]);
    }
    if (k + 1 < 8 && lane == k + 1) dcur = a[k + 1];  // identical value, keeps a[] consistent
  }
  long long t1 = clock64() + (long long)(a[7] * 0.0);
  double x[8];
  double Lrow[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int m = 0; m < i; ++m) Lrow[i][m] = __shfl_sync(0xffffffffu, a[m], i);
  double rd[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rd[i] = __shfl_sync(0xffffffffu, rinv, i);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double sacc = (lane == i) ? 1.0 : 0.0;
#pragma unroll
    for (int m = 0; m < i; ++m) sacc = fma(-Lrow[i][m], x[m], sacc);
    x[i] = sacc * rd[i];
  }
  long long t2 = clock64() + (long long)(x[7] * 0.0);
  if (lane < 8) {
#pragma unroll
    for (int c = 0; c < 8; ++c) D[swz(lane, c)] = (c <= lane) ? a[c] : x[c];
    rdiag[j * 8 + lane] = rinv;
  }
  if (lane == 0) { g_stamp[0] += t1 - t0; g_stamp[1] += t2 - t1; g_stamp[2] += clock64() - t2; }
  return bad;
}

template <int V>
__global__ void lat(double *out, long long *cyc, int reps) {
  double x = 2.0 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) x = 1.0 + (V == 0 ? rsqrt(x) : rsqrt_fast(x));
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[2 + V] = (t1 - t0) / reps; out[2 + V] = x; }
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
    bad |= V == 0 ? diag_factor(sm, rdiag, 0, lane) : (V == 1 ? diag_factor_fast(sm, rdiag, 0, lane) : diag_factor2(sm, rdiag, 0, lane));
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
  }
  if (lane == 0) { cyc[V] = tot / reps; double cs = 0; for (int e = 0; e < 64; ++e) cs += sm[e] * (e + 1); out[V] = cs + rdiag[3] + bad; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  lat<0><<<1, 32>>>(o, c, 1000); lat<1><<<1, 32>>>(o, c, 1000);
  long long hl[4]; double hol[4];
  cudaMemcpy(hl, c, 32, cudaMemcpyDeviceToHost); cudaMemcpy(hol, o, 32, cudaMemcpyDeviceToHost);
  printf("rsqrt(double) chain latency %lld cyc (x=%.17g), rsqrt_fast %lld cyc (x=%.17g)\n", hl[2], hol[2], hl[3], hol[3]);
  k<0><<<1, 32>>>(o, c, 100); k<1><<<1, 32>>>(o, c, 100); k<2><<<1, 32>>>(o, c, 100);
  long long h[3]; double ho[3];
  cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost); cudaMemcpy(ho, o, 24, cudaMemcpyDeviceToHost);
  long long st[4]; cudaMemcpyFromSymbol(st, g_stamp, 32);
  printf("diag_factor2 phases (per call): factor %lld inverse %lld store %lld\n", st[0] / 100, st[1] / 100, st[2] / 100);
  printf("diag_factor %lld cyc (check %.17g)\ndiag_factor_fast %lld cyc (check %.17g)\ndiag_factor2 %lld cyc (check %.17g)\n", h[0], ho[0], h[1], ho[1], h[2], ho[2]);
}
