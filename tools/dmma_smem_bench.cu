// Micro-benchmark: DMMA throughput of the left-looking accumulation pattern of
// k_rasm_setup_tc (operands from the swizzled shared-memory tiles) vs register
// operands; extracted helpers, design evidence only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ int toff(int it, int jt) { return ((it * (it + 1)) / 2 + jt) * 64; }
__device__ __forceinline__ int swz(int r, int c) { return r * 8 + (c ^ (((r >> 1) & 1) << 2)); }

// D += A * B, one 8x8x4 fp64 tensor-core MMA (DMMA on sm_100a).
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Fragment offsets inside a swizzled tile (lane l): A[m][k] = X[m][k] and
// B[k][n] = X[n][k] use "rowk"; B[k][n] = X[k][n] and A[m][k] = X[k][m] use "colk".
__device__ __forceinline__ int frag_rowk(int lane, int h) { return swz(lane >> 2, 4 * h + (lane & 3)); }
__device__ __forceinline__ int frag_colk(int lane, int h) { return swz(4 * h + (lane & 3), lane >> 2); }
__device__ __forceinline__ int frag_acc(int lane) { return swz(lane >> 2, 2 * (lane & 3)); }

struct AccSet {
  double a0, a1, b0, b1;  // two independent DMMA chains (even / odd kt)
  double v0, v1;          // the tile's A_c entries at this lane's accumulator positions
  __device__ __forceinline__ void zero() { a0 = a1 = b0 = b1 = 0.0; }
};

// acc += sum_{kt in [k0, k1)} L(it, kt) L(jt, kt)^T
__device__ __forceinline__ void acc_range_(AccSet &A, const double *sm, int it, int jt, int k0,
                                          int k1, int lane) {
  const double *Li = sm + toff(it, 0), *Lj = sm + toff(jt, 0);
  const int f0 = frag_rowk(lane, 0), f1 = frag_rowk(lane, 1);
  int kt = k0;
  for (; kt + 1 < k1; kt += 2) {
    dmma(A.a0, A.a1, Li[kt * 64 + f0], Lj[kt * 64 + f0]);
    dmma(A.b0, A.b1, Li[(kt + 1) * 64 + f0], Lj[(kt + 1) * 64 + f0]);
    dmma(A.a0, A.a1, Li[kt * 64 + f1], Lj[kt * 64 + f1]);
    dmma(A.b0, A.b1, Li[(kt + 1) * 64 + f1], Lj[(kt + 1) * 64 + f1]);
  }
  if (kt < k1) {
    dmma(A.a0, A.a1, Li[kt * 64 + f0], Lj[kt * 64 + f0]);
    dmma(A.a0, A.a1, Li[kt * 64 + f1], Lj[kt * 64 + f1]);
  }
}

// tile(it, jt) -= acc, in place (accumulator layout)
__device__ __forceinline__ void acc_finish_rmw(const AccSet &A, double *sm, int it, int jt, int lane) {
  double2 *cp = reinterpret_cast<double2 *>(sm + toff(it, jt) + frag_acc(lane));
  double2 cv = *cp;
  cv.x -= A.a0 + A.b0;
  cv.y -= A.a1 + A.b1;
  *cp = cv;
}


template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double *out, int reps, long long *cyc) {
  extern __shared__ double sm[];
  const int T = 29, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < T * (T + 1) / 2 * 64; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  AccSet A;
  A.zero();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const int it = 1 + (warp + r) % 28, jt = it;  // row tiles, 28 kt terms max
    if (MODE == 0) {
      acc_range_(A, sm, it, jt > 14 ? 14 : jt, 0, 14, lane);
    } else if (MODE == 1) {  // register operands, 2 chains
      const double a = sm[lane], b = sm[lane + 32];
      for (int kt = 0; kt < 14; ++kt) {
        dmma(A.a0, A.a1, a, b); dmma(A.b0, A.b1, a, b);
        dmma(A.a0, A.a1, b, a); dmma(A.b0, A.b1, b, a);
      }
    } else {  // register operands, 4 chains
      const double a = sm[lane], b = sm[lane + 32];
      double c0 = 0, c1 = 0, d0 = 0, d1 = 0;
      for (int kt = 0; kt < 14; ++kt) {
        dmma(A.a0, A.a1, a, b); dmma(A.b0, A.b1, a, b);
        dmma(c0, c1, b, a); dmma(d0, d1, b, a);
      }
      A.a0 += c0 + d0; A.a1 += c1 + d1;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = A.a0 + A.a1 + A.b0 + A.b1;
}
int main() {
  const int smem = 29 * 30 / 2 * 64 * 8;
  double *out; long long *cyc;
  cudaMalloc(&out, 148 * 512 * 8); cudaMalloc(&cyc, 148 * 8);
  for (int mode = 0; mode < 3; ++mode) {
    const void *fn = mode == 0 ? (const void *)k<0> : mode == 1 ? (const void *)k<1> : (const void *)k<2>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int reps = 200;
    void *args[] = {&out, &reps, &cyc};
    cudaLaunchKernel(fn, 148, 512, args, smem, 0);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < 148; ++i) mean += h[i]; mean /= 148;
    const double dmma = 16.0 * reps * 28;  // warps x reps x (14 kt x 2 DMMA)
    printf("mode %d (%s): %.0f cycles, %.3f DMMA/cycle/SM (peak 0.25) (%s)\n", mode,
           mode == 0 ? "smem operands, acc_range" : mode == 1 ? "register operands, 2 chains" : "register operands, 4 chains",
           mean, dmma / mean, cudaGetErrorString(cudaGetLastError()));
  }
}
