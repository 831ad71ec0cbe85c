// Microbenchmark: fp64 DMMA.8x8x4 (mma.sync m8n8k4 f64) latency and per-warp throughput
// on sm_100a -- design evidence for the RASM setup kernel's chains.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void chains(double *out, long long *cyc, int reps) {
  double d0[CH], d1[CH];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
#pragma unroll
  for (int c = 0; c < CH; ++c) d0[c] = d1[c] = c;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d0[c], d1[c], a, b);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d0[c] + d1[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[CH] = (t1 - t0);
}
// smem fragment load -> DMMA -> store -> reload chain (the W-phase chain step pattern)
__global__ void ldchain(double *out, long long *cyc, int reps) {
  __shared__ double sm[1024];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < 1024; i += 32) sm[i] = 1e-3 * i;
  __syncwarp();
  double d0 = 0, d1 = 0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    double a = sm[(lane + i) & 511], b = sm[512 + ((lane * 3 + i) & 511)];
    dmma(d0, d1, a, b);
    sm[(lane * 2 + i) & 511] = d0;
    __syncwarp();
  }
  long long t1 = clock64();
  out[threadIdx.x] = d0 + d1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *o; long long *c;
  cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 64 * 8);
  const int reps = 1000;
  long long h[64];
  chains<1><<<1, 32>>>(o, c, reps); chains<2><<<1, 32>>>(o, c, reps); chains<4><<<1, 32>>>(o, c, reps);
  chains<8><<<1, 32>>>(o, c, reps);
  ldchain<<<1, 32>>>(o, c, reps);
  cudaMemcpy(h, c, 64 * 8, cudaMemcpyDeviceToHost);
  printf("one warp: dependent DMMA chain %.1f cyc/DMMA; 2 chains %.1f; 4 chains %.1f; 8 chains %.1f cyc per DMMA\n",
         h[1] / (double)reps, h[2] / (2.0 * reps), h[4] / (4.0 * reps), h[8] / (8.0 * reps));
  printf("LDS -> DMMA -> STS chain step: %.1f cyc\n", h[0] / (double)reps);
  // 4 warps on one SMSP (warps 0,4,8,12 of a 16-warp CTA run; only time warp 0)
  chains<4><<<1, 512>>>(o, c, reps);
  cudaMemcpy(h, c, 64 * 8, cudaMemcpyDeviceToHost);
  printf("16 warps x 4 chains: warp 0 %.1f cyc per own DMMA (SM rate %.3f DMMA/cyc)\n", h[4] / (4.0 * reps),
         16 * 4.0 * reps / h[4]);
  return 0;
}
