// Do DMMA (fp64 tensor) and DFMA (fp64 CUDA-core) work share an SM's issue / pipes?
// Warps [0, nd) run 4 independent DMMA.8x8x4 chains, warps [nd, nd + nf) run 8 DFMA
// chains; one CTA per SM.  Prints the rate of each kind (TF/s) for several mixes.
// Design evidence only: nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void mix(int nd, int nf, int iters, double *out, long long *cyc) {
  const int warp = threadIdx.x >> 5;
  double r = 0.0;
  long long t0 = clock64();
  if (warp < nd) {
    double c[4][2] = {};
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], a, b);
    }
    r = c[0][0] + c[1][0] + c[2][0] + c[3][1];
  } else if (warp < nd + nf) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = 1.0 + u * 1e-3 + threadIdx.x * 1e-9;
    const double m = 0.999999, ad = 1e-7;
    for (int i = 0; i < iters * 2; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], m, ad);
    }
    r = x[0] + x[1] + x[2] + x[3] + x[4] + x[5] + x[6] + x[7];
  }
  long long t1 = clock64();
  if (r == 12345.678) out[0] = r;
  if (threadIdx.x == 0) cyc[2 * blockIdx.x] = t1 - t0;
  if (threadIdx.x == 32 * nd && nf > 0) cyc[2 * blockIdx.x + 1] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o;
  long long *cyc;
  cudaMalloc(&o, 8);
  cudaMalloc(&cyc, sizeof(long long) * 2 * sms);
  const int iters = 20000;
  int cases[][2] = {{16, 0}, {0, 16}, {8, 8}, {16, 16}, {12, 4}, {16, 8}, {4, 12}};
  for (auto &cs : cases) {
    const int nd = cs[0], nf = cs[1];
    mix<<<sms, 32 * (nd + nf)>>>(nd, nf, 10, o, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mix<<<sms, 32 * (nd + nf)>>>(nd, nf, iters, o, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_fl = (double)sms * nd * iters * 4 * 512.0;       // 512 flops per DMMA per warp
    const double dfma_fl = (double)sms * nf * 32 * iters * 2 * 8 * 2.0;  // 2 flops per lane FMA
    long long h[2] = {0, 0};
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    // per-group rates from the group's own duration on SM 0 (clock 1.965 GHz)
    const double td = nd ? h[0] / 1.965e6 : 0.0, tf = nf ? h[1] / 1.965e6 : 0.0;  // ms
    printf("DMMA warps %2d (%.3f ms), DFMA warps %2d (%.3f ms), kernel %.3f ms: DMMA %.2f TF/s, DFMA %.2f TF/s, "
           "sum %.2f TF/s\n", nd, td, nf, tf, ms, nd ? dmma_fl / td / 1e9 : 0.0, nf ? dfma_fl / tf / 1e9 : 0.0,
           (nd ? dmma_fl / td / 1e9 : 0.0) + (nf ? dfma_fl / tf / 1e9 : 0.0));
  }
  return 0;
}
