// FP64 peak microbenchmark (stage 0 of SURVEY.md §7): independent DFMA chains
// per thread, full chip, timed with CUDA events.  Also times CUDA's exp(double)
// throughput for context.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
__global__ void exp_kernel(double *out, int iters, double scale) {
  double acc = 0, x = -1e-3 * (threadIdx.x & 31);
  for (int i = 0; i < iters; ++i) {
    acc += exp(x);
    x -= scale;
    if (x < -18.0) x += 18.0;
  }
  if (acc == 12345.678) out[0] = acc;
}
int main() {
  double *d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  double best = 0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best) best = tf;
  }
  // sustained: 3 s of back-to-back launches
  cudaEventRecord(e0);
  int nl = 0; float msum = 0;
  while (msum < 3000) {
    for (int k = 0; k < 20; ++k) dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    nl += 20; cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&msum, e0, e1);
  }
  double sus = 2.0 * 8 * iters * (double)threads * blocks * nl / (msum * 1e-3) / 1e12;
  float ms;
  const int eiters = 4096;
  cudaEventRecord(e0);
  exp_kernel<<<blocks, threads>>>(d, eiters, 0.37);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventRecord(e0);
  exp_kernel<<<blocks, threads>>>(d, eiters, 0.37);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double gexp = (double)eiters * threads * blocks / (ms * 1e-3) / 1e9;
  printf("{\"fp64_dfma_tflops_burst\": %.3f, \"fp64_dfma_tflops_sustained\": %.3f, \"cuda_exp_gexps\": %.2f, \"sms\": %d, \"clock_khz_attr\": %d}\n",
         best, sus, gexp, sms, clk);
  return 0;
}
