// Microbenchmarks for design decisions (not part of the product):
//  1. DMMA m8n8k4 f64 tensor-core throughput on sm_100a vs DFMA.
//  2. table-driven exp(x), x in [-18.5, 0]: max ulp error vs correctly-rounded-ish
//     reference (long double on host is not available on device; compare to exp())
//     and throughput vs CUDA exp().
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double *out, int iters) {
  double c0[CH], c1[CH];
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int i = 0; i < CH; ++i) { c0[i] = i; c1[i] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c0[i], c1[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c0[i] + c1[i];
  if (s == 1.2345) out[0] = s;
}

// latency: one warp, dependent DMMA chain; and dependent DFMA chain
__global__ void k_lat(double *out, long long *cyc, int iters) {
  double c0 = 1.0, c1 = 0.5, a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(c0, c1, a, b);
  long long t1 = clock64();
  double x = c0;
  for (int i = 0; i < iters; ++i) x = fma(x, b, a);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  if (c0 + c1 + x == 1.2345) out[0] = 1;
}

__constant__ double c_tab[64];

// exp(x) = 2^(k/64) (1 + p(r)),  k = round(64 x / ln2), r = x - k ln2/64
__device__ __forceinline__ double exp_tab(double x, const double *tab) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double inv = 92.33248261689366;     // 64 / ln2
  const double l_hi = 0.010830424696223417; // ln2/64 high part
  const double l_lo = 2.572804622327669e-14;
  double t = fma(x, inv, magic);
  double kd = t - magic;
  int k = __double2loint(t);
  double r = fma(kd, -l_hi, x);
  r = fma(kd, -l_lo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = r * p;
  double T = tab[k & 63];
  double e = fma(T, p, T);
  int hi = __double2hiint(e) + ((k >> 6) << 20);
  return __hiloint2double(hi, __double2loint(e));
}

__global__ void k_exp_acc(int n, double *maxulp, double *worst_x) {
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = c_tab[threadIdx.x];
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = -18.5 * ((double)i / (double)n) - 1e-300 * 0;
  // also perturb to hit non-grid points
  x = x * (1.0 + 1e-13 * (i & 7));
  double a = exp_tab(x, tab);
  double b = exp(x);
  double ulp = fabs(a - b) / (nextafter(b, 1e300) - b);
  unsigned long long u = __double_as_longlong(ulp);
  atomicMax((unsigned long long *)maxulp, u);
  (void)worst_x;
}

__global__ void k_exp_tput(double *out, int iters, int use_tab) {
  __shared__ double tab[64];
  if (threadIdx.x < 64) tab[threadIdx.x] = c_tab[threadIdx.x];
  __syncthreads();
  double acc = 0, x = -1e-3 * (threadIdx.x & 31);
  double acc2 = 0, x2 = -2e-3 * (threadIdx.x & 31);
  for (int i = 0; i < iters; ++i) {
    if (use_tab) { acc += exp_tab(x, tab); acc2 += exp_tab(x2, tab); }
    else { acc += exp(x); acc2 += exp(x2); }
    x -= 0.37; if (x < -18.0) x += 18.0;
    x2 -= 0.41; if (x2 < -18.0) x2 += 18.0;
  }
  if (acc + acc2 == 12345.678) out[0] = acc;
}

int main() {
  double *d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  // DMMA throughput
  const int iters = 2048, threads = 256, blocks = sms * 4;
  float ms = 0;
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_dmma<8><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8.0 * iters * (threads / 32) * blocks;  // 256 FMA per warp-mma
    if (rep) best = fmax(best, fl / (ms * 1e-3) / 1e12);
  }
  printf("{\"dmma_tflops\": %.3f", best);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf(", \"dmma_err\": \"%s\"", cudaGetErrorString(err));
  long long *dc; cudaMalloc(&dc, 16);
  k_lat<<<1, 32>>>(d, dc, 1000);
  long long hc[2]; cudaMemcpy(hc, dc, 16, cudaMemcpyDeviceToHost);
  printf(", \"dmma_latency_cyc\": %.1f, \"dfma_latency_cyc\": %.1f", hc[0] / 1000.0, hc[1] / 1000.0);
  // exp table
  double h[64];
  for (int j = 0; j < 64; ++j) h[j] = exp2((double)j / 64.0);
  cudaMemcpyToSymbol(c_tab, h, sizeof h);
  cudaMemset(d, 0, 64);
  int n = 1 << 24;
  k_exp_acc<<<(n + 255) / 256, 256>>>(n, d, d + 1);
  double maxulp; cudaMemcpy(&maxulp, d, 8, cudaMemcpyDeviceToHost);
  printf(", \"exp_tab_max_ulp_vs_cuda_exp\": %.3f", maxulp);
  for (int use = 0; use < 2; ++use) {
    k_exp_tput<<<sms * 8, 256>>>(d, 1024, use);
    cudaEventRecord(e0);
    k_exp_tput<<<sms * 8, 256>>>(d, 4096, use);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double g = 2.0 * 4096.0 * 256 * sms * 8 / (ms * 1e-3) / 1e9;
    printf(", \"%s_gexp_s\": %.1f", use ? "exp_tab" : "cuda_exp", g);
  }
  printf("}\n");
  return 0;
}
