// Grid-barrier latency on B200 (design evidence for the fused Arnoldi kernel):
// a cooperative launch of G CTAs x 1024 threads runs R barrier rounds, each round =
// block reduction + partial store + grid barrier + every CTA reading all partials.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(double *part, unsigned *bar, double *out, int rounds) {
  __shared__ double sh[32];
  __shared__ double hsh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned G = gridDim.x;
  double x = threadIdx.x * 1e-3 + blockIdx.x;
  for (int r = 0; r < rounds; ++r) {
    double v = x;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
      double t = sh[lane];
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) part[(r & 1) * G + blockIdx.x] = t;
      if (MODE == 2) {
        // nothing here: cg sync below for all threads
      } else if (MODE == 3) {
        // per-CTA flags: publish (partial, round), then wait until every CTA's flag shows this round
        if (lane == 0) {
          __threadfence();
          ((volatile unsigned *)bar)[2 + blockIdx.x] = r + 1;
        }
        for (unsigned b = lane; b < G; b += 32)
          while (((volatile unsigned *)bar)[2 + b] < (unsigned)(r + 1)) {}
        __threadfence();
      } else if (lane == 0) {
        volatile unsigned *vgen = bar + 1;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == G - 1) {
          atomicExch(bar, 0u);
          __threadfence();
          atomicAdd(bar + 1, 1u);
        } else {
          if (MODE == 0) while (*vgen == gen) __nanosleep(20);
          else while (*vgen == gen) {}
        }
        __threadfence();
      }
    }
    if (MODE == 2) cg::this_grid().sync();
    if (warp == 0) {
      __syncwarp();
      double hs = 0.0;
      for (unsigned b = lane; b < G; b += 32) hs += ((volatile double *)part)[(r & 1) * G + b];
      for (int o = 16; o > 0; o >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
      if (lane == 0) hsh = hs;
    }
    __syncthreads();
    x += hsh * 1e-30;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = x;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out; unsigned *bar;
  cudaMalloc(&part, 2 * 1024 * sizeof(double)); cudaMalloc(&out, 8); cudaMalloc(&bar, (2 + 1024) * sizeof(unsigned));
  cudaMemset(bar, 0, 8);
  for (int mode = 0; mode < 4; ++mode)
    for (int G : {16, 32, 74, 148}) {
      int rounds = 2000;
      void *args[] = {&part, &bar, &out, &rounds};
      const void *fn = mode == 0 ? (const void *)k<0> : mode == 1 ? (const void *)k<1> : mode == 2 ? (const void *)k<2> : (const void *)k<3>;
      cudaMemset(bar, 0, (2 + 1024) * sizeof(unsigned));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel(fn, G, 1024, args, 0, 0);
      cudaMemset(bar, 0, (2 + 1024) * sizeof(unsigned));
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchCooperativeKernel(fn, G, 1024, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s) G=%d: %.2f us per round (%s)\n", mode, mode == 0 ? "atomic+nanosleep" : mode == 1 ? "atomic spin" : mode == 2 ? "cg grid.sync" : "per-CTA flags",
             G, ms * 1e3 / rounds, cudaGetErrorString(err));
    }
}
