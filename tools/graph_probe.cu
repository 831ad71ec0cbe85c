#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void coop_step(unsigned *cnt, double *acc, cudaGraphConditionalHandle h, int limit) {
  cg::grid_group g = cg::this_grid();
  if (threadIdx.x == 0) atomicAdd((unsigned long long *)acc, 0ULL);
  g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned c = ++cnt[0];
    acc[1] += c;
    cudaGraphSetConditional(h, c < (unsigned)limit ? 1u : 0u);
  }
}
__global__ void init(unsigned *cnt, double *acc) { cnt[0] = 0; acc[1] = 0; }
int main() {
  unsigned *cnt; double *acc;
  cudaMalloc(&cnt, 8); cudaMalloc(&acc, 16);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  printf("handle %s\n", cudaGetErrorString(e));
  // init node via capture
  cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
  init<<<1, 1, 0, s>>>(cnt, acc);
  e = cudaStreamEndCapture(s, &g);
  printf("capture init %s\n", cudaGetErrorString(e));
  cudaGraphNode_t leaf; size_t nn = 1; cudaGraphGetNodes(g, &leaf, &nn);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  e = cudaGraphAddNode(&cnode, g, &leaf, 1, &cp);
  printf("add cond %s\n", cudaGetErrorString(e));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
  printf("begin body %s\n", cudaGetErrorString(e));
  int limit = 1000;
  void *args[] = {&cnt, &acc, &h, &limit};
  e = cudaLaunchCooperativeKernel((const void *)coop_step, 148, 256, args, 0, s);
  printf("coop launch in capture %s\n", cudaGetErrorString(e));
  e = cudaStreamEndCapture(s, &body);
  printf("end body %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  e = cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned hc; double ha[2];
  cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost); cudaMemcpy(ha, acc, 16, cudaMemcpyDeviceToHost);
  printf("launch %s sync %s count %u sum %.0f (expect %d, %.0f) time %.3f ms -> %.2f us/iter\n", cudaGetErrorString(e),
         cudaGetErrorString(e2), hc, ha[1], limit, limit * (limit + 1) / 2.0, ms, ms * 1e3 / limit);
}
