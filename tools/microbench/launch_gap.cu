// Back-to-back launch cost on one stream: empty kernels, direct vs CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n = 200;
  for (int blocks : {1, 148, 1184}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s);
      for (int i = 0; i < n; ++i) empty_k<<<blocks, 128, 0, s>>>(nullptr);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("direct  blocks=%4d: %.2f us per launch\n", blocks, 1e3 * ms / n);
    }
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) empty_k<<<blocks, 128, 0, s>>>(nullptr);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("graph   blocks=%4d: %.2f us per launch\n", blocks, 1e3 * ms / n);
    }
  }
  return 0;
}
