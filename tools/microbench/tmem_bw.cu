// TMEM -> register read bandwidth probe (tcgen05.ld 32x32b.xN), per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

template <int NW, int X>
__global__ void __launch_bounds__(NW * 32, 1) probe(int iters, unsigned long long* cycles, int* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  int acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 512; c += 32 * (X / 32)) {
      int v[32];
      ptx::tmem_ld32(base + ((c + warp * 32) & 511), v);
      if constexpr (X >= 64) {
        int w[32];
        ptx::tmem_ld32(base + ((c + 32 + warp * 32) & 511), w);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j] + w[j];
      } else {
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
      }
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(slot, 512);
}

template <int NW, int X>
void run(const char* name) {
  const int iters = 2000, blocks = 148;
  unsigned long long* d_c;
  int* d_s;
  cudaMalloc(&d_c, blocks * 8);
  cudaMalloc(&d_s, blocks * NW * 32 * 4);
  probe<NW, X><<<blocks, NW * 32>>>(10, d_c, d_s);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NW, X><<<blocks, NW * 32>>>(iters, d_c, d_s);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
  const double bytes_per_sm = (double)iters * NW * 512 * 32 * 4;  // each warp reads 512 cols x 32 lanes
  printf("%s warps=%d: %.1f B/cycle/SM (clock64), %.2f TB/s chip, err=%s\n", name, NW,
         bytes_per_sm / (double)h[0], bytes_per_sm * blocks / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d_c);
  cudaFree(d_s);
}

int main() {
  run<4, 32>("ld32x32b.x32");
  run<8, 32>("ld32x32b.x32");
  run<16, 32>("ld32x32b.x32");
  run<4, 64>("ld32x32b.x32 x2 in flight");
  run<8, 64>("ld32x32b.x32 x2 in flight");
  run<16, 64>("ld32x32b.x32 x2 in flight");
  return 0;
}
