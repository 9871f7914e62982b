// tcgen05.mma kind::i8 issue-rate probe with the library's smem layout/descriptors.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

template <int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 64; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 64;
    constexpr uint32_t idesc = ptx::idesc_i8(128, N);
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * (N * 16), N * 16, 128);
        ptx::umma_i8(tm + (it & 1) * N, ad, bd, idesc, ks);
      }
    }
    ptx::umma_commit(ptx::smem_u32(&bar));
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

template <int N>
void run() {
  const int iters = 20000, blocks = 148;
  unsigned long long* d_c;
  cudaMalloc(&d_c, blocks * 8);
  const int smem = (128 + 256) * 64;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<blocks, 128, smem>>>(100, d_c);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<N><<<blocks, 128, smem>>>(iters, d_c);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
  const double macs = (double)iters * 128 * N * 64;
  printf("i8 MMA M=128 N=%d K=64: %.0f MACs/cycle/SM, %.1f TOPS chip (%.3f ms) err=%s\n", N,
         macs / (double)h[0], 2 * macs * blocks / (ms * 1e-3) / 1e12, ms,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<128>();
  run<256>();
  return 0;
}
