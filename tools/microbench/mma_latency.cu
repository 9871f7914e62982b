// tcgen05.mma kind::i8 latency probe: issue -> commit -> mbarrier observed, per
// iteration, for K = 32 * ks (M=128, N=256), one accumulator, one thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

__global__ void __launch_bounds__(128, 1) probe(int iters, int ks_n, int sleep, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = ptx::idesc_i8(128, 256);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        ptx::umma_i8(tm, ad, bd, idesc, ks ? 1u : 0u);
      }
      ptx::umma_commit(ptx::smem_u32(&bar));
      if (sleep) ptx::mbar_wait_sleep(ptx::smem_u32(&bar), it & 1);
      else ptx::mbar_wait(ptx::smem_u32(&bar), it & 1);
      ptx::tc_fence_after();
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

int main() {
  const int iters = 2000, blocks = 148;
  unsigned long long* d_c;
  cudaMalloc(&d_c, blocks * 8);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int sleep = 0; sleep < 2; ++sleep)
    for (int ks = 1; ks <= 4; ++ks) {
      probe<<<blocks, 128, smem>>>(10, ks, sleep, d_c);
      probe<<<blocks, 128, smem>>>(iters, ks, sleep, d_c);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
      printf("K=%3d sleep=%d: %.0f cycles per MMA->commit->wait round trip (%s)\n", 32 * ks, sleep,
             (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
