// Where does the MMA-issuing thread spend its time?  One warp issues groups of
// ks MMAs (M=128, N=256, kind::i8) into 2 accumulators; variant W adds per
// group: 0 nothing, 1 commit, 2 commit + wait on the commit of 2 groups ago,
// 3 wait only (on a barrier completed long ago).  Average cycles per group
// spent in: MMA issue, commit, wait, rest.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

__global__ void __launch_bounds__(128, 1) probe(int iters, int ks_n, int W, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[8];
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), 1);
    ptx::mbar_init(ptx::smem_u32(&done), 1);
    ptx::fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 3) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) ptx::mbar_arrive(ptx::smem_u32(&done));  // phase 0 completes now
  __syncthreads();
  const uint32_t tm = slot;
  const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
  constexpr uint32_t idesc = ptx::idesc_i8(128, 256);
  if (warp == 1) {
    unsigned long long s_mma = 0, s_commit = 0, s_wait = 0;
    int nc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const unsigned long long c0 = clock64();
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        ptx::umma_i8_elect(tm + (it & 1) * 256, ad, bd, idesc, ks ? 1u : 0u);
      }
      const unsigned long long c1 = clock64();
      if (W == 1 || W == 2) {
        ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
        ++nc;
      }
      const unsigned long long c2 = clock64();
      if (W == 2 && nc >= 3) {
        const int w = nc - 3;
        ptx::mbar_wait(ptx::smem_u32(&bars[w & 7]), (w >> 3) & 1);
      }
      if (W == 3) ptx::mbar_wait(ptx::smem_u32(&done), 0);
      const unsigned long long c3 = clock64();
      s_mma += c1 - c0;
      s_commit += c2 - c1;
      s_wait += c3 - c2;
    }
    ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
    ptx::mbar_wait(ptx::smem_u32(&bars[nc & 7]), (nc >> 3) & 1);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) {
      out[0] = t1 - t0; out[1] = s_mma; out[2] = s_commit; out[3] = s_wait;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 3) ptx::tmem_dealloc(tm, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  for (int ks = 1; ks <= 3; ++ks)
    for (int W = 0; W < 4; ++W) {
      probe<<<148, 128, smem>>>(64, ks, W, d);
      probe<<<148, 128, smem>>>(iters, ks, W, d);
      cudaDeviceSynchronize();
      unsigned long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("K=%3d W=%d: %5.0f cycles/group (floor %3d): issue %5.1f commit %5.1f wait %5.1f (%s)\n", 32 * ks, W,
             (double)h[0] / iters, 128 * ks, (double)h[1] / iters, (double)h[2] / iters, (double)h[3] / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
