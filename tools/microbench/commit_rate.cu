// MMA issue throughput with commits but no consumers: one warp issues
// `iters` accumulator groups (K = 32*ks, M=128, N) round-robin over NACC
// TMEM accumulators, committing to an mbarrier every `every` groups
// (nobody waits except the final drain).  Cycles per group vs the floor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

template <int N, int NACC, int SINGLE>
__global__ void __launch_bounds__(128, 1) probe(int iters, int ks_n, int every, int wait_each, int pat, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = pat == 0 ? (uint8_t)(i * 7 + 3) : pat == 1 ? (uint8_t)0 : pat == 2 ? (uint8_t)(i * 7) : (uint8_t)((i * 2654435761u) >> 24);
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) ptx::mbar_init(ptx::smem_u32(&bar[i]), 1); ptx::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 1 && (!SINGLE || threadIdx.x == 32)) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = ptx::idesc_i8(128, N);
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    int nc = 0;
    for (int h = 0; h < iters; ++h) {
      const int acc = h % NACC;
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        if (SINGLE) ptx::umma_i8(tm + acc * N, ad, bd, idesc, ks ? 1u : 0u);
        else ptx::umma_i8_elect(tm + acc * N, ad, bd, idesc, ks ? 1u : 0u);
      }
      if ((h + 1) % every == 0) {
        const int bi = nc & 7;
        if (SINGLE) ptx::umma_commit(ptx::smem_u32(&bar[bi]));
        else ptx::umma_commit_elect(ptx::smem_u32(&bar[bi]));
        ++nc;
        // wait for the commit issued `wait_each` commits ago (0: never until the end)
        if (wait_each && nc >= wait_each) {
          const int w = nc - wait_each;
          ptx::mbar_wait(ptx::smem_u32(&bar[w & 7]), (w >> 3) & 1);
        }
      }
    }
    if (SINGLE) ptx::umma_commit(ptx::smem_u32(&bar[nc & 7]));
    else ptx::umma_commit_elect(ptx::smem_u32(&bar[nc & 7]));
    ptx::mbar_wait(ptx::smem_u32(&bar[nc & 7]), (nc >> 3) & 1);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    (void)ph;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

template <int N, int NACC, int SINGLE = 0>
void run(int ks, int every, int wait_each, int pat = 0) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe<N, NACC, SINGLE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  probe<N, NACC, SINGLE><<<148, 128, smem>>>(64, ks, every, wait_each, pat, d);
  probe<N, NACC, SINGLE><<<148, 128, smem>>>(iters, ks, every, wait_each, pat, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("pat=%d single=%d N=%3d NACC=%d K=%3d commit every %d, wait lag %d: %6.0f cycles/group (floor %4d) (%s)\n", pat, SINGLE, N, NACC,
         32 * ks, every, wait_each, (double)h / iters, N * ks / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int pat = 0; pat < 4; ++pat) {
    run<256, 2, 0>(2, 1000000, 0, pat);
    run<256, 2, 0>(3, 1000000, 0, pat);
    run<256, 2, 0>(3, 1, 1, pat);
    run<128, 4, 0>(3, 1000000, 0, pat);
  }
  return 0;
}
