// Which issue-loop detail costs the tcgen05.mma rate?  Variants of mma_rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

// V: 0 mma_rate as is (thread 0, unrolled ks=2, A at 0 / B at 8 KB)
//    1 runtime ks_n loop
//    2 warp 1 lane 0 issues
//    3 warp 1, elect variant, unrolled
//    4 warp 1, elect, runtime ks loop, acc = h % 2 (commit_rate's loop minus commits)
//    5 as 0 but B at 16 KB (commit_rate's layout)
template <int V>
__global__ void __launch_bounds__(128, 1) probe(int iters, int ks_n, int every, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bars[8];
  int nc = 0;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); for (int i = 0; i < 8; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), 1); ptx::fence_mbar_init(); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 3) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t a = ptx::smem_u32(smem), b = a + (V == 5 || V == 4 ? 128 * 128 : 128 * 64);
  constexpr uint32_t idesc = ptx::idesc_i8(128, 256);
  const bool single = (V == 0 || V == 1 || V == 5) ? threadIdx.x == 0 : (V == 2 ? threadIdx.x == 32 : false);
  const bool warp1 = V >= 3 && V != 5 && warp == 1;
  unsigned long long t0 = clock64();
  if (single) {
    for (int it = 0; it < iters; ++it) {
      if (V == 1) {
        for (int ks = 0; ks < ks_n; ++ks) {
          const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
          const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
          ptx::umma_i8(tm + (it & 1) * 256, ad, bd, idesc, ks);
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
          const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
          ptx::umma_i8(tm + (it & 1) * 256, ad, bd, idesc, ks);
        }
      }
    }
    ptx::umma_commit(ptx::smem_u32(&bar));
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    cycles[blockIdx.x] = clock64() - t0;
  } else if (warp1) {
    for (int it = 0; it < iters; ++it) {
      if (V >= 4) {
        const int acc = it % 2;
        for (int ks = 0; ks < ks_n; ++ks) {
          const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
          const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
          ptx::umma_i8_elect(tm + acc * 256, ad, bd, idesc, ks ? 1u : 0u);
        }
        if (V == 6 && (it + 1) % every == 0) {
          ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
          ++nc;
        }
        if (V == 7) {
          ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
          ++nc;
        }
        if (V == 8) {
          ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
          ++nc;
          if (nc >= 2) { const int w = nc - 2; ptx::mbar_wait(ptx::smem_u32(&bars[w & 7]), (w >> 3) & 1); }
        }
        if (V == 9) {
          ptx::umma_commit_elect(ptx::smem_u32(&bars[nc & 7]));
          ++nc;
          if (nc >= 2) { const int w = nc - 2; ptx::mbar_wait_sleep(ptx::smem_u32(&bars[w & 7]), (w >> 3) & 1); }
        }
      } else {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
          const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
          ptx::umma_i8_elect(tm + (it & 1) * 256, ad, bd, idesc, ks);
        }
      }
    }
    ptx::umma_commit_elect(ptx::smem_u32(&bar));
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    if (threadIdx.x == 32) cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 3) ptx::tmem_dealloc(tm, 512);
}

template <int V>
void run(int ks = 2) {
  const int iters = 20000, blocks = 148;
  unsigned long long* d_c;
  cudaMalloc(&d_c, blocks * 8);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<V><<<blocks, 128, smem>>>(100, ks, 1000000, d_c);
  probe<V><<<blocks, 128, smem>>>(iters, ks, 1000000, d_c);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
  printf("V=%d K=%d: %.0f cycles per group (floor %d) err=%s\n", V, 32 * ks, (double)h[0] / iters, 128 * ks,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  for (int ks = 2; ks <= 3; ++ks) {
    run<4>(ks);
    run<6>(ks);
    run<7>(ks);
    run<8>(ks);
    run<9>(ks);
  }
  return 0;
}
