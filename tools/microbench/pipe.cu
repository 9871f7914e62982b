// MMA -> epilogue handshake pipeline probe: one MMA warp fills NACC TMEM
// accumulators (M=128, N=256/NACC*2.., K = 32*ks), EPI epilogue warps drain
// each accumulator with tcgen05.ld and release it.  Cycles per accumulator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

template <int EPI, int NACC, int N, int GROUPS, int SPIN>
__global__ void __launch_bounds__((4 + EPI) * 32, 1) probe(int iters, int ks_n, int work, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[2 * NACC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = (uint8_t)(i * 7 + 3);
  if (threadIdx.x == 0) {
    for (int b = 0; b < NACC; ++b) {
      ptx::mbar_init(ptx::smem_u32(&bars[b]), 1);
      ptx::mbar_init(ptx::smem_u32(&bars[NACC + b]), EPI / GROUPS);
    }
    ptx::fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  unsigned long long t0 = clock64();
  int sink = 0;
  if (warp == 1) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = ptx::idesc_i8(128, N);
    for (int h = 0; h < iters; ++h) {
      const int acc = h % NACC;
      if (SPIN & 1) ptx::mbar_wait(ptx::smem_u32(&bars[NACC + acc]), ((h / NACC) & 1) ^ 1);
      else ptx::mbar_wait_sleep(ptx::smem_u32(&bars[NACC + acc]), ((h / NACC) & 1) ^ 1);
      ptx::tc_fence_after();
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        ptx::umma_i8_elect(tm + acc * N, ad, bd, idesc, ks ? 1u : 0u);
      }
      ptx::umma_commit_elect(ptx::smem_u32(&bars[acc]));
    }
  } else if (warp >= 4) {
    const int e = warp - 4, sp = warp & 3;
    const int per_group = EPI / GROUPS;           // warps per group
    const int grp = e / per_group, eg = e % per_group;
    const int cols_per = N * 4 / per_group;       // columns per warp
    const uint32_t base = tm + ((uint32_t)(sp * 32) << 16) + (eg >> 2) * cols_per;
    for (int h = grp; h < iters; h += GROUPS) {
      const int acc = h % NACC;
      if (SPIN & 2) ptx::mbar_wait(ptx::smem_u32(&bars[acc]), (h / NACC) & 1);
      else ptx::mbar_wait_sleep(ptx::smem_u32(&bars[acc]), (h / NACC) & 1);
      ptx::tc_fence_after();
      int v[32], u[32];
      if (cols_per >= 64) {
        for (int c = 0; c < cols_per; c += 64) {
          ptx::tmem_ld32(base + acc * N + c, v);
          ptx::tmem_ld32(base + acc * N + c + 32, u);
          ptx::tmem_wait_ld();
          for (int j = 0; j < 32; ++j) sink += v[j] ^ u[j];
        }
      } else {
        for (int c = 0; c < cols_per; c += 32) {
          ptx::tmem_ld32(base + acc * N + c, v);
          ptx::tmem_wait_ld();
          for (int j = 0; j < 32; ++j) sink += v[j];
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&bars[NACC + acc]));
      for (int w = 0; w < work; ++w) sink = sink * 3 + w;
    }
  }
  unsigned long long t1 = clock64();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tm, 512);
  if (threadIdx.x == 128) out[blockIdx.x] = t1 - t0;
  if (sink == 12345) out[blockIdx.x + 1000] = sink;
}

template <int EPI, int NACC, int N, int GROUPS = 1, int SPIN = 0>
void run(int ks, int work) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe<EPI, NACC, N, GROUPS, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  probe<EPI, NACC, N, GROUPS, SPIN><<<148, (4 + EPI) * 32, smem>>>(50, ks, work, d);
  probe<EPI, NACC, N, GROUPS, SPIN><<<148, (4 + EPI) * 32, smem>>>(iters, ks, work, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("SPIN=%d G=%d EPI=%2d NACC=%d N=%d K=%3d work=%3d: %6.0f cycles/acc, %6.0f per 128x256 tile (%s)\n", SPIN, GROUPS, EPI, NACC, N,
         32 * ks, work, (double)h / iters, (double)h / iters * 256 / N, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int ks = 1; ks <= 3; ++ks) {
    run<16, 2, 256, 2, 0>(ks, 0);
    run<16, 2, 256, 2, 1>(ks, 0);
    run<16, 2, 256, 2, 2>(ks, 0);
    run<16, 2, 256, 2, 3>(ks, 0);
    run<16, 4, 128, 4, 0>(ks, 0);
    run<16, 4, 128, 4, 3>(ks, 0);
    run<16, 2, 256, 1, 3>(ks, 0);
  }
  return 0;
}
