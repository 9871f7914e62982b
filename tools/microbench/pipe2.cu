// Handshake sweep: NACC TMEM accumulators of N columns (M=128, K=32*ks,
// kind::i8 from smem), EPI epilogue warps in G groups; group g drains the
// accumulator uses h == g (mod G).  Each warp covers its sub-partition's 32
// lanes and a slice of N*4*G/EPI columns, loaded in 64-column chunks (two
// x32 loads, one wait), reduced with a VIMNMX3 tree like tc_scan_kernel's
// epilogue; the accumulator is released after the last chunk's loads.
// Prints cycles per 128x256 tile-equivalent and the MMA floor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

__device__ __forceinline__ int min8(const int* v) {
  return __vimin3_s32(__vimin3_s32(v[0], v[1], v[2]), __vimin3_s32(v[3], v[4], v[5]), min(v[6], v[7]));
}

template <int EPI, int NACC, int N, int G, int ISS>
__global__ void __launch_bounds__((4 + EPI) * 32, 1) probe(int iters, int ks_n, unsigned long long* out, long long* ts) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[2 * NACC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) smem[i] = (uint8_t)(i * 7 + 3);
  constexpr int kPerGroup = EPI / G;              // warps per group (multiple of 4)
  constexpr int kCols = N * 4 / kPerGroup;        // columns per warp and accumulator use
  if (threadIdx.x == 0) {
    for (int b = 0; b < NACC; ++b) {
      ptx::mbar_init(ptx::smem_u32(&bars[b]), 1);
      ptx::mbar_init(ptx::smem_u32(&bars[NACC + b]), kPerGroup);
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
  int best = 0x7fffffff;
  if (warp < ISS) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = ptx::idesc_i8(128, N);
    for (int h = warp; h < iters; h += ISS) {
      const int acc = h % NACC;
      ptx::mbar_wait_sleep(ptx::smem_u32(&bars[NACC + acc]), ((h / NACC) & 1) ^ 1);
      ptx::tc_fence_after();
      if (blockIdx.x == 0 && lane == 0 && h >= 1000 && h < 1064) ts[(h - 1000) * 4 + 0] = clock64();
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        ptx::umma_i8_elect(tm + acc * N, ad, bd, idesc, ks ? 1u : 0u);
      }
      ptx::umma_commit_elect(ptx::smem_u32(&bars[acc]));
      if (blockIdx.x == 0 && lane == 0 && h >= 1000 && h < 1064) ts[(h - 1000) * 4 + 1] = clock64();
    }
  } else if (warp >= 4) {
    const int e = warp - 4, sp = warp & 3;
    const int grp = e / kPerGroup, eg = (e % kPerGroup) >> 2;
    const uint32_t base = tm + ((uint32_t)(sp * 32) << 16) + eg * kCols;
    for (int h = grp; h < iters; h += G) {
      const int acc = h % NACC;
      ptx::mbar_wait_sleep(ptx::smem_u32(&bars[acc]), (h / NACC) & 1);
      ptx::tc_fence_after();
      const bool rec = blockIdx.x == 0 && lane == 0 && (e % kPerGroup) == 0 && h >= 1000 && h < 1064;
      if (rec) ts[(h - 1000) * 4 + 2] = clock64();
      int v[64];
#pragma unroll 1
      for (int c = 0; c < kCols; c += 64) {
        if (kCols >= 64) {
          ptx::tmem_ld32(base + acc * N + c, *reinterpret_cast<int(*)[32]>(v));
          ptx::tmem_ld32(base + acc * N + c + 32, *reinterpret_cast<int(*)[32]>(v + 32));
        } else {
          ptx::tmem_ld32(base + acc * N + c, *reinterpret_cast<int(*)[32]>(v));
        }
        ptx::tmem_wait_ld();
        if (c + 64 >= kCols) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&bars[NACC + acc]));
          if (rec) ts[(h - 1000) * 4 + 3] = clock64();
        }
        int m = min8(v);
#pragma unroll
        for (int j = 8; j < (kCols >= 64 ? 64 : 32); j += 8) m = min(m, min8(v + j));
        best = min(best, m);
      }
    }
  }
  unsigned long long t1 = clock64();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tm, 512);
  if (threadIdx.x == 128) out[blockIdx.x] = t1 - t0;
  if (best == 12345) out[blockIdx.x + 1000] = best;
}

template <int EPI, int NACC, int N, int G, int ISS = 1>
void run(int ks) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 2048);
  long long* dts;
  cudaMalloc(&dts, 8 * 4 * 64);
  const int smem = (128 + 256) * 128;
  cudaFuncSetAttribute(probe<EPI, NACC, N, G, ISS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  probe<EPI, NACC, N, G, ISS><<<148, (4 + EPI) * 32, smem>>>(64, ks, d, dts);
  probe<EPI, NACC, N, G, ISS><<<148, (4 + EPI) * 32, smem>>>(iters, ks, d, dts);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per_tile = (double)h / iters * 256 / N;
  printf("ISS=%d EPI=%2d NACC=%d N=%3d G=%d K=%3d: %6.0f cycles/acc, %6.0f per 128x256 tile, MMA floor %4d (%s)\n",
         ISS, EPI, NACC, N, G, 32 * ks, (double)h / iters, per_tile, 128 * ks,
         cudaGetErrorString(cudaGetLastError()));
  long long t[256];
  cudaMemcpy(t, dts, sizeof t, cudaMemcpyDeviceToHost);
  double issue_full = 0, hold = 0, rel_issue = 0, issue_dur = 0;
  int n = 0;
  for (int h = 0; h + NACC < 64; ++h) {
    issue_full += t[h * 4 + 2] - t[h * 4 + 0];
    hold += t[h * 4 + 3] - t[h * 4 + 2];
    rel_issue += t[(h + NACC) * 4 + 0] - t[h * 4 + 3];
    issue_dur += t[h * 4 + 1] - t[h * 4 + 0];
    ++n;
  }
  printf("    issue->full %.0f (exec %d)  full->release %.0f  release->next issue %.0f  issue+commit %.0f\n",
         issue_full / n, 128 * ks * N / 256, hold / n, rel_issue / n, issue_dur / n);
  cudaFree(dts);
  cudaFree(d);
}

int main() {
  for (int ks = 2; ks <= 3; ++ks) {
    run<16, 2, 256, 2, 1>(ks);
    run<16, 2, 256, 2, 2>(ks);
    run<16, 4, 128, 4, 2>(ks);
    run<16, 4, 128, 4, 4>(ks);
    run<16, 4, 128, 2, 4>(ks);
    run<16, 8, 64, 4, 4>(ks);
    run<16, 8, 64, 2, 4>(ks);
  }
  return 0;
}
