// TMEM write (tcgen05.st 32x32b.x32) and read+write bandwidth probe, per SM.
// Question: can the epilogue re-initialise an accumulator with per-column
// constants (tcgen05.st after its tcgen05.ld) at a cost below the TMEM read?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1502_00324_b200/csrc/fc_tc_ptx.cuh"

using namespace fcb;

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const int (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
        "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
        "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]),
        "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: ld only, 1: st only, 2: ld then st of the same columns
template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) probe(int iters, unsigned long long* cycles, int* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  int acc = 0;
  int w[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) w[j] = threadIdx.x * 7 + j;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 512; c += 32) {
      const uint32_t a = base + ((c + (warp >> 2) * 32) & 511);
      if constexpr (MODE != 1) {
        int v[32];
        ptx::tmem_ld32(a, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= v[j];
      }
      if constexpr (MODE != 0) {
        tmem_st32(a, w);
        w[0] += acc;
      }
    }
    if constexpr (MODE != 0) tmem_wait_st();
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + w[0];
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(slot, 512);
}

template <int NW, int MODE>
void run(const char* name) {
  const int iters = 2000, blocks = 148;
  unsigned long long* d_c;
  int* d_s;
  cudaMalloc(&d_c, blocks * 8);
  cudaMalloc(&d_s, blocks * NW * 32 * 4);
  probe<NW, MODE><<<blocks, NW * 32>>>(10, d_c, d_s);
  cudaDeviceSynchronize();
  probe<NW, MODE><<<blocks, NW * 32>>>(iters, d_c, d_s);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d_c, sizeof h, cudaMemcpyDeviceToHost);
  // each warp touches 512 columns x 32 lanes x 4 B per iteration (once per direction)
  const double bytes_per_sm = (double)iters * NW * 512 * 32 * 4;
  printf("%-10s warps=%2d: %.1f B/cycle/SM per direction, err=%s\n", name, NW,
         bytes_per_sm / (double)h[0], cudaGetErrorString(cudaGetLastError()));
  cudaFree(d_c);
  cudaFree(d_s);
}

int main() {
  run<4, 0>("ld");
  run<8, 0>("ld");
  run<16, 0>("ld");
  run<4, 1>("st");
  run<8, 1>("st");
  run<16, 1>("st");
  run<4, 2>("ld+st");
  run<8, 2>("ld+st");
  run<16, 2>("ld+st");
  return 0;
}
