// Which pipe do the 3-input integer / float minima use?  Each thread runs
// 8 independent chains of N minima; cycles per warp instruction per SMSP for
// VIMNMX3 alone, FMNMX3 alone and both interleaved (if they share a pipe the
// mixed rate equals the single rates; if not, it doubles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float fmin3(float a, float b, float c) {
  return fminf(fminf(a, b), c);
}
__device__ __forceinline__ int imin3(int a, int b, int c) {
  return __vimin3_s32(a, b, c);
}

template <int MODE>
__global__ void k(int n, int* out, unsigned long long* cyc) {
  int a[8];
  float f[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 7 + j; f[j] = __int_as_float(threadIdx.x * 5 + j); }
  const int b = threadIdx.x ^ 3, c = threadIdx.x ^ 5;
  const float fb = __int_as_float(b), fc = __int_as_float(c);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0 || MODE == 2) a[j] = imin3(a[j], b + i, c);
      if (MODE == 1 || MODE == 2) f[j] = fmin3(f[j], fb, fc);
    }
  }
  unsigned long long t1 = clock64();
  int s = 0;
  for (int j = 0; j < 8; ++j) s += a[j] + __float_as_int(f[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int n = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int w = 8; w <= 32; w *= 2) {
      unsigned long long h;
      if (mode == 0) { k<0><<<148, w * 32>>>(n, out, cyc); }
      if (mode == 1) { k<1><<<148, w * 32>>>(n, out, cyc); }
      if (mode == 2) { k<2><<<148, w * 32>>>(n, out, cyc); }
      cudaDeviceSynchronize();
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double inst = (double)n * 8 * (mode == 2 ? 2 : 1) * w / 4;  // warp instructions per SMSP
      printf("mode %d (%s) warps %2d: %.2f cycles per warp-instruction per SMSP\n", mode,
             mode == 0 ? "VIMNMX3" : mode == 1 ? "FMNMX3" : "both", w, (double)h / inst);
    }
  }
  return 0;
}
