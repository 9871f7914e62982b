// In-run roofline probe: dense tcgen05.mma kind::i8 issue rate on this GPU
// with the same shared-memory layout / descriptors as tc_scan_kernel
// (M=128, N=256, K=32 per instruction, operands resident in smem, no
// epilogue).  bench.py uses it as the int8 tensor-core peak denominator.
#include "fc_internal.cuh"
#include "fc_tc_ptx.cuh"

namespace fcb {
namespace {

__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 64; i += blockDim.x) smem[i] = (uint8_t)(i * 7);
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 64;
    constexpr uint32_t idesc = ptx::idesc_i8(128, 256);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t ad = ptx::umma_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = ptx::umma_desc(b + ks * 2 * 4096, 4096, 128);
        ptx::umma_i8(tm + (it & 1) * 256, ad, bd, idesc, ks);
      }
    }
    ptx::umma_commit(ptx::smem_u32(&bar));
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) ptx::tmem_dealloc(tm, 512);
}

}  // namespace
}  // namespace fcb

using namespace fcb;

extern "C" int fc_probe_int8_peak(fc_ctx* cp, double* tops) {
  Ctx* c = reinterpret_cast<Ctx*>(cp);
  cudaSetDevice(c->device);
  const int iters = 20000, smem = (128 + 256) * 64;
  DevBuf cyc;
  FC_CUDA(c, cyc.reserve(c->sm_count * 8));
  FC_CUDA(c, cudaFuncSetAttribute(mma_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
  mma_peak_kernel<<<c->sm_count, 128, smem, c->stream>>>(200, cyc.as<unsigned long long>());
  FC_CUDA(c, cudaGetLastError());
  FC_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  mma_peak_kernel<<<c->sm_count, 128, smem, c->stream>>>(iters, cyc.as<unsigned long long>());
  FC_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  FC_CUDA(c, cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  cyc.release();
  const double ops = 2.0 * iters * 128.0 * 256.0 * 64.0 * c->sm_count;
  *tops = ops / (ms * 1e-3) / 1e12;
  c->total_launches += 2;
  return FC_OK;
}
