// Domain-pool construction on the device (pool.py:88-178, image.py:116-130).
//
//  1. entropy_kernel   : one warp per 2Bx2B lattice window (raster order,
//                        pool.py:120-135); 256-bin shared-memory histogram,
//                        then H = -sum_b t[count_b] with t[k] = p*log(p) from the
//                        host-numpy LUT, summed in numpy's exact pairwise order
//                        (two 128-bin halves, 8 running accumulators each,
//                        ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), half0+half1) so the
//                        float64 bits equal pool.py:88-92 on the same host.
//  2. CUB stable radix sort on key ~bits(|H|): entropy descending, raster order
//     among exact ties (np.argsort(-ent, kind="stable"), pool.py:171).
//  3. survivor_kernel  : one warp per kept window: floor 2x2 decimation,
//                        exact sum / sum of squares, mean, centered norm
//                        (pool.py:138-152).
#include <cub/cub.cuh>

#include "fc_internal.cuh"

namespace fcb {

namespace {

constexpr int kEntWarps = 8;

__device__ __forceinline__ uint64_t entropy_key(double h) {
  // |h|: maps the -0.0 of a constant window onto +0.0 (they compare equal in numpy).
  uint64_t bits = static_cast<uint64_t>(__double_as_longlong(h)) & 0x7fffffffffffffffull;
  return ~bits;  // ascending key == descending entropy
}

template <int D>
__global__ void __launch_bounds__(kEntWarps * 32)
entropy_kernel(const uint8_t* __restrict__ img, int width, int nx, int64_t nwin, int stride,
               const double* __restrict__ lut, double tau, int use_tau,
               double* __restrict__ ent_out, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
               unsigned long long* __restrict__ above) {
  __shared__ int hist[kEntWarps][256];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int* h = hist[warp];
  int local_above = 0;
  for (int64_t w = (int64_t)blockIdx.x * kEntWarps + warp; w < nwin;
       w += (int64_t)gridDim.x * kEntWarps) {
#pragma unroll
    for (int i = 0; i < 8; ++i) h[lane + 32 * i] = 0;
    __syncwarp();
    const int64_t wy = w / nx, wx = w - wy * nx;
    const uint8_t* base = img + (wy * stride) * (int64_t)width + wx * stride;
#pragma unroll 4
    for (int p = lane; p < D * D; p += 32) {
      const int r = p / D, col = p - r * D;
      atomicAdd(&h[base[(int64_t)r * width + col]], 1);
    }
    __syncwarp();
    // numpy pairwise sum of the 256 terms (lanes 16..31 mirror lanes 0..15)
    const int half = (lane >> 3) & 1, j = lane & 7;
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int cnt = h[half * 128 + i * 8 + j];
      const double t = cnt ? lut[cnt - 1] : 0.0;
      acc = (i == 0) ? t : acc + t;
    }
    acc = acc + __shfl_xor_sync(0xffffffffu, acc, 1);
    acc = acc + __shfl_xor_sync(0xffffffffu, acc, 2);
    acc = acc + __shfl_xor_sync(0xffffffffu, acc, 4);
    acc = acc + __shfl_xor_sync(0xffffffffu, acc, 8);
    const double hval = -acc;
    if (lane == 0) {
      ent_out[w] = hval;
      keys[w] = entropy_key(hval);
      vals[w] = static_cast<uint32_t>(w);
      if (use_tau && hval > tau) ++local_above;
    }
    __syncwarp();
  }
  if (use_tau && lane == 0 && local_above) atomicAdd(above, (unsigned long long)local_above);
}

// One warp per survivor: decimate, moments, coordinates.
__global__ void survivor_kernel(const uint8_t* __restrict__ img, int width, int nx, int stride,
                                int D, const uint32_t* __restrict__ order,
                                const double* __restrict__ ent_all, int64_t count,
                                uint32_t* __restrict__ xy, double* __restrict__ ent,
                                uint8_t* __restrict__ tiles, int32_t* __restrict__ sum,
                                int64_t* __restrict__ sumsq, double* __restrict__ mean,
                                double* __restrict__ cnorm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= count) return;
  const uint32_t w = order[warp];
  const int wy = w / nx, wx = w - wy * nx;
  const int x0 = wx * stride, y0 = wy * stride;
  const int B = D / 2, n = B * B;
  const uint8_t* base = img + (int64_t)y0 * width + x0;
  uint8_t* out = tiles + (int64_t)warp * n;
  int s1 = 0;
  long long s2 = 0;
  for (int p = lane; p < n; p += 32) {
    const int r = p / B, c = p - r * B;
    const uint8_t* q = base + (int64_t)(2 * r) * width + 2 * c;
    const int v = (q[0] + q[1] + q[width] + q[width + 1]) >> 2;  // floor mean, image.py:125-130
    out[p] = static_cast<uint8_t>(v);
    s1 += v;
    s2 += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    xy[warp] = static_cast<uint32_t>(x0) | (static_cast<uint32_t>(y0) << 16);
    ent[warp] = ent_all[w];
    sum[warp] = s1;
    sumsq[warp] = s2;
    // mean = s1 / n; cnorm = s2 - s1*s1/n with Python float semantics (pool.py:144-151)
    mean[warp] = __ddiv_rn((double)s1, (double)n);
    cnorm[warp] = __dsub_rn((double)s2, __ddiv_rn((double)((long long)s1 * s1), (double)n));
  }
}

// Moments of explicitly supplied decimated tiles (fc_pool_set_level).
__global__ void moments_kernel(const uint8_t* __restrict__ tiles, int n, int64_t count,
                               uint32_t* __restrict__ xy, double* __restrict__ ent,
                               int32_t* __restrict__ sum, int64_t* __restrict__ sumsq,
                               double* __restrict__ mean, double* __restrict__ cnorm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= count) return;
  const uint8_t* t = tiles + (int64_t)warp * n;
  int s1 = 0;
  long long s2 = 0;
  for (int p = lane; p < n; p += 32) {
    const int v = t[p];
    s1 += v;
    s2 += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    xy[warp] = 0;
    ent[warp] = 0.0;
    sum[warp] = s1;
    sumsq[warp] = s2;
    mean[warp] = __ddiv_rn((double)s1, (double)n);
    cnorm[warp] = __dsub_rn((double)s2, __ddiv_rn((double)((long long)s1 * s1), (double)n));
  }
}

// Threshold compaction predicate: window index -> entropy > tau (keeps raster order).
struct AboveTau {
  const double* ent;
  double tau;
  __device__ __forceinline__ bool operator()(const uint32_t& w) const { return ent[w] > tau; }
};

__global__ void gather_keys_kernel(const uint32_t* __restrict__ idx, const double* __restrict__ ent,
                                   int64_t n, uint64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = entropy_key(ent[idx[i]]);
}

// Lexicographic (key, index) minimum: the first window of the highest
// entropy, i.e. np.argsort(-ent, kind="stable")[0] (cap = 1 levels).
__device__ __forceinline__ void lex_min(uint64_t& k, uint32_t& i, uint64_t k2, uint32_t i2) {
  if (k2 < k || (k2 == k && i2 < i)) {
    k = k2;
    i = i2;
  }
}

__global__ void argmin_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                              int64_t n, uint64_t* __restrict__ out_k, uint32_t* __restrict__ out_i) {
  uint64_t bk = ~0ull;
  uint32_t bi = 0xffffffffu;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    lex_min(bk, bi, keys[i], vals ? vals[i] : (uint32_t)i);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
    const uint32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    lex_min(bk, bi, k2, i2);
  }
  __shared__ uint64_t sk[32];
  __shared__ uint32_t si[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sk[warp] = bk;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    bk = lane < (int)(blockDim.x >> 5) ? sk[lane] : ~0ull;
    bi = lane < (int)(blockDim.x >> 5) ? si[lane] : 0xffffffffu;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
      const uint32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      lex_min(bk, bi, k2, i2);
    }
    if (lane == 0) {
      out_k[blockIdx.x] = bk;
      out_i[blockIdx.x] = bi;
    }
  }
}

int alloc_level(Ctx* c, Level& L, int64_t E) {
  const int n = L.n;
  FC_CUDA(c, L.xy.reserve(E * 4 + 16));
  FC_CUDA(c, L.ent.reserve(E * 8 + 16));
  FC_CUDA(c, L.tiles.reserve(E * n + 16));
  FC_CUDA(c, L.sum.reserve(E * 4 + 16));
  FC_CUDA(c, L.sumsq.reserve(E * 8 + 16));
  FC_CUDA(c, L.mean.reserve(E * 8 + 16));
  FC_CUDA(c, L.cnorm.reserve(E * 8 + 16));
  return FC_OK;
}

}  // namespace

// Two-level argmin over n keys (index = position): out_k[0], out_i[0].
static int argmin_windows(Ctx* c, const uint64_t* keys, int64_t n, uint64_t* out_k,
                          uint32_t* out_i) {
  const int nb = (int)std::min<int64_t>((n + 1023) / 1024, 1024);
  argmin_kernel<<<nb, 1024, 0, c->stream>>>(keys, nullptr, n, out_k + 1, out_i + 1);
  argmin_kernel<<<1, 1024, 0, c->stream>>>(out_k + 1, out_i + 1, nb, out_k, out_i);
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 2;
  return FC_OK;
}

// All four levels are launched back to back with per-level scratch; the only
// synchronisation reads the threshold-survivor counts.  On return the pool
// sizes are known; the survivor data is produced in stream order.
int pool_build(Ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
               const int32_t use_tau[4], int64_t out_sizes[4]) {
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  for (int li = 0; li < kLevels; ++li) {
    if (strides[li] < 1) return set_error(c, FC_ERR_ARG, "strides must be 4 positive integers");
    if (!use_tau[li] && caps[li] < 1) return set_error(c, FC_ERR_ARG, "caps must be >= 1");
  }
  for (int li = 0; li < kLevels; ++li) {
    const int D = kDomainSide[li];
    if (D > c->width || D > c->height) {
      char buf[160];
      snprintf(buf, sizeof buf, "level %d domain side %d exceeds image %dx%d", li + 1, D, c->width,
               c->height);
      return set_error(c, FC_ERR_POOL_CONFIG, buf);
    }
    const int slot = lut_slot(D * D);
    if (!c->lut_set[slot]) return set_error(c, FC_ERR_STATE, "entropy LUT not set");
  }
  FC_CUDA(c, c->count_buf.reserve(64 * 4));
  FC_CUDA(c, c->pool_rb.reserve(64));
  int* d_nsel = reinterpret_cast<int*>(c->count_buf.ptr);
  int* h_nsel = c->pool_rb.as<int>();
  int nx_l[kLevels], any_tau = 0;
  // ---- phase 1: entropies and ranking for every level ----
  for (int li = 0; li < kLevels; ++li) {
    Level& L = c->lv[li];
    const int D = kDomainSide[li];
    L.side = kRangeSide[li];
    L.n = L.side * L.side;
    L.stride = strides[li];
    L.synthetic = false;
    L.prepared = false;
    L.tc.ready = false;
    const int nx = (c->width - D) / L.stride + 1;
    const int ny = (c->height - D) / L.stride + 1;
    nx_l[li] = nx;
    const int64_t nwin = (int64_t)nx * ny;
    FC_CUDA(c, L.win_ent.reserve(nwin * 8));
    FC_CUDA(c, L.win_key.reserve(nwin * 8));
    FC_CUDA(c, L.win_key2.reserve(nwin * 8 + 8 * 1032));
    FC_CUDA(c, L.win_val.reserve(nwin * 4));
    FC_CUDA(c, L.win_val2.reserve(nwin * 4 + 4 * 1032));
    const double* lut = c->lut[lut_slot(D * D)].as<double>();
    const int64_t blocks64 = (nwin + kEntWarps - 1) / kEntWarps;
    const int blocks = (int)std::min<int64_t>(blocks64, (int64_t)c->sm_count * 64);
#define FC_LAUNCH_ENT(DD)                                                                       \
    entropy_kernel<DD><<<blocks, kEntWarps * 32, 0, c->stream>>>(                               \
        c->img_ptr, c->width, nx, nwin, L.stride, lut, 0.0, 0, L.win_ent.as<double>(),          \
        L.win_key.as<uint64_t>(), L.win_val.as<uint32_t>(), nullptr)
    switch (D) {
      case 32: FC_LAUNCH_ENT(32); break;
      case 16: FC_LAUNCH_ENT(16); break;
      case 8: FC_LAUNCH_ENT(8); break;
      default: FC_LAUNCH_ENT(4); break;
    }
#undef FC_LAUNCH_ENT
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
    size_t tmp = 0;
    if (use_tau[li]) {
      // threshold compaction {ent > tau} in raster order
      any_tau = 1;
      AboveTau pred{L.win_ent.as<double>(), taus[li]};
      FC_CUDA(c, cub::DeviceSelect::If(nullptr, tmp, L.win_val.as<uint32_t>(),
                                        L.win_val2.as<uint32_t>(), d_nsel + li, (int)nwin, pred,
                                        c->stream));
      FC_CUDA(c, c->cub_tmp.reserve(tmp));
      FC_CUDA(c, cub::DeviceSelect::If(c->cub_tmp.ptr, tmp, L.win_val.as<uint32_t>(),
                                        L.win_val2.as<uint32_t>(), d_nsel + li, (int)nwin, pred,
                                        c->stream));
      FC_CUDA(c, cudaMemcpyAsync(h_nsel + li, d_nsel + li, 4, cudaMemcpyDeviceToHost, c->stream));
      c->total_launches += 1;
    } else if (caps[li] == 1) {
      FC_TRY(argmin_windows(c, L.win_key.as<uint64_t>(), nwin, L.win_key2.as<uint64_t>(),
                            L.win_val2.as<uint32_t>()));
      L.count = 1;
    } else {
      FC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, L.win_key.as<uint64_t>(),
                                                 L.win_key2.as<uint64_t>(), L.win_val.as<uint32_t>(),
                                                 L.win_val2.as<uint32_t>(), (int)nwin, 0, 64,
                                                 c->stream));
      FC_CUDA(c, c->cub_tmp.reserve(tmp));
      FC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.ptr, tmp, L.win_key.as<uint64_t>(),
                                                 L.win_key2.as<uint64_t>(), L.win_val.as<uint32_t>(),
                                                 L.win_val2.as<uint32_t>(), (int)nwin, 0, 64,
                                                 c->stream));
      L.count = std::min<int64_t>(caps[li], nwin);
    }
  }
  if (any_tau) FC_TRY(sync_stream(c));
  // ---- phase 2: survivors (sorted threshold sets), decimation and moments ----
  for (int li = 0; li < kLevels; ++li) {
    Level& L = c->lv[li];
    const int D = kDomainSide[li];
    const int nx = nx_l[li];
    const int64_t nwin = (int64_t)nx * ((c->height - D) / L.stride + 1);
    const uint32_t* order = L.win_val2.as<uint32_t>();
    if (use_tau[li]) {
      const int nsel = h_nsel[li];
      if (nsel == 0) {
        // caps are >= 1 (pool.py:47-48): keep the single highest-entropy window
        FC_TRY(argmin_windows(c, L.win_key.as<uint64_t>(), nwin, L.win_key2.as<uint64_t>(),
                              L.win_val2.as<uint32_t>()));
        L.count = 1;
      } else {
        const int64_t E = nsel;
        const unsigned tpb = 256;
        gather_keys_kernel<<<(unsigned)((E + tpb - 1) / tpb), tpb, 0, c->stream>>>(
            L.win_val2.as<uint32_t>(), L.win_ent.as<double>(), E, L.win_key2.as<uint64_t>());
        size_t tmp = 0;
        FC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, tmp, L.win_key2.as<uint64_t>(),
                                                   L.win_key.as<uint64_t>(), L.win_val2.as<uint32_t>(),
                                                   L.win_val.as<uint32_t>(), (int)E, 0, 64,
                                                   c->stream));
        FC_CUDA(c, c->cub_tmp.reserve(tmp));
        FC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.ptr, tmp, L.win_key2.as<uint64_t>(),
                                                   L.win_key.as<uint64_t>(), L.win_val2.as<uint32_t>(),
                                                   L.win_val.as<uint32_t>(), (int)E, 0, 64,
                                                   c->stream));
        order = L.win_val.as<uint32_t>();
        L.count = E;
        c->total_launches += 1;
      }
    }
    FC_CUDA(c, cudaGetLastError());
    const int64_t E = L.count;
    FC_TRY(alloc_level(c, L, E));
    const int threads = 256;
    const int64_t grid = (E * 32 + threads - 1) / threads;
    survivor_kernel<<<(unsigned)grid, threads, 0, c->stream>>>(
        c->img_ptr, c->width, nx, L.stride, D, order, L.win_ent.as<double>(), E,
        L.xy.as<uint32_t>(), L.ent.as<double>(), L.tiles.as<uint8_t>(), L.sum.as<int32_t>(),
        L.sumsq.as<int64_t>(), L.mean.as<double>(), L.cnorm.as<double>());
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
    out_sizes[li] = E;
  }
  return FC_OK;
}

int pool_set_level(Ctx* c, int level, int64_t count, const uint8_t* tiles) {
  Level& L = c->lv[level - 1];
  L.side = kRangeSide[level - 1];
  L.n = L.side * L.side;
  L.stride = 1;
  L.count = count;
  L.synthetic = true;
  L.prepared = false;
  L.tc.ready = false;
  if (count == 0) return FC_OK;
  FC_TRY(alloc_level(c, L, count));
  FC_TRY(stage_h2d(c, L.tiles.ptr, tiles, count * L.n));
  const int threads = 256;
  const int64_t grid = (count * 32 + threads - 1) / threads;
  moments_kernel<<<(unsigned)grid, threads, 0, c->stream>>>(
      L.tiles.as<uint8_t>(), L.n, count, L.xy.as<uint32_t>(), L.ent.as<double>(),
      L.sum.as<int32_t>(), L.sumsq.as<int64_t>(), L.mean.as<double>(), L.cnorm.as<double>());
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 1;
  return FC_OK;
}

}  // namespace fcb
