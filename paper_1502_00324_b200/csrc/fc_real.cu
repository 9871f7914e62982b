// Real-valued slope search behind the s-histogram analysis
// (bench.py:104-139: _level_basis + _real_s_matches; codec.py:164 _gather_tiles).
//
// For range r (n pixels, R1 = sum r) and domain entry e (decimated tile d,
// D1 = sum d, centered norm cnorm) the reference evaluates, per isometry,
//     cross = <iso(d - D1/n), r - R1/n>,   gain = cross*cross / cnorm,
//     err   = max(rnorm - gain, 0),        s    = cross / cnorm
// (gain = 0, s = 0 for a flat domain, cnorm == 0), and keeps the first
// minimum of err over the flat index e*8 + iso.
//
// Exactness: every factor of the fp64 GEMM the reference runs is an integer
// multiple of 1/n with magnitude <= 255, so every product and partial sum is
// an integer multiple of 1/n^2 below 2^53: numpy's `basis @ rc.T` is exact
// whatever its summation order, and equals (n*X - D1*R1) / n with the integer
// X = sum iso(d) * r.  Likewise rnorm = (n*R2 - R1^2) / n exactly.  So X comes
// from u8 x u8 dp4a dot products and the three rounded fp64 steps the
// reference takes (cross*cross, / cnorm, rnorm - gain) are repeated with the
// IEEE intrinsics: the result is bit-identical to the reference.
//
// Layout: one block per 4 ranges x one chunk of entries.  The 32 (range,
// isometry) rows are permuted into shared memory once (isometry as a pixel
// permutation of the range: sum iso(d)*r = sum d * r[inv_iso]); each thread
// streams whole entries and keeps the 32 dot products in registers.  The
// per-chunk winners are merged in chunk order by a second kernel.
#include <cfloat>
#include <cstdint>

#include "fc_internal.cuh"

namespace fcb {
namespace {

constexpr int kRealRanges = 4;  // x 8 isometries = 32 rows; <= 128 registers, 2 blocks per SM
constexpr int kRealRows = kRealRanges * 8;
constexpr int kRealThreads = 256;

template <int N>
__global__ void __launch_bounds__(kRealThreads, 2)
real_s_kernel(const uint8_t* __restrict__ rtiles, int64_t M, const uint16_t* __restrict__ inv,
              const uint8_t* __restrict__ dtiles, const int32_t* __restrict__ dsum,
              const double* __restrict__ dnorm, int64_t E, int64_t e_chunk,
              double* __restrict__ part_err, double* __restrict__ part_s,
              int64_t* __restrict__ part_idx) {
  constexpr int W = N / 4;            // 32-bit words per tile
  constexpr int CW = W >= 4 ? 4 : W;  // words per load
  __shared__ __align__(16) uint32_t a_s[kRealRows][W];
  __shared__ int32_t r1_s[kRealRanges];
  __shared__ double rnorm_s[kRealRanges];
  __shared__ double red_err[kRealThreads / 32][kRealRanges];
  __shared__ double red_s[kRealThreads / 32][kRealRanges];
  __shared__ int64_t red_idx[kRealThreads / 32][kRealRanges];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * kRealRanges;
  uint8_t* a_b = reinterpret_cast<uint8_t*>(&a_s[0][0]);
  for (int i = tid; i < kRealRows * N; i += kRealThreads) {
    const int row = i / N, j = i - row * N;
    const int64_t m = m0 + (row >> 3);
    a_b[i] = m < M ? rtiles[m * N + inv[(row & 7) * N + j]] : (uint8_t)0;
  }
  if (warp < kRealRanges) {  // one warp per range: R1 and rnorm
    const int64_t m = m0 + warp;
    long long s1 = 0, s2 = 0;
    if (m < M)
      for (int p = lane; p < N; p += 32) {
        const int v = rtiles[m * N + p];
        s1 += v;
        s2 += v * v;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      r1_s[warp] = (int32_t)s1;
      rnorm_s[warp] = __dmul_rn((double)((long long)N * s2 - s1 * s1), 1.0 / N);  // exact
    }
  }
  __syncthreads();

  double best_err[kRealRanges], best_cross[kRealRanges], best_norm[kRealRanges];
  int64_t best_idx[kRealRanges];
#pragma unroll
  for (int r = 0; r < kRealRanges; ++r) {
    best_err[r] = DBL_MAX;
    best_cross[r] = 0.0;
    best_norm[r] = 0.0;
    best_idx[r] = INT64_MAX;
  }
  const int64_t e0 = (int64_t)blockIdx.y * e_chunk;
  const int64_t e1 = min(E, e0 + e_chunk);
  for (int64_t e = e0 + tid; e < e1; e += kRealThreads) {
    unsigned acc[kRealRows];
#pragma unroll
    for (int r = 0; r < kRealRows; ++r) acc[r] = 0u;
    const uint8_t* dt = dtiles + e * N;
#pragma unroll 1
    for (int w0 = 0; w0 < W; w0 += CW) {
      uint32_t dw[CW];
      if constexpr (CW == 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(dt + 4 * w0));
        dw[0] = v.x; dw[1] = v.y; dw[2] = v.z; dw[3] = v.w;
      } else {
#pragma unroll
        for (int k = 0; k < CW; ++k) dw[k] = __ldg(reinterpret_cast<const uint32_t*>(dt) + w0 + k);
      }
#pragma unroll
      for (int r = 0; r < kRealRows; ++r) {
        if constexpr (CW == 4) {
          const uint4 a = *reinterpret_cast<const uint4*>(&a_s[r][w0]);
          unsigned x = acc[r];
          x = __dp4a(dw[0], a.x, x);
          x = __dp4a(dw[1], a.y, x);
          x = __dp4a(dw[2], a.z, x);
          x = __dp4a(dw[3], a.w, x);
          acc[r] = x;
        } else {
#pragma unroll
          for (int k = 0; k < CW; ++k) acc[r] = __dp4a(dw[k], a_s[r][w0 + k], acc[r]);
        }
      }
    }
    const long long d1 = dsum[e];
    const double norm = dnorm[e];
    const bool flat = norm == 0.0;
    const double rcp = flat ? 0.0 : __drcp_rn(norm);
#pragma unroll
    for (int r = 0; r < kRealRanges; ++r) {
      const long long r1 = r1_s[r];
      const double rn = rnorm_s[r];
#pragma unroll
      for (int iso = 0; iso < 8; ++iso) {
        const long long num = (long long)N * (long long)acc[r * 8 + iso] - d1 * r1;
        const double cross = __dmul_rn((double)num, 1.0 / N);  // exact (power of two)
        const double cc = __dmul_rn(cross, cross);
        if (!flat) {
          // screen with the entry's reciprocal: |cc*rcp - fl(cc/norm)| <= 4e-16*gain, so
          // when even the screened error clears best by 1e-14*(rn + gain) the
          // exact one is >= best and cannot win (ties keep the earlier index)
          const double g_est = __dmul_rn(cc, rcp);
          if (__dsub_rn(rn, g_est) > best_err[r] + 1e-14 * (rn + g_est)) continue;
        }
        const double gain = flat ? 0.0 : __ddiv_rn(cc, norm);
        const double err = fmax(__dsub_rn(rn, gain), 0.0);
        if (err < best_err[r]) {  // e, iso ascending: the first minimum stays
          best_err[r] = err;
          best_cross[r] = cross;
          best_norm[r] = norm;
          best_idx[r] = e * 8 + iso;
        }
      }
    }
  }
  // block minimum per range, lexicographic on (err, idx)
#pragma unroll
  for (int r = 0; r < kRealRanges; ++r) {
    double be = best_err[r];
    int64_t bi = best_idx[r];
    double bs = best_norm[r] == 0.0 ? 0.0 : __ddiv_rn(best_cross[r], best_norm[r]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double oe = __shfl_xor_sync(0xffffffffu, be, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const double os = __shfl_xor_sync(0xffffffffu, bs, o);
      if (oe < be || (oe == be && oi < bi)) {
        be = oe;
        bi = oi;
        bs = os;
      }
    }
    if (lane == 0) {
      red_err[warp][r] = be;
      red_idx[warp][r] = bi;
      red_s[warp][r] = bs;
    }
  }
  __syncthreads();
  if (tid < kRealRanges) {
    const int64_t m = m0 + tid;
    double be = red_err[0][tid], bs = red_s[0][tid];
    int64_t bi = red_idx[0][tid];
    for (int w = 1; w < kRealThreads / 32; ++w)
      if (red_err[w][tid] < be || (red_err[w][tid] == be && red_idx[w][tid] < bi)) {
        be = red_err[w][tid];
        bi = red_idx[w][tid];
        bs = red_s[w][tid];
      }
    if (m < M) {
      const int64_t slot = (int64_t)blockIdx.y * M + m;
      part_err[slot] = be;
      part_s[slot] = bs;
      part_idx[slot] = bi;
    }
  }
}

__global__ void real_s_merge_kernel(const double* __restrict__ part_err,
                                    const double* __restrict__ part_s,
                                    const int64_t* __restrict__ part_idx, int64_t M, int chunks,
                                    double* __restrict__ out_err, double* __restrict__ out_s,
                                    int64_t* __restrict__ out_idx) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  double be = part_err[m], bs = part_s[m];
  int64_t bi = part_idx[m];
  for (int c = 1; c < chunks; ++c) {  // chunks hold ascending entry ranges
    const double e = part_err[(int64_t)c * M + m];
    if (e < be) {
      be = e;
      bs = part_s[(int64_t)c * M + m];
      bi = part_idx[(int64_t)c * M + m];
    }
  }
  out_err[m] = be;
  out_s[m] = bs;
  out_idx[m] = bi;
}

}  // namespace

int real_s_match(Ctx* c, Level& L, int64_t M, double* d_err, double* d_s, int64_t* d_idx) {
  if (M == 0) return FC_OK;
  FC_TRY(ensure_iso_tables(c));
  // B >= 4: X on the tcgen05 contraction (fc_scan_tc.cu, tc_scan_kernel<2>);
  // this CUDA-core kernel remains for B = 2 (n = 4 < one MMA K step)
  if (L.n >= 16 && !c->real_cuda_cores) return real_tc_match(c, L, (int)(&L - c->lv) + 1, M, d_err, d_s, d_idx);
  const int64_t E = L.count;
  const int64_t gx = (M + kRealRanges - 1) / kRealRanges;
  // enough blocks for ~2 waves over the SMs; chunks of at least one entry per thread
  int64_t gy = (2 * 2 * (int64_t)c->sm_count + gx - 1) / gx;
  gy = std::max<int64_t>(1, std::min<int64_t>(gy, (E + kRealThreads - 1) / kRealThreads));
  gy = std::min<int64_t>(gy, 65535);
  const int64_t e_chunk = (E + gy - 1) / gy;
  gy = (E + e_chunk - 1) / e_chunk;
  FC_CUDA(c, c->real_part.reserve(gy * M * 24));
  double* p_err = c->real_part.as<double>();
  double* p_s = p_err + gy * M;
  int64_t* p_idx = reinterpret_cast<int64_t*>(p_s + gy * M);
  const uint16_t* inv = c->iso_inv.as<uint16_t>() + iso_table_offset(L.side);
  const dim3 grid((unsigned)gx, (unsigned)gy);
  const uint8_t* rt = c->rtiles.as<uint8_t>();
  const uint8_t* dt = L.tiles.as<uint8_t>();
  const int32_t* ds = L.sum.as<int32_t>();
  const double* dn = L.cnorm.as<double>();
  switch (L.n) {
    case 256: real_s_kernel<256><<<grid, kRealThreads, 0, c->stream>>>(rt, M, inv, dt, ds, dn, E, e_chunk, p_err, p_s, p_idx); break;
    case 64: real_s_kernel<64><<<grid, kRealThreads, 0, c->stream>>>(rt, M, inv, dt, ds, dn, E, e_chunk, p_err, p_s, p_idx); break;
    case 16: real_s_kernel<16><<<grid, kRealThreads, 0, c->stream>>>(rt, M, inv, dt, ds, dn, E, e_chunk, p_err, p_s, p_idx); break;
    case 4: real_s_kernel<4><<<grid, kRealThreads, 0, c->stream>>>(rt, M, inv, dt, ds, dn, E, e_chunk, p_err, p_s, p_idx); break;
    default: return set_error(c, FC_ERR_ARG, "unsupported range side");
  }
  FC_CUDA(c, cudaGetLastError());
  real_s_merge_kernel<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(
      p_err, p_s, p_idx, M, (int)gy, d_err, d_s, d_idx);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 2;
  return FC_OK;
}

}  // namespace fcb
