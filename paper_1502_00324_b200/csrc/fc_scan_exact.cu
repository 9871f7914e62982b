// Exact CUDA-core candidate scan (the correctness anchor and the path for
// levels/modes the tensor contraction does not take: baseline mode, 2x2
// ranges, clamp-active (range, column) pairs).
//
// Semantics follow _scan.py:14-63: for every range and candidate
// c = (e*8 + iso)*S + si the error is the exact SSD of clip(q + o, 0, 255)
// against the range; the winner is the lexicographically first minimum.
// Order independence comes from a packed key (err << 32) | c reduced with
// warp shuffles and a global atomicMin, so grid shape never changes results.
//
// Isometries are applied to the RANGE (one inverse pixel permutation per
// isometry, precomputed into shared memory) instead of copying the domain
// pool 8x as matcher.py:148-151 does:  sum_k f(iso(q)[k], r[k]) =
// sum_j f(q[j], r[src_iso^-1(j)]).
//
// Inner loop per 16 pixels of one (column, range): the clipped
// reconstruction x = clip(q + o) is formed once as packed bytes (vadd2 /
// vmaxs2 / vmins2 / byte_perm) and reused by all 8 isometries, each costing
// one broadcast LDS.128 plus 4 x (vabsdiffu4 + dp4a).
#include <cub/cub.cuh>

#include <algorithm>

#include "fc_internal.cuh"

namespace fcb {

namespace {

constexpr int kRB = 8;          // ranges per block (drop-in row kernel)
constexpr int kColsPerBlock = 128;

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__device__ __forceinline__ int rint_offset_baseline(double rmean, double s, double dmean) {
  // _scan.py:39-43: clip(round(rmean - s*dmean), 0, 255); product rounded first.
  double v = rint(__dsub_rn(rmean, __dmul_rn(s, dmean)));
  int o = (int)v;
  return o < 0 ? 0 : (o > 255 ? 255 : o);
}

template <int N>
struct ExactSmem {
  static constexpr int RB = ranges_per_block(N);
  uint8_t rperm[RB][8][N];
  int m[RB];
  double rmean[RB];
};

// One block: RB ranges (s.m[], -1 = none) x 128 columns (one per thread,
// col < 0 = none).  Every (range, column, isometry) error is exact.  The
// reduction packs (err << 3 | iso) so one 3-input min tree yields the
// first-isometry minimum per thread; the warp then takes the minimum error
// and, among the lanes holding it, the minimum candidate index (REDUX).
template <int N>
__device__ __forceinline__ void exact_block(ExactSmem<N>& s, const int16_t* __restrict__ qbase,
                                            int S, const double* __restrict__ svals,
                                            const double* __restrict__ dmean,
                                            const uint8_t* __restrict__ rtiles,
                                            const uint16_t* __restrict__ inv, int64_t col_in,
                                            int baseline, unsigned long long* __restrict__ keys) {
  constexpr int RB = ExactSmem<N>::RB;
  constexpr int CH = N >= 16 ? 16 : N;  // pixels per inner chunk
  constexpr int W = CH / 4;             // packed words per chunk
  auto& rperm = s.rperm;
  const int tid = threadIdx.x;
  for (int i = tid; i < RB * 8 * N; i += kColsPerBlock) {
    const int mm = i / (8 * N);
    const int rem = i - mm * 8 * N;
    const int iso = rem / N, j = rem - iso * N;
    const int m = s.m[mm];
    rperm[mm][iso][j] = m >= 0 ? rtiles[(int64_t)m * N + inv[iso * N + j]] : 0;
  }
  __syncthreads();

  const bool valid = col_in >= 0;
  const int64_t col = valid ? col_in : 0;
  const int64_t e = col / S;
  const int si = (int)(col - e * S);

  int o[RB];
#pragma unroll
  for (int mm = 0; mm < RB; ++mm) {
    o[mm] = baseline ? rint_offset_baseline(s.rmean[mm], svals[si], dmean[e])
                     : (int)rint(s.rmean[mm]);
  }
  unsigned acc[RB][8];
#pragma unroll
  for (int mm = 0; mm < RB; ++mm)
#pragma unroll
    for (int iso = 0; iso < 8; ++iso) acc[mm][iso] = 0u;

  const int16_t* qcol = qbase + col * N;
#pragma unroll 1
  for (int k = 0; k < N; k += CH) {
    unsigned qw[CH / 2];
    if constexpr (CH == 16) {
      const uint4 a = *reinterpret_cast<const uint4*>(qcol + k);
      const uint4 b = *reinterpret_cast<const uint4*>(qcol + k + 8);
      qw[0] = a.x; qw[1] = a.y; qw[2] = a.z; qw[3] = a.w;
      qw[4] = b.x; qw[5] = b.y; qw[6] = b.z; qw[7] = b.w;
    } else {
      const uint2 a = *reinterpret_cast<const uint2*>(qcol + k);
      qw[0] = a.x; qw[1] = a.y;
    }
#pragma unroll
    for (int mm = 0; mm < RB; ++mm) {
      const unsigned o2 = (unsigned)o[mm] | ((unsigned)o[mm] << 16);
      unsigned x4[W];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        unsigned lo = __vmins2(__vmaxs2(__vadd2(qw[2 * w], o2), 0u), 0x00ff00ffu);
        unsigned hi = __vmins2(__vmaxs2(__vadd2(qw[2 * w + 1], o2), 0u), 0x00ff00ffu);
        x4[w] = __byte_perm(lo, hi, 0x6420);
      }
#pragma unroll
      for (int iso = 0; iso < 8; ++iso) {
        unsigned a = acc[mm][iso];
        if constexpr (W == 4) {
          const uint4 r4 = *reinterpret_cast<const uint4*>(&rperm[mm][iso][k]);
          unsigned d;
          d = __vabsdiffu4(x4[0], r4.x); a = __dp4a(d, d, a);
          d = __vabsdiffu4(x4[1], r4.y); a = __dp4a(d, d, a);
          d = __vabsdiffu4(x4[2], r4.z); a = __dp4a(d, d, a);
          d = __vabsdiffu4(x4[3], r4.w); a = __dp4a(d, d, a);
        } else {
          const unsigned r4 = *reinterpret_cast<const unsigned*>(&rperm[mm][iso][k]);
          const unsigned d = __vabsdiffu4(x4[0], r4);
          a = __dp4a(d, d, a);
        }
        acc[mm][iso] = a;
      }
    }
  }
  const int lane = tid & 31;
#pragma unroll
  for (int mm = 0; mm < RB; ++mm) {
    // err <= 256 * 255^2 < 2^24, so (err << 3 | iso) fits 27 bits
    const unsigned k01 = min(acc[mm][0] << 3, (acc[mm][1] << 3) | 1u);
    const unsigned k = __vimin3_u32(__vimin3_u32(k01, (acc[mm][2] << 3) | 2u, (acc[mm][3] << 3) | 3u),
                                    __vimin3_u32((acc[mm][4] << 3) | 4u, (acc[mm][5] << 3) | 5u,
                                                 (acc[mm][6] << 3) | 6u),
                                    (acc[mm][7] << 3) | 7u);
    const unsigned err = valid ? (k >> 3) : 0xffffffffu;
    const unsigned cidx = (unsigned)((e * 8 + (k & 7)) * S + si);
    const unsigned werr = __reduce_min_sync(0xffffffffu, err);
    const unsigned wcidx = __reduce_min_sync(0xffffffffu, err == werr ? cidx : 0xffffffffu);
    if (lane == 0 && s.m[mm] >= 0 && werr != 0xffffffffu)
      atomicMin(&keys[s.m[mm]], ((unsigned long long)werr << 32) | wcidx);
  }
}

// Grid-mapped scan: blockIdx.x = 128-column chunk, blockIdx.y = block of kRB
// ranges (identity or an explicit range list), optional explicit column list.
template <int N>
__global__ void __launch_bounds__(kColsPerBlock)
scan_exact_kernel(const int16_t* __restrict__ qbase, int64_t ncols, int S,
                  const double* __restrict__ svals, const double* __restrict__ dmean,
                  const uint8_t* __restrict__ rtiles, const double* __restrict__ rmean,
                  int64_t M, const int32_t* __restrict__ d_M, const uint16_t* __restrict__ inv,
                  const int32_t* __restrict__ range_list, int64_t n_range_list, int64_t range_base,
                  const int32_t* __restrict__ col_list, int64_t n_col_list, int baseline,
                  unsigned long long* __restrict__ keys, unsigned long long* __restrict__ tspan) {
  __shared__ __align__(16) ExactSmem<N> s;
  constexpr int RB = ExactSmem<N>::RB;
  const int tid = threadIdx.x;
  if (d_M) M = *d_M;
  const int64_t nrange = range_list ? n_range_list : M;
  const int64_t r0 = range_base + (int64_t)blockIdx.y * RB;
  if (r0 >= nrange) return;  // block-uniform (device range count below the launch bound)
  if (tspan && tid == 0) atomicMin(&tspan[0], global_ns());
  if (tid < RB) {
    const int64_t idx = r0 + tid;
    int m = -1;
    if (idx < nrange) m = range_list ? range_list[idx] : (int)idx;
    s.m[tid] = m;
    s.rmean[tid] = m >= 0 ? rmean[m] : 0.0;
  }
  const int64_t ci = (int64_t)blockIdx.x * kColsPerBlock + tid;
  const int64_t ncol_eff = col_list ? n_col_list : ncols;
  const int64_t col = ci < ncol_eff ? (col_list ? (int64_t)col_list[ci] : ci) : -1;
  __syncthreads();
  exact_block<N>(s, qbase, S, svals, dmean, rtiles, inv, col, baseline, keys);
  if (tspan && tid == 0) {
    const unsigned long long t = global_ns();
    atomicMax(&tspan[1], t);
    atomicMax(&tspan[2], t);
  }
}

// Drop-in for _scan.py:14 with arbitrary candidate rows (reference layout).
__global__ void __launch_bounds__(128)
scan_rows_kernel(const int16_t* __restrict__ q, int64_t rows, int n, int S,
                 const double* __restrict__ svals, const double* __restrict__ dmean,
                 const int16_t* __restrict__ ranges, const double* __restrict__ rmean, int64_t M,
                 int baseline, unsigned long long* __restrict__ keys) {
  extern __shared__ int16_t sr[];  // [kRB][n]
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * kRB;
  for (int i = tid; i < kRB * n; i += blockDim.x) {
    const int64_t m = r0 + i / n;
    sr[i] = m < M ? ranges[m * n + (i % n)] : 0;
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + tid;
  const bool valid = c < rows;
  const int64_t e = valid ? c / (8 * S) : 0;
  const int si = valid ? (int)(c % S) : 0;
  const int lane = tid & 31;
  for (int mm = 0; mm < kRB; ++mm) {
    const int64_t m = r0 + mm;
    unsigned long long key = ~0ull;
    if (valid && m < M) {
      const int o = baseline ? rint_offset_baseline(rmean[m], svals[si], dmean[e])
                             : (int)rint(rmean[m]);
      long long err = 0;
      for (int k = 0; k < n; ++k) {
        int v = q[c * n + k] + o;
        v = v < 0 ? 0 : (v > 255 ? 255 : v);
        const int d = v - sr[mm * n + k];
        err += (long long)d * d;
      }
      if (err > 0x7fffffffLL) err = 0x7fffffffLL;
      key = ((unsigned long long)err << 32) | (unsigned long long)c;
    }
    key = warp_min_u64(key);
    if (lane == 0 && m < M && key != ~0ull) atomicMin(&keys[m], key);
  }
}

// Gather range tiles at origins and their exact moments (codec.py:164-168,
// matcher.py:171: rmean = sum / n exactly).  The range count is M, or *d_M
// when given (device-driven quadtree); hist[o] counts offsets o = rint(rmean).
__global__ void gather_kernel(const uint8_t* __restrict__ img, int width,
                              const int32_t* __restrict__ origins, int64_t M,
                              const int32_t* __restrict__ d_M, int B,
                              uint8_t* __restrict__ rtiles, double* __restrict__ rmean,
                              int32_t* __restrict__ roff, int32_t* __restrict__ rsq,
                              int32_t* __restrict__ hist) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (d_M) M = *d_M;
  if (warp >= M) return;
  const int x = origins[2 * warp], y = origins[2 * warp + 1];
  const int n = B * B;
  int s1 = 0, s2 = 0;
  for (int p = lane; p < n; p += 32) {
    const int r = p / B, col = p - r * B;
    const int v = img[(int64_t)(y + r) * width + x + col];
    rtiles[warp * n + p] = (uint8_t)v;
    s1 += v;
    s2 += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    const double mean = __ddiv_rn((double)s1, (double)n);
    const int o = (int)rint(mean);
    rmean[warp] = mean;
    roff[warp] = o;
    rsq[warp] = s2;
    if (hist) atomicAdd(&hist[o], 1);
  }
}

__global__ void roff_hist_kernel(const int32_t* __restrict__ roff, int64_t M,
                                 int32_t* __restrict__ hist) {
  __shared__ int32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[roff[i]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Moments of explicitly supplied range tiles (fc_match_tiles).
__global__ void range_moments_kernel(const uint8_t* __restrict__ rtiles, int64_t M, int n,
                                     double* __restrict__ rmean, int32_t* __restrict__ roff,
                                     int32_t* __restrict__ rsq) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= M) return;
  int s1 = 0, s2 = 0;
  for (int p = lane; p < n; p += 32) {
    const int v = rtiles[warp * n + p];
    s1 += v;
    s2 += v * v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    const double mean = __ddiv_rn((double)s1, (double)n);
    rmean[warp] = mean;
    roff[warp] = (int)rint(mean);
    rsq[warp] = s2;
  }
}

// q base operand: column (e, si) -> rint(s*(d - mean)) or rint(s*d)
// (matcher.py:143-152), LPC lanes per column with PPL pixels each (coalesced
// 8/16-byte loads and stores).  With `stats` it also emits the tensor-path
// column statistics {Q1 = sum q, Q2 = sum q^2, qmin, qmax}, the parity flag
// and the qmin / qmax histograms (fc_scan_tc.cu).
struct QLevel {
  const uint8_t* tiles;
  const double* mean;
  const double* svals;
  int16_t* q;
  int4* col_stats;
  int32_t* odd;
  unsigned* hist;       // qmin | qmax | q2max (block-aggregated), stats levels only
  int32_t* chunk_odd;   // odd columns per 1024-column chunk, stats levels only
  int4* bconst;         // baseline stats levels: tensor-epilogue column constants
  int64_t ncols;
  int S, n, baseline, stats, shift;
  int block_begin, nblocks;
};
struct QParams {
  QLevel lv[4];
  int n_levels;
};

// q base operand: column (e, si) -> rint(s*(d - mean)) or rint(s*d)
// (matcher.py:143-152), LPC lanes per column with PPL pixels each (coalesced
// 8/16-byte loads and stores).  Stats levels also emit the tensor-path column
// statistics {Q1 = sum q, Q2 = sum q^2, qmin, qmax}, the parity flag, the
// qmin / qmax histograms and the per-chunk parity counts.
template <int N>
__device__ __forceinline__ void qprep_level(const QLevel& L, int block, unsigned* sh) {
  constexpr int LPC = N >= 8 ? N / 8 : 1;
  constexpr int PPL = N / LPC;
  const int S = L.S;
  const int64_t ncols = L.ncols;
  const int stats = L.stats;
  if (stats) {
    for (int i = threadIdx.x; i < 2049; i += blockDim.x) sh[i] = 0;
    __syncthreads();
  }
  const int64_t total = ncols * LPC;
  const int64_t stride = (int64_t)L.nblocks * blockDim.x;
  const int lane = threadIdx.x & 31;
  // every lane of a warp runs the same trip count (shuffles below)
  for (int64_t base = (int64_t)block * blockDim.x; base < total; base += stride) {
    const int64_t t = base + threadIdx.x;
    const int64_t col = t / LPC;
    const int part = (int)(t - col * LPC);
    const bool valid = col < ncols;
    int s1 = 0, s2 = 0, lo = 1 << 20, hi = -(1 << 20);
    if (valid) {
      const int64_t e = col / S;
      const int si = (int)(col - e * S);
      const double sv = L.svals[si];
      const double dm = L.mean[e];
      const uint8_t* src = L.tiles + e * N + part * PPL;
      uint8_t px[PPL];
      if constexpr (PPL == 8) {
        *reinterpret_cast<uint2*>(px) = *reinterpret_cast<const uint2*>(src);
      } else {
        *reinterpret_cast<uint32_t*>(px) = *reinterpret_cast<const uint32_t*>(src);
      }
      int16_t qv[PPL];
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const double d = (double)px[k];
        const double x = L.baseline ? d : __dsub_rn(d, dm);
        const int v = (int)rint(__dmul_rn(sv, x));
        qv[k] = (int16_t)v;
        s1 += v;
        s2 += v * v;
        lo = min(lo, v);
        hi = max(hi, v);
      }
      int16_t* dst = L.q + col * N + part * PPL;
      if constexpr (PPL == 8) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(qv);
      } else {
        *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(qv);
      }
    }
    if (!stats) continue;
#pragma unroll
    for (int o = 1; o < LPC; o <<= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const bool lead = valid && part == 0;
    if (lead && L.baseline) {
      // baseline mode (u8 x u8 contraction, fc_scan_tc.cu): the epilogue forms
      // o = clip(rint(rmean - s*dmean), 0, 255) per (range, column) from the
      // range sum R1 with integer ops.  With V = n * fl(s * dmean) (exact,
      // n a power of two) the reference's fp64 rmean - s*dmean equals
      // (R1 - V) / n exactly, so rint is floor((R1 + W') / n) with
      // W' = floor(n/2 - V) when V is not an integer, and round-half-even
      // (R1 + W' + ((R1 - V) >> shift & 1)) >> shift with W' = n/2 - 1 - V
      // (tie mask set) when it is.  Clamping (q + o > 255) needs o >= 256 -
      // qmax, i.e. a range sum from about V + n (256 - qmax) - n/2 on: the
      // column's clamp bucket b = floor(R1_min / n), rounded DOWN so the
      // correction lists only ever over-include (an exactly evaluated pair
      // is exact either way).  The bucket rides in the qmax slot as 256 - b
      // so the proposed-mode reach tables apply unchanged (qmin slot 0:
      // q + o never drops below 0).
      const int64_t e = col / S;
      const int si = (int)(col - e * S);
      const double V = __dmul_rn(L.svals[si], L.mean[e]) * (double)L.n;
      const int half = L.n >> 1;
      const bool whole = floor(V) == V;
      const int W = whole ? half - 1 - (int)V : (int)floor((double)half - V);
      int bucket = 256;
      if (hi > 0) {
        const double X = V + (double)(L.n * (256 - hi) - half);
        long long A = (long long)floor(X) - 1;
        if (A < 0) A = 0;
        if (A <= 255ll * L.n) bucket = (int)(A >> L.shift);
      }
      L.col_stats[col] = make_int4(s1, s2, 0, 256 - bucket);
      L.bconst[col] = make_int4(W, 2 * s1, s2, whole ? -1 : 0);
      L.odd[col] = 0;  // no parity groups: columns stay in candidate order
      atomicAdd(&sh[512], 1u);
      atomicAdd(&sh[1024 + 256 - bucket + 512], 1u);
      atomicMax(&sh[2048], (unsigned)s2);
    } else if (lead) {
      L.col_stats[col] = make_int4(s1, s2, lo, hi);
      L.odd[col] = s2 & 1;  // == s1 & 1
      atomicAdd(&sh[lo + 512], 1u);
      atomicAdd(&sh[1024 + hi + 512], 1u);
      atomicMax(&sh[2048], (unsigned)s2);
    }
    // a warp's columns never straddle a 1024-column chunk (32 / LPC divides 1024)
    const unsigned oddb = __ballot_sync(0xffffffffu, lead && !L.baseline && (s2 & 1));
    if (lane == 0 && oddb) {
      const int64_t col0 = (base + (threadIdx.x & ~31)) / LPC;
      atomicAdd(&L.chunk_odd[col0 >> 10], __popc(oddb));
    }
  }
  if (!stats) return;
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (sh[i]) atomicAdd(&L.hist[i], sh[i]);
  if (threadIdx.x == 0) atomicMax(&L.hist[2048], sh[2048]);
}

__global__ void __launch_bounds__(256) qprep_multi_kernel(QParams P) {
  __shared__ unsigned sh[2048 + 1];
  int l = 0;
  for (int k = 1; k < P.n_levels; ++k)
    if ((int)blockIdx.x >= P.lv[k].block_begin) l = k;
  const QLevel& L = P.lv[l];
  const int block = blockIdx.x - L.block_begin;
  switch (L.n) {
    case 256: qprep_level<256>(L, block, sh); break;
    case 64: qprep_level<64>(L, block, sh); break;
    case 16: qprep_level<16>(L, block, sh); break;
    default: qprep_level<4>(L, block, sh); break;
  }
}

// Parity slots: odd_prefix[col] = #odd columns before col (exclusive scan of
// the parity flags, in column order), one 1024-column chunk per block; the
// chunk's base sums the per-chunk counts qprep produced.  The last chunk of a
// level stores the level's odd total next to its histograms.
struct SlotLevel {
  const int32_t* odd;
  int32_t* odd_prefix;
  const int32_t* chunk_odd;
  unsigned* n_odd_out;
  int64_t ncols;
  int chunk_begin;
};
struct SlotParams {
  SlotLevel lv[4];
  int n_levels;
};
__global__ void __launch_bounds__(1024) parity_slot_kernel(SlotParams P) {
  using Scan = cub::BlockScan<int, 1024>;
  using Red = cub::BlockReduce<int, 1024>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ typename Red::TempStorage red_tmp;
  int l = 0;
  for (int k = 1; k < P.n_levels; ++k)
    if ((int)blockIdx.x >= P.lv[k].chunk_begin) l = k;
  const SlotLevel& L = P.lv[l];
  const int chunk = blockIdx.x - L.chunk_begin;
  int part = 0;
  for (int k = threadIdx.x; k < chunk; k += blockDim.x) part += L.chunk_odd[k];
  const int base = Red(red_tmp).Sum(part);
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = base;
  __syncthreads();
  const int64_t col = (int64_t)chunk * 1024 + threadIdx.x;
  const int f = col < L.ncols ? L.odd[col] : 0;
  int excl, agg;
  Scan(scan_tmp).ExclusiveSum(f, excl, agg);
  if (col < L.ncols) L.odd_prefix[col] = s_base + excl;
  if (threadIdx.x == 0 && (int64_t)(chunk + 1) * 1024 >= L.ncols) *L.n_odd_out = s_base + agg;
}

__global__ void decode_keys_kernel(const unsigned long long* __restrict__ keys, int64_t M,
                                   int64_t* __restrict__ err, int64_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const unsigned long long k = keys[i];
  err[i] = (int64_t)(k >> 32);
  idx[i] = (int64_t)(k & 0xffffffffull);
}

}  // namespace

int iso_table_offset(int side) {
  return side == 16 ? 0 : side == 8 ? 8 * 256 : side == 4 ? 8 * (256 + 64) : 8 * (256 + 64 + 16);
}

// Inverse isometry maps per range side, packed [side][8][n]:
// inv[iso][j] = output pixel k with src_iso(k) = j, where out[k] = t[src_iso(k)]
// restates apply_isometry (image.py:140-155).
int ensure_iso_tables(Ctx* c) {
  if (c->iso_ready) return FC_OK;
  std::vector<uint16_t> h(8 * (256 + 64 + 16 + 4), 0);
  const int sides[4] = {16, 8, 4, 2};
  for (int s = 0; s < 4; ++s) {
    const int B = sides[s], b = B - 1, n = B * B;
    uint16_t* t = h.data() + iso_table_offset(B);
    for (int iso = 0; iso < 8; ++iso) {
      for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j) {
          int r = 0, cc = 0;  // out[i][j] = t[r][cc]
          switch (iso) {
            case 0: r = i; cc = j; break;
            case 1: r = b - j; cc = i; break;
            case 2: r = b - i; cc = b - j; break;
            case 3: r = j; cc = b - i; break;
            case 4: r = i; cc = b - j; break;
            case 5: r = j; cc = i; break;
            case 6: r = b - i; cc = j; break;
            default: r = b - j; cc = b - i; break;
          }
          t[iso * n + r * B + cc] = (uint16_t)(i * B + j);
        }
    }
  }
  FC_CUDA(c, c->iso_inv.reserve(h.size() * 2));
  FC_TRY(stage_h2d(c, c->iso_inv.ptr, h.data(), h.size() * 2));
  c->iso_ready = true;
  return FC_OK;
}

// Device half of the operand preparation for several levels at once:
// s values, q operands (+ tensor-path statistics for `stats` levels: the
// qmin / qmax histograms, max Q2 and odd total in c->prep_dev, which
// tc_tables_kernel turns into the level's tables on the device), parity slots.
int prep_launch(Ctx* c, Level* const* levels, const int* stats, int count) {
  QParams QP{};
  SlotParams SP{};
  int qblocks = 0, chunks = 0, any_stats = 0;
  int64_t chunk_total = 0;
  for (int i = 0; i < count; ++i)
    if (stats[i]) chunk_total += (levels[i]->count * levels[i]->s_count + 1023) / 1024;
  // one buffer (one memset): the levels' histograms, then the chunk parity counts
  FC_CUDA(c, c->prep_dev.reserve(kLevels * kTcHistWords * 4 + chunk_total * 4 + 64));
  int32_t* chunk_odd = c->prep_dev.as<int32_t>() + kLevels * kTcHistWords;
  for (int i = 0; i < count; ++i) {
    Level& L = *levels[i];
    const int li = (int)(&L - c->lv);
    const int64_t cols = L.count * L.s_count;
    FC_CUDA(c, L.qbase.reserve(cols * L.n * 2 + 64));
    FC_CUDA(c, L.svals_d.reserve(kMaxS * 8));
    // the s values change rarely: upload only when they (or the buffer) did
    if (L.svals_up_ptr != L.svals_d.ptr || L.svals_up_count != L.s_count ||
        memcmp(L.svals_up, L.svals, L.s_count * 8) != 0) {
      FC_TRY(stage_h2d(c, L.svals_d.ptr, L.svals, L.s_count * 8));
      memcpy(L.svals_up, L.svals, L.s_count * 8);
      L.svals_up_count = L.s_count;
      L.svals_up_ptr = L.svals_d.ptr;
    }
    TcOperands& T = L.tc;
    if (stats[i]) {
      FC_CUDA(c, T.col_stats.reserve(cols * 16 + 16));
      FC_CUDA(c, T.odd.reserve(cols * 8 + 16));
      // padded to whole 256-column tiles: the epilogue stages a tile's constants unconditionally
      if (L.baseline) FC_CUDA(c, T.bconst.reserve(((cols + 255) / 256 + 1) * 256 * 16));
      T.ncols = cols;
      any_stats = 1;
    }
    if (cols == 0) continue;
    QLevel& Q = QP.lv[QP.n_levels++];
    Q.tiles = L.tiles.as<uint8_t>();
    Q.mean = L.mean.as<double>();
    Q.svals = L.svals_d.as<double>();
    Q.q = L.qbase.as<int16_t>();
    Q.col_stats = T.col_stats.as<int4>();
    Q.odd = T.odd.as<int32_t>();
    Q.hist = c->prep_dev.as<unsigned>() + li * kTcHistWords;
    Q.chunk_odd = chunk_odd + chunks;
    Q.ncols = cols;
    Q.S = L.s_count;
    Q.n = L.n;
    Q.baseline = L.baseline;
    Q.stats = stats[i];
    Q.bconst = L.baseline && stats[i] ? T.bconst.as<int4>() : nullptr;
    Q.shift = L.n == 256 ? 8 : L.n == 64 ? 6 : L.n == 16 ? 4 : 2;
    const int lpc = L.n >= 8 ? L.n / 8 : 1;
    // full occupancy (8 blocks of 256 per SM): the loop is load-latency bound
    Q.nblocks = (int)std::min<int64_t>((cols * lpc + 255) / 256, c->sm_count * 8);
    Q.block_begin = qblocks;
    qblocks += Q.nblocks;
    if (stats[i]) {
      SlotLevel& Sl = SP.lv[SP.n_levels++];
      Sl.odd = T.odd.as<int32_t>();
      Sl.odd_prefix = T.odd.as<int32_t>() + cols;
      Sl.chunk_odd = Q.chunk_odd;
      Sl.n_odd_out = c->prep_dev.as<unsigned>() + li * kTcHistWords + 2049;
      Sl.ncols = cols;
      Sl.chunk_begin = chunks;
      chunks += (int)((cols + 1023) / 1024);
    }
  }
  if (any_stats) {
    FC_CUDA(c, cudaMemsetAsync(c->prep_dev.ptr, 0, kLevels * kTcHistWords * 4 + chunk_total * 4 + 4,
                               c->stream));
  }
  if (qblocks > 0) {
    qprep_multi_kernel<<<qblocks, 256, 0, c->stream>>>(QP);
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
  }
  if (chunks > 0) {
    parity_slot_kernel<<<chunks, 1024, 0, c->stream>>>(SP);
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
  }
  return FC_OK;
}

int reserve_ranges(Ctx* c, Level& L, int64_t M) {
  FC_CUDA(c, c->rtiles.reserve(M * L.n + 64));
  FC_CUDA(c, c->rmean.reserve(M * 8 + 64));
  FC_CUDA(c, c->roff.reserve(M * 4 + 64));
  FC_CUDA(c, c->rsq.reserve(M * 4 + 64));
  return FC_OK;
}

int gather_ranges(Ctx* c, Level& L, const int32_t* d_origins, int64_t M) {
  FC_TRY(reserve_ranges(c, L, M));
  if (M == 0) return FC_OK;
  const int threads = 256;
  gather_kernel<<<(unsigned)((M * 32 + threads - 1) / threads), threads, 0, c->stream>>>(
      c->img_ptr, c->width, d_origins, M, nullptr, L.side, c->rtiles.as<uint8_t>(),
      c->rmean.as<double>(), c->roff.as<int32_t>(), c->rsq.as<int32_t>(), nullptr);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;
  return FC_OK;
}

int gather_ranges_dev(Ctx* c, Level& L, const int32_t* d_origins, const int32_t* d_M,
                      int64_t M_bound, int32_t* d_hist) {
  FC_TRY(reserve_ranges(c, L, M_bound));
  if (M_bound == 0) return FC_OK;
  const int threads = 256;
  gather_kernel<<<(unsigned)((M_bound * 32 + threads - 1) / threads), threads, 0, c->stream>>>(
      c->img_ptr, c->width, d_origins, M_bound, d_M, L.side, c->rtiles.as<uint8_t>(),
      c->rmean.as<double>(), c->roff.as<int32_t>(), c->rsq.as<int32_t>(), d_hist);
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 1;
  return FC_OK;
}

int roff_hist(Ctx* c, int64_t M, int32_t* d_hist) {
  FC_CUDA(c, cudaMemsetAsync(d_hist, 0, 256 * 4, c->stream));
  if (M == 0) return FC_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((M + 255) / 256, c->sm_count);
  roff_hist_kernel<<<grid, 256, 0, c->stream>>>(c->roff.as<int32_t>(), M, d_hist);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;
  return FC_OK;
}

int load_ranges(Ctx* c, Level& L, const uint8_t* h_tiles, int64_t M) {
  FC_TRY(reserve_ranges(c, L, M));
  if (M == 0) return FC_OK;
  FC_TRY(stage_h2d(c, c->rtiles.ptr, h_tiles, M * L.n));
  const int threads = 256;
  range_moments_kernel<<<(unsigned)((M * 32 + threads - 1) / threads), threads, 0, c->stream>>>(
      c->rtiles.as<uint8_t>(), M, L.n, c->rmean.as<double>(), c->roff.as<int32_t>(),
      c->rsq.as<int32_t>());
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;
  return FC_OK;
}

int scan_exact(Ctx* c, Level& L, int64_t M, const int32_t* d_range_list, int64_t n_range_list,
               const int32_t* d_col_list, int64_t n_col_list, uint64_t* d_keys,
               const int32_t* d_M, unsigned long long* d_time) {
  FC_TRY(ensure_iso_tables(c));
  const int64_t ncols = L.count * L.s_count;
  const int64_t nr = d_range_list ? n_range_list : M;
  const int64_t nc = d_col_list ? n_col_list : ncols;
  if (nr == 0 || nc == 0) return FC_OK;
  const double* d_s = L.svals_d.as<double>();
  const uint16_t* inv = c->iso_inv.as<uint16_t>() + iso_table_offset(L.side);
  auto* keys = reinterpret_cast<unsigned long long*>(d_keys);
  const unsigned gx = (unsigned)((nc + kColsPerBlock - 1) / kColsPerBlock);
  const int RB = ranges_per_block(L.n);
  const int64_t slab = 65535LL * RB;
  for (int64_t base = 0; base < nr; base += slab) {
    const int64_t cnt = std::min<int64_t>(slab, nr - base);
    dim3 grid(gx, (unsigned)((cnt + RB - 1) / RB));
    const int64_t nlist = d_range_list ? n_range_list : M;
#define FC_LAUNCH_EXACT(NN)                                                                     \
    FC_CUDA(c, launch_k(c, scan_exact_kernel<NN>, grid, dim3(kColsPerBlock), 0,                 \
        L.qbase.as<int16_t>(), ncols, L.s_count, d_s, L.mean.as<double>(),                      \
        c->rtiles.as<uint8_t>(), c->rmean.as<double>(), nlist, d_M, inv, d_range_list,          \
        n_range_list,                                                                           \
        base, d_col_list, n_col_list, L.baseline, keys, d_time))
    switch (L.n) {
      case 256: FC_LAUNCH_EXACT(256); break;
      case 64: FC_LAUNCH_EXACT(64); break;
      case 16: FC_LAUNCH_EXACT(16); break;
      default: FC_LAUNCH_EXACT(4); break;
    }
#undef FC_LAUNCH_EXACT
    FC_CUDA(c, cudaGetLastError());
    c->stats.kernel_launches += 1;
  }
  return FC_OK;
}

int decode_keys(Ctx* c, const uint64_t* d_keys, int64_t M, int64_t* d_err, int64_t* d_idx) {
  if (M == 0) return FC_OK;
  decode_keys_kernel<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(
      reinterpret_cast<const unsigned long long*>(d_keys), M, d_err, d_idx);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;
  return FC_OK;
}

int scan_rows_dropin(Ctx* c, const int16_t* ranges, const double* rmeans, int64_t M, int32_t n,
                     const int16_t* q, const double* dmeans, int64_t E, const double* svals,
                     int32_t S, int32_t baseline, int64_t* out_err, int64_t* out_idx) {
  if (M == 0) return FC_OK;
  const int64_t rows = E * 8 * S;
  DevBuf dq, dr, drm, ddm, ds, dk, de, di;
  auto cleanup = [&]() {
    dq.release(); dr.release(); drm.release(); ddm.release(); ds.release(); dk.release();
    de.release(); di.release();
  };
  cudaError_t e = cudaSuccess;
  if ((e = dq.reserve(rows * n * 2 + 16)) || (e = dr.reserve(M * n * 2 + 16)) ||
      (e = drm.reserve(M * 8 + 16)) || (e = ddm.reserve(E * 8 + 16)) || (e = ds.reserve(S * 8 + 16)) ||
      (e = dk.reserve(M * 8 + 16)) || (e = de.reserve(M * 8 + 16)) || (e = di.reserve(M * 8 + 16))) {
    cleanup();
    return cuda_check(c, e, "scan_rows_dropin alloc");
  }
  cudaStream_t s = c->stream;
  cudaMemcpyAsync(dq.ptr, q, rows * n * 2, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dr.ptr, ranges, M * n * 2, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(drm.ptr, rmeans, M * 8, cudaMemcpyHostToDevice, s);
  if (E) cudaMemcpyAsync(ddm.ptr, dmeans, E * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(ds.ptr, svals, S * 8, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(dk.ptr, 0xff, M * 8, s);
  if (rows > 0) {
    dim3 grid((unsigned)((rows + 127) / 128), (unsigned)((M + kRB - 1) / kRB));
    scan_rows_kernel<<<grid, 128, kRB * n * 2, s>>>(
        dq.as<int16_t>(), rows, n, S, ds.as<double>(), ddm.as<double>(), dr.as<int16_t>(),
        drm.as<double>(), M, baseline, dk.as<unsigned long long>());
  }
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    decode_keys_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(
        dk.as<unsigned long long>(), M, de.as<int64_t>(), di.as<int64_t>());
    cudaMemcpyAsync(out_err, de.ptr, M * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(out_idx, di.ptr, M * 8, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
  }
  cleanup();
  if (e != cudaSuccess) return cuda_check(c, e, "scan_rows_dropin");
  if (rows == 0) {
    for (int64_t i = 0; i < M; ++i) { out_err[i] = (int64_t)1 << 62; out_idx[i] = -1; }
  }
  return FC_OK;
}

}  // namespace fcb
