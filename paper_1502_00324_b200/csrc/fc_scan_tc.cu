// tcgen05 int8 contraction for the exhaustive range-domain search (proposed
// mode, range sides 16 / 8 / 4).  Replaces the inner loops of
// _scan.py:29-61 for every (range, domain, isometry, s) candidate.
//
// Algebra (per range m with offset o = rint(rmean), candidate column
// c = (e, si) with base operand q = rint(s*(d - dmean)), isometry iso applied
// to the range as a pixel permutation r_iso):
//     err = sum_k (q_k + o - r_iso,k)^2                    (no clamping)
//         = Q2_c + 2 o Q1_c - 2 <q_c, r_iso> + R_m ,  R_m = sum (r - o)^2
// The tensor cores produce acc = <-q_c, r_iso> (u8 range x s8 operand, s32
// accumulate, K = B*B, 1 or 2 s8 planes).  Columns are sorted by Q1 so one
// 256-column tile has a single Q1 and o*Q1 is a per-row constant; with
// hq = floor(Q2 / 2), par = Q2 & 1:
//     kh = acc + hq_c + o*Q1_tile,   err - R_m = 2*kh + par_c.
// The epilogue keeps, per TMEM lane (row = (range, iso)), the running min of
// (acc + hq) with one VIADDMNMX per element and rescans a tile exactly only
// when its minimum can reach the row's current best (ties included, since
// candidate order is restored from the packed key (err << 32) | c).
//
// Clamping: the GEMM error is exact unless some pixel of q + o leaves
// [0, 255]; it is then an UPPER bound of the true error for the SAME
// candidate index, so keeping it in the argmin is harmless as long as every
// clamp-active (range, column) pair is ALSO evaluated exactly.  The host
// buckets ranges by o and launches the exact CUDA-core kernel on the columns
// whose qmin < -o or qmax > 255 - o (prefixes of two sorted column lists).
//
// Kernel layout: persistent, one CTA per SM, 12 warps:
//   warp 0  producer: cp.async.bulk (TMA engine) of the A row tiles and the
//           B column tiles + per-column hq/meta into a STAGES-deep ring
//   warp 1  MMA issuer: one elected lane issues tcgen05.mma.kind::i8
//           (M=128, N=256, K=32 per instruction) into one of two TMEM
//           accumulators (2 x 256 columns = all 512 TMEM columns)
//   warp 2  TMEM allocator
//   warps 4..11 epilogue: tcgen05.ld 32x32b, VIADDMNMX running minimum,
//           exact rescans, per-range atomicMin of packed keys
#include <cub/cub.cuh>

#include <algorithm>

#include "fc_internal.cuh"
#include "fc_tc_ptx.cuh"

namespace fcb {
namespace {

constexpr int kTileN = 256;
constexpr int kTileM = 128;
constexpr int kEpiWarps = 8;
constexpr int kThreads = (4 + kEpiWarps) * 32;
constexpr int kPadHq = 1 << 30;
constexpr int kThrInit = 1 << 29;

struct TcParams {
  const uint8_t* a_tiles;   // [rt_pad][128 * kpad]
  const int4* row_meta;     // [rt_pad * 128] {o, R, m, unused}
  const int8_t* b_tiles;    // [ntiles][256 * kpad]
  const int32_t* hq;        // [ntiles * 256]
  const uint32_t* meta;     // [ntiles * 256]
  const int2* tile_info;    // [ntiles] {Q1 of the tile, smallest column index in the tile}
  unsigned long long* keys; // [M]
  unsigned long long* rescans;  // statistics: warp rescans
  int S;
  int n_rgroups;
  int ntiles;
  int tiles_per_unit;
  int64_t n_units;
};

template <int KPAD, int RG, int STAGES>
struct TcLayout {
  static constexpr uint32_t kABytes = RG * kTileM * KPAD;
  static constexpr uint32_t kBBytes = kTileN * KPAD;
  static constexpr uint32_t kStageBytes = kBBytes + 2 * kTileN * 4;
  static constexpr uint32_t kBarOff = kABytes + STAGES * kStageBytes;
  static constexpr uint32_t kNumBars = 2 * STAGES + 6;
  // + alignment slack; >= 116 KB so only one CTA (which owns all 512 TMEM
  // columns) is ever resident per SM
  static constexpr uint32_t kSmemRaw = kBarOff + kNumBars * 8 + 16 + 1024;
  static constexpr uint32_t kSmem = kSmemRaw < 116 * 1024 ? 116 * 1024 : kSmemRaw;
};

// Exact re-evaluation of one 128-column half tile for the 32 rows of a warp
// (rare: only when the fast pass shows the tile can reach a row's best).
// Returns the row's best packed key, min-shared over its 8 isometry lanes.
__device__ __noinline__ unsigned long long rescan_half(uint32_t taddr, const int* hq_s,
                                                       const uint32_t* meta_s, int oq, int thr,
                                                       int Rm, bool need, int S, int iso,
                                                       unsigned long long b) {
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    int v[32];
    ptx::tmem_ld32(taddr + c * 32, v);
    ptx::tmem_wait_ld();
    if (need) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int kh = v[j] + hq_s[c * 32 + j] + oq;
        if (kh <= thr) {
          const uint32_t mt = meta_s[c * 32 + j];
          const int col = (int)(mt & 0x7fffffffu);
          const long long err = 2LL * kh + (long long)(mt >> 31) + Rm;
          const int e_idx = col / S, si = col - e_idx * S;
          const unsigned long long cidx = (unsigned long long)((e_idx * 8 + iso) * S + si);
          const unsigned long long key = ((unsigned long long)err << 32) | cidx;
          b = key < b ? key : b;
        }
      }
    }
  }
  unsigned long long w = __shfl_xor_sync(0xffffffffu, b, 1);
  b = w < b ? w : b;
  w = __shfl_xor_sync(0xffffffffu, b, 2);
  b = w < b ? w : b;
  w = __shfl_xor_sync(0xffffffffu, b, 4);
  b = w < b ? w : b;
  return b;
}

template <int KPAD, int RG, int STAGES>
__global__ void __launch_bounds__(kThreads, 1) tc_scan_kernel(const TcParams p) {
  using Lay = TcLayout<KPAD, RG, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sStage = smem + Lay::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::kBarOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Lay::kNumBars);
  const uint32_t bar_base = ptx::smem_u32(bars);
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + 2 + b); };
  const uint32_t afull_bar = bar_base + 8u * (2 * STAGES + 4);
  const uint32_t aempty_bar = bar_base + 8u * (2 * STAGES + 5);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 1);
      ptx::mbar_init(empty_bar(s), 1 + kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(tfull_bar(b), 1);
      ptx::mbar_init(tempty_bar(b), kEpiWarps);
    }
    ptx::mbar_init(afull_bar, 1);
    ptx::mbar_init(aempty_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_rg = p.n_rgroups;
  const int CT = p.tiles_per_unit;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      uint32_t L = 0, U = 0;
      for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++U) {
        const int g = (int)(u % n_rg);
        const int t0 = (int)(u / n_rg) * CT;
        const int t1 = min(p.ntiles, t0 + CT);
        ptx::mbar_wait(aempty_bar, (U & 1) ^ 1);
        ptx::mbar_expect_tx(afull_bar, Lay::kABytes);
        ptx::bulk_g2s(ptx::smem_u32(sA), p.a_tiles + (size_t)g * Lay::kABytes, Lay::kABytes,
                      afull_bar);
        for (int t = t0; t < t1; ++t, ++L) {
          const int s = L % STAGES;
          ptx::mbar_wait(empty_bar(s), ((L / STAGES) & 1) ^ 1);
          uint8_t* st = sStage + s * Lay::kStageBytes;
          ptx::mbar_expect_tx(full_bar(s), Lay::kStageBytes);
          ptx::bulk_g2s(ptx::smem_u32(st), p.b_tiles + (size_t)t * Lay::kBBytes, Lay::kBBytes,
                        full_bar(s));
          ptx::bulk_g2s(ptx::smem_u32(st + Lay::kBBytes), p.hq + (size_t)t * kTileN, kTileN * 4,
                        full_bar(s));
          ptx::bulk_g2s(ptx::smem_u32(st + Lay::kBBytes + kTileN * 4), p.meta + (size_t)t * kTileN,
                        kTileN * 4, full_bar(s));
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t kIdesc = ptx::idesc_i8(kTileM, kTileN);
    uint32_t L = 0, T = 0, U = 0;
    for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x, ++U) {
      const int t0 = (int)(u / n_rg) * CT;
      const int t1 = min(p.ntiles, t0 + CT);
      ptx::mbar_wait(afull_bar, U & 1);
      ptx::tc_fence_after();
      for (int t = t0; t < t1; ++t, ++L) {
        const int s = L % STAGES;
        ptx::mbar_wait(full_bar(s), (L / STAGES) & 1);
        ptx::tc_fence_after();
        const uint32_t b_addr = ptx::smem_u32(sStage + s * Lay::kStageBytes);
#pragma unroll 1
        for (int r = 0; r < RG; ++r, ++T) {
          const int buf = T & 1;
          ptx::mbar_wait(tempty_bar(buf), ((T >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = ptx::smem_u32(sA) + r * (kTileM * KPAD);
#pragma unroll
            for (int ks = 0; ks < KPAD / 32; ++ks) {
              const uint64_t ad = ptx::umma_desc(a_addr + ks * 2 * (kTileM * 16), kTileM * 16, 128);
              const uint64_t bd = ptx::umma_desc(b_addr + ks * 2 * (kTileN * 16), kTileN * 16, 128);
              ptx::umma_i8(tmem_base + buf * kTileN, ad, bd, kIdesc, ks > 0 ? 1u : 0u);
            }
            ptx::umma_commit(tfull_bar(buf));
          }
          __syncwarp();
        }
        if (lane == 0) ptx::umma_commit(empty_bar(s));
        __syncwarp();
      }
      if (lane == 0) ptx::umma_commit(aempty_bar);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int e = warp - 4;
    const int sp = warp & 3;     // TMEM sub-partition this warp may access
    const int half = e >> 2;     // column half of the 256-wide tile
    const int row = sp * 32 + lane;
    const int S = p.S;
    uint32_t L = 0, T = 0;
    for (int64_t u = blockIdx.x; u < p.n_units; u += gridDim.x) {
      const int g = (int)(u % n_rg);
      const int t0 = (int)(u / n_rg) * CT;
      const int t1 = min(p.ntiles, t0 + CT);
      // per row-tile state (dynamically indexed -> local memory, touched once per tile)
      int thr[RG], tie_e[RG];
      unsigned long long best[RG];
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        thr[r] = kThrInit;
        tie_e[r] = 0x7fffffff;
        best[r] = ~0ull;
      }
      for (int t = t0; t < t1; ++t, ++L) {
        const int s = L % STAGES;
        ptx::mbar_wait(full_bar(s), (L / STAGES) & 1);
        const uint8_t* st = sStage + s * Lay::kStageBytes;
        const int* hq_s = reinterpret_cast<const int*>(st + Lay::kBBytes) + half * 128;
        const uint32_t* meta_s =
            reinterpret_cast<const uint32_t*>(st + Lay::kBBytes + kTileN * 4) + half * 128;
        const int2 tinfo = p.tile_info[t];
        const int q1 = tinfo.x;
        const int tile_e = tinfo.y / S;
#pragma unroll 1
        for (int r = 0; r < RG; ++r, ++T) {
          const int4 rm = p.row_meta[(size_t)(g * RG + r) * kTileM + row];  // {o, R, m, -}
          const int buf = T & 1;
          ptx::mbar_wait(tfull_bar(buf), (T >> 1) & 1);
          ptx::tc_fence_after();
          const uint32_t taddr =
              tmem_base + ((uint32_t)(sp * 32) << 16) + buf * kTileN + half * 128;
          const int oq = rm.x * q1;
          int m0 = 0x7fffffff, m1 = 0x7fffffff, m2 = 0x7fffffff, m3 = 0x7fffffff;
#pragma unroll
          for (int c = 0; c < 4; c += 2) {
            int va[32], vb[32];
            ptx::tmem_ld32(taddr + c * 32, va);
            ptx::tmem_ld32(taddr + (c + 1) * 32, vb);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const int4 h = *reinterpret_cast<const int4*>(hq_s + c * 32 + j);
              m0 = __viaddmin_s32(va[j], h.x, m0);
              m1 = __viaddmin_s32(va[j + 1], h.y, m1);
              m2 = __viaddmin_s32(va[j + 2], h.z, m2);
              m3 = __viaddmin_s32(va[j + 3], h.w, m3);
            }
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const int4 h = *reinterpret_cast<const int4*>(hq_s + (c + 1) * 32 + j);
              m0 = __viaddmin_s32(vb[j], h.x, m0);
              m1 = __viaddmin_s32(vb[j + 1], h.y, m1);
              m2 = __viaddmin_s32(vb[j + 2], h.z, m2);
              m3 = __viaddmin_s32(vb[j + 3], h.w, m3);
            }
          }
          // a tile can improve the row's best iff some kh < thr, or kh == thr with
          // a smaller parity / earlier candidate (ties resolve by candidate order)
          const int tmin = min(min(m0, m1), min(m2, m3)) + oq;
          const int th = thr[r];
          const bool need = tmin < th || (tmin == th && tile_e <= tie_e[r]);
          if (__any_sync(0xffffffffu, need)) {
            if (lane == 0 && p.rescans) atomicAdd(p.rescans, 1ull);
            const unsigned long long b =
                rescan_half(taddr, hq_s, meta_s, oq, th, rm.y, need, S, lane & 7, best[r]);
            best[r] = b;
            if (b != ~0ull) {
              const long long key2 = (long long)(b >> 32) - rm.y;
              thr[r] = (int)(key2 >> 1);
              const int eb = (int)((b & 0xffffffffull) / (unsigned long long)(8 * S));
              tie_e[r] = (key2 & 1) ? 0x7fffffff : eb;
            }
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(tempty_bar(buf));
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(empty_bar(s));
      }
#pragma unroll 1
      for (int r = 0; r < RG; ++r) {
        const int m = p.row_meta[(size_t)(g * RG + r) * kTileM + row].z;
        if ((lane & 7) == 0 && m >= 0 && best[r] != ~0ull) atomicMin(&p.keys[m], best[r]);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
}

// ---------------------------------------------------------------------------
// operand preparation
// ---------------------------------------------------------------------------

// Per column: Q1 = sum q, Q2 = sum q^2, qmin, qmax; histograms for the host.
__global__ void col_stats_kernel(const int16_t* __restrict__ qbase, int64_t ncols, int n,
                                 int4* __restrict__ stats, uint32_t* __restrict__ q1_key,
                                 uint32_t* __restrict__ qmin_key, uint32_t* __restrict__ qmax_key,
                                 int32_t* __restrict__ ids, unsigned* __restrict__ hist_q1,
                                 unsigned* __restrict__ hist_qmin, unsigned* __restrict__ hist_qmax) {
  const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  const int16_t* q = qbase + col * n;
  int s1 = 0, s2 = 0, lo = 1 << 20, hi = -(1 << 20);
  for (int k = 0; k < n; ++k) {
    const int v = q[k];
    s1 += v;
    s2 += v * v;
    lo = min(lo, v);
    hi = max(hi, v);
  }
  stats[col] = make_int4(s1, s2, lo, hi);
  q1_key[col] = (uint32_t)(s1 + 32768);
  qmin_key[col] = (uint32_t)(lo + 512);
  qmax_key[col] = (uint32_t)(512 - hi);  // ascending key == qmax descending
  ids[col] = (int32_t)col;
  atomicAdd(&hist_q1[min(max(s1 + 2048, 0), 4095)], 1u);
  atomicAdd(&hist_qmin[lo + 512], 1u);
  atomicAdd(&hist_qmax[hi + 512], 1u);
}

// Fill the padded B operand: every sorted column goes to its slot in the
// Q1-grouped, 256-padded layout; K-major canonical UMMA layout per tile.
__global__ void build_b_kernel(const int16_t* __restrict__ qbase, int n, int kpad, int planes,
                               const int32_t* __restrict__ sorted_cols, int64_t ncols,
                               const int4* __restrict__ stats, const int32_t* __restrict__ grp_sorted,
                               const int32_t* __restrict__ grp_padded,
                               int8_t* __restrict__ b_tiles, int32_t* __restrict__ hq,
                               uint32_t* __restrict__ meta, int2* __restrict__ tile_info) {
  const int chunks = kpad / 16;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncols * chunks) return;
  const int64_t sp = i / chunks;
  const int kc = (int)(i - sp * chunks);
  const int col = sorted_cols[sp];
  const int4 st = stats[col];
  const int bin = min(max(st.x + 2048, 0), 4095);
  const int64_t slot = (int64_t)grp_padded[bin] + (sp - grp_sorted[bin]);
  const int64_t tile = slot / kTileN;
  const int cc = (int)(slot - tile * kTileN);
  const int16_t* q = qbase + (int64_t)col * n;
  uint32_t w[4];
#pragma unroll
  for (int b4 = 0; b4 < 4; ++b4) {
    uint32_t word = 0;
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) {
      const int k = kc * 16 + b4 * 4 + bb;
      int v = 0;
      if (planes == 1) {
        if (k < n) v = -q[k];
      } else {
        if (k < n) {
          v = min(max(-(int)q[k], -127), 127);
        } else if (k < 2 * n) {
          const int x = -(int)q[k - n];
          v = x - min(max(x, -127), 127);
        }
      }
      word |= (uint32_t)(uint8_t)(int8_t)v << (8 * bb);
    }
    w[b4] = word;
  }
  int8_t* dst = b_tiles + tile * ((int64_t)kTileN * kpad) + (int64_t)kc * (kTileN * 16) +
                (cc >> 3) * 128 + (cc & 7) * 16;
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  if (kc == 0) {
    hq[slot] = st.y >> 1;
    meta[slot] = ((uint32_t)(st.y & 1) << 31) | (uint32_t)col;
    if (cc == 0) tile_info[tile] = make_int2(st.x, col);  // first slot = smallest column
  }
}

__global__ void fill_u32_kernel(uint32_t* __restrict__ p, int64_t n, uint32_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// A operand: row (range, iso) of each 128-row tile = 16 ranges x 8 isometries;
// bytes = r_iso (and again for the second plane), zero padded to kpad.
__global__ void build_a_kernel(const uint8_t* __restrict__ rtiles, const double* __restrict__ rmean,
                               const int32_t* __restrict__ rsq, int64_t M, int n, int kpad,
                               int planes, const uint16_t* __restrict__ inv, int64_t rows_pad,
                               uint8_t* __restrict__ a_tiles, int4* __restrict__ row_meta) {
  const int chunks = kpad / 16;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_pad * chunks) return;
  const int64_t row = i / chunks;
  const int kc = (int)(i - row * chunks);
  const int64_t m = row >> 3;
  const int iso = (int)(row & 7);
  const int64_t tile = row / kTileM;
  const int rr = (int)(row - tile * kTileM);
  uint32_t w[4] = {0, 0, 0, 0};
  if (m < M) {
    const uint8_t* r = rtiles + m * n;
#pragma unroll
    for (int b4 = 0; b4 < 4; ++b4) {
      uint32_t word = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        int k = kc * 16 + b4 * 4 + bb;
        if (planes == 2 && k >= n) k -= n;
        const uint32_t v = k < n ? r[inv[iso * n + k]] : 0u;
        word |= v << (8 * bb);
      }
      w[b4] = word;
    }
  }
  uint8_t* dst = a_tiles + tile * ((int64_t)kTileM * kpad) + (int64_t)kc * (kTileM * 16) +
                 (rr >> 3) * 128 + (rr & 7) * 16;
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  if (kc == 0) {
    if (m < M) {
      const double mean = rmean[m];
      const int o = (int)rint(mean);
      const int s1 = (int)rint(mean * n);  // exact: mean = s1 / n, n a power of two
      const int R = rsq[m] - 2 * o * s1 + n * o * o;
      row_meta[row] = make_int4(o, R, (int)m, 0);
    } else {
      row_meta[row] = make_int4(0, 0, -1, 0);
    }
  }
}

template <int KPAD, int RG, int STAGES>
int launch_tc(Ctx* c, const TcParams& prm) {
  using Lay = TcLayout<KPAD, RG, STAGES>;
  auto kern = tc_scan_kernel<KPAD, RG, STAGES>;
  static_assert(Lay::kSmem <= 227 * 1024, "shared memory budget");
  FC_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::kSmem));
  const int grid = (int)std::min<int64_t>(prm.n_units, c->sm_count);
  kern<<<grid, kThreads, Lay::kSmem, c->stream>>>(prm);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;
  return FC_OK;
}

int tc_row_group(int kpad) { return kpad >= 256 ? 2 : kpad >= 64 ? 4 : 8; }

}  // namespace

int level_prepare_tc(Ctx* c, Level& L) {
  TcOperands& T = L.tc;
  T.ready = false;
  if (L.baseline || L.n < 16) return set_error(c, FC_ERR_ARG, "tensor path: proposed mode, B >= 4");
  const int64_t ncols = L.count * L.s_count;
  if (ncols >= (1ll << 31)) return set_error(c, FC_ERR_ARG, "too many columns");
  T.ncols = ncols;
  // scratch: keys / values for the sorts, histograms
  const size_t hist_words = 4096 + 1024 + 1024;
  FC_CUDA(c, T.col_stats.reserve(ncols * 16));
  FC_CUDA(c, c->key_in.reserve(ncols * 8));
  FC_CUDA(c, c->key_out.reserve(ncols * 8));
  FC_CUDA(c, c->val_in.reserve(ncols * 4));
  FC_CUDA(c, c->val_out.reserve(ncols * 4));
  FC_CUDA(c, c->tc_scratch.reserve(ncols * 8 + hist_words * 4));
  uint32_t* k_q1 = c->key_in.as<uint32_t>();
  uint32_t* k_min = k_q1 + ncols;
  uint32_t* k_max = c->tc_scratch.as<uint32_t>();
  unsigned* hist = reinterpret_cast<unsigned*>(k_max + ncols);
  FC_CUDA(c, cudaMemsetAsync(hist, 0, hist_words * 4, c->stream));
  col_stats_kernel<<<(unsigned)((ncols + 255) / 256), 256, 0, c->stream>>>(
      L.qbase.as<int16_t>(), ncols, L.n, T.col_stats.as<int4>(), k_q1, k_min, k_max,
      c->val_in.as<int32_t>(), hist, hist + 4096, hist + 5120);
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 1;
  std::vector<unsigned> h(hist_words);
  FC_CUDA(c, cudaMemcpyAsync(h.data(), hist, hist_words * 4, cudaMemcpyDeviceToHost, c->stream));
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  const unsigned* hq1 = h.data();
  const unsigned* hmin = h.data() + 4096;
  const unsigned* hmax = h.data() + 5120;
  int gmin = 1 << 20, gmax = -(1 << 20);
  for (int v = 0; v < 1024; ++v) {
    if (hmin[v]) gmin = std::min(gmin, v - 512);
    if (hmax[v]) gmax = std::max(gmax, v - 512);
  }
  if (gmin < -254 || gmax > 254) return set_error(c, FC_ERR_ARG, "operand outside two s8 planes");
  T.planes = (gmin >= -127 && gmax <= 127) ? 1 : 2;
  T.kpad = ((T.planes * L.n + 31) / 32) * 32;
  // clamp-reach counts: low_count[o] = #{qmin < -o}, high_count[o] = #{qmax > 255 - o}
  for (int o = 0; o < 256; ++o) {
    int64_t lo = 0, hi = 0;
    for (int v = 0; v < 1024; ++v) {
      const int q = v - 512;
      if (q < -o) lo += hmin[v];
      if (q > 255 - o) hi += hmax[v];
    }
    T.low_count[o] = lo;
    T.high_count[o] = hi;
  }
  // Q1 groups, each padded to a multiple of 256 columns
  std::vector<int32_t> grp_sorted(4096), grp_padded(4096);
  std::vector<int32_t> tile_q1;  // becomes int2 {Q1, cmin}; cmin filled on the device
  int64_t acc_sorted = 0, acc_tiles = 0;
  for (int b = 0; b < 4096; ++b) {
    grp_sorted[b] = (int32_t)acc_sorted;
    grp_padded[b] = (int32_t)(acc_tiles * kTileN);
    const int64_t cnt = hq1[b];
    const int64_t tiles = (cnt + kTileN - 1) / kTileN;
    for (int64_t t = 0; t < tiles; ++t) {
      tile_q1.push_back(b - 2048);
      tile_q1.push_back(0);
    }
    acc_sorted += cnt;
    acc_tiles += tiles;
  }
  if (acc_tiles * kTileN >= (1ll << 31)) return set_error(c, FC_ERR_ARG, "too many columns");
  T.ntiles = acc_tiles;
  // sorts: by Q1 (stable -> ascending column order inside a group), qmin asc, qmax desc
  size_t tmp = 0, need = 0;
  FC_CUDA(c, cub::DeviceRadixSort::SortPairs(nullptr, need, k_q1, c->key_out.as<uint32_t>(),
                                             c->val_in.as<int32_t>(), c->val_out.as<int32_t>(),
                                             (int)ncols, 0, 16, c->stream));
  tmp = need;
  FC_CUDA(c, c->cub_tmp.reserve(tmp));
  FC_CUDA(c, T.reach_low.reserve(ncols * 4));
  FC_CUDA(c, T.reach_high.reserve(ncols * 4));
  FC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.ptr, tmp, k_q1, c->key_out.as<uint32_t>(),
                                             c->val_in.as<int32_t>(), c->val_out.as<int32_t>(),
                                             (int)ncols, 0, 16, c->stream));
  // (val_in keeps the identity permutation: SortPairs does not modify its inputs)
  FC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.ptr, tmp, k_min, c->key_out.as<uint32_t>() + ncols,
                                             c->val_in.as<int32_t>(), T.reach_low.as<int32_t>(),
                                             (int)ncols, 0, 16, c->stream));
  FC_CUDA(c, cub::DeviceRadixSort::SortPairs(c->cub_tmp.ptr, tmp, k_max, c->key_out.as<uint32_t>() + ncols,
                                             c->val_in.as<int32_t>(), T.reach_high.as<int32_t>(),
                                             (int)ncols, 0, 16, c->stream));
  // padded operand + metadata
  const int64_t slots = T.ntiles * kTileN;
  FC_CUDA(c, T.b_tiles.reserve(slots * T.kpad));
  FC_CUDA(c, T.hq.reserve(slots * 4));
  FC_CUDA(c, T.meta.reserve(slots * 4));
  FC_CUDA(c, T.tile_q1.reserve(T.ntiles * 8));
  FC_CUDA(c, cudaMemsetAsync(T.b_tiles.ptr, 0, slots * T.kpad, c->stream));
  fill_u32_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, c->stream>>>(T.hq.as<uint32_t>(), slots,
                                                                          (uint32_t)kPadHq);
  FC_CUDA(c, cudaMemsetAsync(T.meta.ptr, 0, slots * 4, c->stream));
  FC_CUDA(c, cudaMemcpyAsync(T.tile_q1.ptr, tile_q1.data(), T.ntiles * 8, cudaMemcpyHostToDevice,
                             c->stream));
  int32_t* d_grp = c->fix_prefix.as<int32_t>();
  FC_CUDA(c, c->fix_prefix.reserve(2 * 4096 * 4));
  d_grp = c->fix_prefix.as<int32_t>();
  FC_CUDA(c, cudaMemcpyAsync(d_grp, grp_sorted.data(), 4096 * 4, cudaMemcpyHostToDevice, c->stream));
  FC_CUDA(c, cudaMemcpyAsync(d_grp + 4096, grp_padded.data(), 4096 * 4, cudaMemcpyHostToDevice,
                             c->stream));
  const int64_t work = ncols * (T.kpad / 16);
  build_b_kernel<<<(unsigned)((work + 255) / 256), 256, 0, c->stream>>>(
      L.qbase.as<int16_t>(), L.n, T.kpad, T.planes, c->val_out.as<int32_t>(), ncols,
      T.col_stats.as<int4>(), d_grp, d_grp + 4096, T.b_tiles.as<int8_t>(), T.hq.as<int32_t>(),
      T.meta.as<uint32_t>(), T.tile_q1.as<int2>());
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 2;  // fill + build
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  T.ready = true;
  return FC_OK;
}

int scan_tc(Ctx* c, Level& L, int64_t M, uint64_t* d_keys) {
  TcOperands& T = L.tc;
  if (!T.ready) return set_error(c, FC_ERR_STATE, "tensor operands not prepared");
  FC_TRY(ensure_iso_tables(c));
  const int RG = tc_row_group(T.kpad);
  const int64_t n_rtiles = (M * 8 + kTileM - 1) / kTileM;
  const int n_rgroups = (int)((n_rtiles + RG - 1) / RG);
  const int64_t rows_pad = (int64_t)n_rgroups * RG * kTileM;
  FC_CUDA(c, c->a_tiles.reserve(rows_pad * T.kpad));
  FC_CUDA(c, c->row_meta.reserve(rows_pad * 16));
  // the host needs each range's offset o to plan the clamp corrections
  c->h_roff.resize(M);
  FC_CUDA(c, cudaMemcpyAsync(c->h_roff.data(), c->roff.ptr, M * 4, cudaMemcpyDeviceToHost, c->stream));
  FC_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  const uint16_t* inv = c->iso_inv.as<uint16_t>() + iso_table_offset(L.side);
  const int64_t work = rows_pad * (T.kpad / 16);
  build_a_kernel<<<(unsigned)((work + 255) / 256), 256, 0, c->stream>>>(
      c->rtiles.as<uint8_t>(), c->rmean.as<double>(), c->rsq.as<int32_t>(), M, L.n, T.kpad, T.planes,
      inv, rows_pad, c->a_tiles.as<uint8_t>(), c->row_meta.as<int4>());
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 1;

  TcParams prm;
  prm.a_tiles = c->a_tiles.as<uint8_t>();
  prm.row_meta = c->row_meta.as<int4>();
  prm.b_tiles = T.b_tiles.as<int8_t>();
  prm.hq = T.hq.as<int32_t>();
  prm.meta = T.meta.as<uint32_t>();
  prm.tile_info = T.tile_q1.as<int2>();
  FC_CUDA(c, c->count_buf.reserve(64));
  prm.rescans = c->count_buf.as<unsigned long long>() + 1;
  prm.keys = reinterpret_cast<unsigned long long*>(d_keys);
  prm.S = L.s_count;
  prm.n_rgroups = n_rgroups;
  prm.ntiles = (int)T.ntiles;
  // split the column tiles into spans: minimise the per-CTA makespan
  // ceil(units / grid) * (tiles per unit + unit overhead) over the span count
  {
    const int64_t grid = c->sm_count;
    double best_cost = 1e300;
    int64_t best_ct = T.ntiles;
    for (int64_t s = 1; s <= std::min<int64_t>(T.ntiles, 8192); ++s) {
      const int64_t ct = (T.ntiles + s - 1) / s;
      const int64_t nsp = (T.ntiles + ct - 1) / ct;
      const int64_t units = nsp * n_rgroups;
      const int64_t per_cta = (units + grid - 1) / grid;
      const double cost = (double)per_cta * (double)(ct + 2);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best_ct = ct;
      }
    }
    prm.tiles_per_unit = (int)best_ct;
  }
  const int64_t n_spans = (T.ntiles + prm.tiles_per_unit - 1) / prm.tiles_per_unit;
  prm.n_units = n_spans * n_rgroups;

  FC_CUDA(c, c->count_buf.reserve(64));
  FC_CUDA(c, cudaMemsetAsync(c->count_buf.as<unsigned long long>() + 1, 0, 8, c->stream));
  cudaEvent_t m0, m1;
  cudaEventCreate(&m0);
  cudaEventCreate(&m1);
  cudaEventRecord(m0, c->stream);
  int rc;
  switch (T.kpad) {
    case 32: rc = launch_tc<32, 8, 8>(c, prm); break;
    case 64: rc = launch_tc<64, 4, 6>(c, prm); break;
    case 128: rc = launch_tc<128, 4, 3>(c, prm); break;
    case 256: rc = launch_tc<256, 2, 2>(c, prm); break;
    case 512: rc = launch_tc<512, 1, 1>(c, prm); break;
    default: rc = set_error(c, FC_ERR_ARG, "unsupported K");
  }
  cudaEventRecord(m1, c->stream);
  if (rc != FC_OK) {
    cudaEventDestroy(m0);
    cudaEventDestroy(m1);
    return rc;
  }

  // ---- clamp corrections (exact kernel on clamp-active pairs) ----
  FC_CUDA(c, cudaEventSynchronize(c->ev1));
  std::vector<int32_t> order(M);
  std::vector<int64_t> start(257, 0);
  for (int64_t i = 0; i < M; ++i) start[c->h_roff[i] + 1]++;
  for (int o = 0; o < 256; ++o) start[o + 1] += start[o];
  {
    std::vector<int64_t> pos(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < M; ++i) order[pos[c->h_roff[i]]++] = (int32_t)i;
  }
  std::vector<int4> jobs;
  std::vector<int64_t> prefix(1, 0);
  int64_t fix_pairs = 0;
  const int RB = 8, CB = 128;
  for (int o = 0; o < 256; ++o) {
    const int64_t cnt = start[o + 1] - start[o];
    if (!cnt) continue;
    const int64_t lists[2] = {T.low_count[o], T.high_count[o]};
    for (int kind = 0; kind < 2; ++kind) {
      const int64_t ncol = lists[kind];
      if (!ncol) continue;
      jobs.push_back(make_int4(kind, (int)start[o], (int)cnt, (int)ncol));
      prefix.push_back(prefix.back() + ((cnt + RB - 1) / RB) * ((ncol + CB - 1) / CB));
      fix_pairs += cnt * ncol;
    }
  }
  c->stats.fix_pairs = fix_pairs;
  float fix_ms = 0.f;
  if (!jobs.empty()) {
    FC_CUDA(c, c->fix_rows.reserve(M * 4));
    FC_CUDA(c, c->fix_jobs.reserve(jobs.size() * 16));
    FC_CUDA(c, c->fix_cols.reserve(prefix.size() * 8));
    FC_CUDA(c, cudaMemcpyAsync(c->fix_rows.ptr, order.data(), M * 4, cudaMemcpyHostToDevice, c->stream));
    FC_CUDA(c, cudaMemcpyAsync(c->fix_jobs.ptr, jobs.data(), jobs.size() * 16, cudaMemcpyHostToDevice,
                               c->stream));
    FC_CUDA(c, cudaMemcpyAsync(c->fix_cols.ptr, prefix.data(), prefix.size() * 8,
                               cudaMemcpyHostToDevice, c->stream));
    rc = scan_exact_jobs(c, L, c->fix_jobs.as<int4>(), c->fix_cols.as<int64_t>(), (int)jobs.size(),
                         prefix.back(), c->fix_rows.as<int32_t>(), T.reach_low.as<int32_t>(),
                         T.reach_high.as<int32_t>(), d_keys);
    if (rc != FC_OK) {
      cudaEventDestroy(m0);
      cudaEventDestroy(m1);
      return rc;
    }
    cudaEventRecord(c->ev1, c->stream);
    FC_CUDA(c, cudaEventSynchronize(c->ev1));
    cudaEventElapsedTime(&fix_ms, m1, c->ev1);
  }
  FC_CUDA(c, cudaEventSynchronize(m1));
  float main_ms = 0.f;
  cudaEventElapsedTime(&main_ms, m0, m1);
  c->stats.main_ms = main_ms;
  unsigned long long resc = 0;
  FC_CUDA(c, cudaMemcpy(&resc, c->count_buf.as<unsigned long long>() + 1, 8, cudaMemcpyDeviceToHost));
  c->stats.rescans = (int64_t)resc;
  c->stats.fix_ms = fix_ms;
  cudaEventDestroy(m0);
  cudaEventDestroy(m1);
  return FC_OK;
}

}  // namespace fcb
