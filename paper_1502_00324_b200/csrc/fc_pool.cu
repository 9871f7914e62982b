// Domain-pool construction on the device (pool.py:88-178, image.py:116-130).
//
//  1. entropy_all_kernel (one launch for all four levels): a warp owns 32
//     adjacent window columns x 16 window rows; every lane keeps its window's
//     256-bin histogram in shared memory (hist[bin][lane], conflict-free) and
//     slides it down the lattice (remove the rows that leave, add the rows
//     that enter).  H = -sum_b t[count_b] with t[k] = p*log(p) from the
//     host-numpy LUT, summed in numpy's exact pairwise order (two 128-bin
//     halves, 8 running accumulators each, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//     half0+half1) so the float64 bits equal pool.py:88-92 on the same host.
//     Threshold levels append {ent > tau} survivors with warp-aggregated
//     atomics (order-free; the ranking below restores the reference order).
//  2. ranking, key = ~bits(|H|) (ascending == entropy descending), ties by
//     raster index (np.argsort(-ent, kind="stable"), pool.py:171):
//     threshold survivors: chunk bitonic sort + cross-chunk rank (2 launches
//     for all levels); general caps: CUB stable radix sort; cap 1: argmin.
//  3. survivors_all_kernel (one launch, all levels): a thread per decimated
//     pixel (floor 2x2 mean), segmented reductions for the exact sum / sum of
//     squares, mean and centred norm per survivor (pool.py:138-152).
#include <cub/cub.cuh>

#include "fc_internal.cuh"

namespace fcb {

namespace {

// Entropy kernel geometry per histogram width: u16 counts (windows of up to
// 32x32 = 1024 pixels, 16 KB of histograms per warp) or u8 counts (windows of
// up to 8x8 = 64 pixels, 8 KB per warp: twice the resident warps).
constexpr int kEntBlocksPerSm = 2;  // shared-memory bound
template <int BPW> __host__ __device__ constexpr int ent_warps() { return BPW == 2 ? 6 : 12; }
constexpr int kLutWords = 4 + 16 + 64 + 256 + 1024;  // the four [0, p*log(p)...] LUTs in smem

__device__ __forceinline__ uint64_t entropy_key(double h) {
  // |h|: maps the -0.0 of a constant window onto +0.0 (they compare equal in numpy).
  uint64_t bits = static_cast<uint64_t>(__double_as_longlong(h)) & 0x7fffffffffffffffull;
  return ~bits;  // ascending key == descending entropy
}

// Per-level description for the fused entropy kernel.
struct EntLevel {
  const uint8_t* img;  // the level's image (a batch launch covers several contexts)
  int width;
  int D, stride, nx, ny, strips_x, task_begin, lut_off;
  int y_lo, y_hi;  // the window rows this launch covers (all: 0, ny)
  int rows;  // window rows per task (one lane slides through them)
  int mode;  // 0: write key/val of every window (sort / argmin), 1: append {ent > tau}
  double tau;
  double* ent;
  uint64_t* key;
  uint32_t* val;
  int* sel_count;
};
// CAP levels per launch: 4 for one context, kEntBatchLevels for a batch of
// contexts (fc_pool_entropy_batch; kernel parameters up to 32 KB).  LUTs by
// window size (n = 1024 / 256 / 64 / 16) at fixed shared-memory offsets.
constexpr int kEntBatchLevels = 144;
template <int CAP>
struct EntParamsT {
  EntLevel lv[CAP];      // this launch's levels (n_levels of them), task ranges ascending
  const double* lut[4];  // device LUTs by lut_slot (nullptr: not used by the launch)
  int n_levels;
  int total_tasks;
};
using EntParams = EntParamsT<4>;
__host__ __device__ constexpr int ent_lut_off(int D) {
  return D == 32 ? 0 : D == 16 ? 1025 : D == 8 ? 1025 + 257 : 1025 + 257 + 65;
}

// Shared-memory accesses with explicit 32-bit shared addresses (generic
// pointers into shared memory cost an address-window conversion per access).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Pin a value in a register (keeps the compiler from re-deriving a shared
// address from SR_CgaCtaId inside hot loops).
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  uint32_t y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32_ordered(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void reds_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u32_ordered(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Lane-private histogram of BPW bins per 32-bit word: word (v / BPW) * 32 +
// lane packs the counts of bins BPW*(v/BPW) .. +BPW-1 (u16 pairs or u8
// quads, low bin in the low bits), so every access of a warp hits bank =
// lane (conflict-free).  Updates are shared-memory reductions without return
// (pipelined); sign = 1 adds a pixel, 0xffffffff removes one (a removal never
// borrows across fields: only counted pixels are removed).  hw = shared
// address of this lane's word 0.
template <int D, int BPW>
__device__ __forceinline__ void hist_rows(uint32_t hw, const uint8_t* __restrict__ img, int width,
                                          int x, int r0, int r1, uint32_t sign) {
  constexpr int kShift = 32 / BPW;
  for (int r = r0; r < r1; ++r) {
    const uint8_t* row = img + (int64_t)r * width + x;
#pragma unroll 8
    for (int k = 0; k < D; ++k) {
      const uint32_t v = __ldg(row + k);
      reds_add(hw + (v / BPW) * 128, sign << (kShift * (v % BPW)));
    }
  }
}

// numpy pairwise sum of the 256 terms t[count] (pool.py:88-92): two 128-bin
// halves, 8 running accumulators each, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)).
// Zero bins add +0.0 (exact): lut[0] holds 0.0 and lut[k] = t(k).  Every term
// is <= 0, so adding a zero term never changes an accumulator's bits, and an
// 8-bin group (one term per accumulator, in bin order) that is empty in all
// 32 windows of the warp is skipped with a warp-uniform branch: neighbouring
// windows share most pixels, so typically 2/3 of the groups are skipped.
// Must be called by the full warp (inactive lanes hold an all-zero histogram).
template <int BPW>
__device__ __forceinline__ double window_entropy(uint32_t hw, uint32_t lut) {
  constexpr int kWpg = 8 / BPW;  // words per 8-bin group
  double half_sum[2];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      uint32_t w[kWpg];
      uint32_t any = 0;
#pragma unroll
      for (int q = 0; q < kWpg; ++q) {
        w[q] = lds_u32_ordered(hw + ((half * 16 + g) * kWpg + q) * 128);
        any |= w[q];
      }
      if (__any_sync(0xffffffffu, any != 0u)) {
#pragma unroll
        for (int q = 0; q < kWpg; ++q) {
          if constexpr (BPW == 2) {
            // counts <= 1024 < 2^13, so (w >> 13) == 8 * (w >> 16)
            acc[2 * q] = acc[2 * q] + lds_f64(lut + ((w[q] & 0xffffu) << 3));
            acc[2 * q + 1] = acc[2 * q + 1] + lds_f64(lut + (w[q] >> 13));
          } else {
#pragma unroll
            for (int b = 0; b < 4; ++b)
              acc[4 * q + b] = acc[4 * q + b] + lds_f64(lut + (((w[q] >> (8 * b)) & 0xffu) << 3));
          }
        }
      }
    }
    half_sum[half] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
  return -(half_sum[0] + half_sum[1]);
}

// One warp per task = 32 adjacent window columns x L.rows window rows of
// one level.  Each lane keeps its window's 256-bin histogram and slides it
// down by `stride` rows (remove the rows that leave, add the rows that
// enter), so a window costs 2*stride*D updates instead of D*D.
template <int D, int BPW>
__device__ __forceinline__ void entropy_task(const EntLevel& L, const uint8_t* __restrict__ img,
                                             int width, int task, uint32_t h, uint32_t lut,
                                             int lane) {
  const int t = task - L.task_begin;
  const int sy = t / L.strips_x, sx = t - sy * L.strips_x;
  const int wx = sx * 32 + lane;
  const bool active = wx < L.nx;
  const int wy0 = L.y_lo + sy * L.rows;
  const int wy1 = min(wy0 + L.rows, L.y_hi);
  const int s = L.stride;
  const int x = wx * s;
  static_assert(BPW == 2 || D * D < 256, "u8 histogram counts");
#pragma unroll 8
  for (int b = 0; b < 256 / BPW; ++b) sts_u32_ordered(h + b * 128, 0u);
  if (active) hist_rows<D, BPW>(h, img, width, x, wy0 * s, wy0 * s + D, 1u);
  for (int wy = wy0; wy < wy1; ++wy) {
    if (wy > wy0 && active) {
      const int yp = (wy - 1) * s, yn = wy * s;
      hist_rows<D, BPW>(h, img, width, x, yp, yp + min(s, D), 0xffffffffu);
      hist_rows<D, BPW>(h, img, width, x, max(yp + D, yn), yn + D, 1u);
    }
    const double H = window_entropy<BPW>(h, lut);  // whole warp (see window_entropy)
    const int64_t w = (int64_t)wy * L.nx + wx;
    if (L.mode == 0) {
      if (active) {
        L.ent[w] = H;
        L.key[w] = entropy_key(H);
        L.val[w] = (uint32_t)w;
      }
    } else {
      if (active) L.ent[w] = H;
      const bool keep = active && H > L.tau;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (bal) {
        int base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(L.sel_count, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
        if (keep) {
          const int slot = base + __popc(bal & ((1u << lane) - 1));
          L.key[slot] = entropy_key(H);
          L.val[slot] = (uint32_t)w;
        }
      }
    }
  }
}

// One launch per histogram width: BPW = 2 for the 32x32 / 16x16 windows,
// BPW = 4 for the 8x8 / 4x4 windows (P holds only the launch's levels).
template <int BPW, int CAP>
__global__ void __launch_bounds__(ent_warps<BPW>() * 32)
entropy_all_kernel(const __grid_constant__ EntParamsT<CAP> P) {
  constexpr int kWarps = ent_warps<BPW>();
  extern __shared__ __align__(16) uint8_t ent_smem[];
  double* lut_s = reinterpret_cast<double*>(ent_smem);
  uint32_t* hist_all = reinterpret_cast<uint32_t*>(ent_smem + kLutWords * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = 0; t < 4; ++t) {
    if (!P.lut[t]) continue;
    const int D = 4 << t;  // lut_slot: 0 -> 4x4, 1 -> 8x8, 2 -> 16x16, 3 -> 32x32
    const int n = D * D;
    for (int i = threadIdx.x; i <= n; i += blockDim.x)
      lut_s[ent_lut_off(D) + i] = i ? P.lut[t][i - 1] : 0.0;
  }
  __syncthreads();
  const uint32_t h = opaque_u32(smem_addr(hist_all + warp * ((256 / BPW) * 32) + lane));
  const uint32_t lut_base = opaque_u32(smem_addr(lut_s));
  for (int task = blockIdx.x * kWarps + warp; task < P.total_tasks; task += gridDim.x * kWarps) {
    int l = 0;
    if constexpr (CAP <= 4) {
#pragma unroll
      for (int k = 1; k < CAP; ++k)
        if (k < P.n_levels && task >= P.lv[k].task_begin) l = k;
    } else {
      int lo = 0, hi = P.n_levels - 1;  // last level whose range starts at or before task
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (task >= P.lv[mid].task_begin) lo = mid; else hi = mid - 1;
      }
      l = lo;
    }
    const EntLevel& L = P.lv[l];
    const uint32_t lut = lut_base + L.lut_off * 8;
    if constexpr (BPW == 2) {
      if (L.D == 32) entropy_task<32, 2>(L, L.img, L.width, task, h, lut, lane);
      else entropy_task<16, 2>(L, L.img, L.width, task, h, lut, lane);
    } else {
      if (L.D == 8) entropy_task<8, 4>(L, L.img, L.width, task, h, lut, lane);
      else entropy_task<4, 4>(L, L.img, L.width, task, h, lut, lane);
    }
  }
}

template <int BPW>
__host__ __device__ constexpr int ent_smem() { return kLutWords * 8 + ent_warps<BPW>() * (256 / BPW) * 32 * 4; }

// ---- rank sort of the threshold survivors: (key asc, window asc) ----
// chunk size: 1024 elements (512 threads) while the survivor sets are small,
// else 2048 (1024 threads)
constexpr int kChunkSmall = 1024;
constexpr int kChunk = 2048;
constexpr int kMaxChunks = 64;

struct SortLevel {
  uint64_t* key;      // survivors (unordered), sorted in place per chunk
  uint32_t* val;
  uint32_t* out;      // window ids in rank order
  int count;
  int chunk_begin;    // first chunk (block) index of this level
};
struct SortParams {
  SortLevel lv[4];
  int n_levels;
  int total_chunks;
};

__device__ __forceinline__ bool lex_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ int sort_level_of(const SortParams& P, int chunk) {
  int l = 0;
  for (int k = 1; k < P.n_levels; ++k)
    if (chunk >= P.lv[k].chunk_begin) l = k;
  return l;
}

// One chunk sorted by (key, window) with CUB's block merge sort (CHUNK / 2
// threads, 2 items each).
struct KeyIdx {
  uint64_t k;
  uint32_t v;
};
struct KeyIdxLess {
  __device__ __forceinline__ bool operator()(const KeyIdx& a, const KeyIdx& b) const {
    return a.k < b.k || (a.k == b.k && a.v < b.v);
  }
};

template <int kChunk>
__global__ void __launch_bounds__(kChunk / 2) chunk_sort_kernel(SortParams P, int32_t* rank) {
  using Sorter = cub::BlockMergeSort<KeyIdx, kChunk / 2, 2>;
  __shared__ typename Sorter::TempStorage tmp;
  // this chunk's rank accumulators, filled by chunk_pair_rank_kernel next
  // (none for the merge path)
  if (rank)
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x) rank[blockIdx.x * kChunk + i] = 0;
  const int l = sort_level_of(P, blockIdx.x);
  const SortLevel& L = P.lv[l];
  const int c = blockIdx.x - L.chunk_begin;
  const int base = c * kChunk;
  const int n = min(kChunk, L.count - base);
  KeyIdx items[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = threadIdx.x * 2 + k;  // blocked arrangement
    items[k] = i < n ? KeyIdx{L.key[base + i], L.val[base + i]} : KeyIdx{~0ull, 0xffffffffu};
  }
  Sorter(tmp).Sort(items, KeyIdxLess());
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = threadIdx.x * 2 + k;
    if (i < n) {
      L.key[base + i] = items[k].k;
      L.val[base + i] = items[k].v;
    }
  }
}

// Global rank = position in the own sorted chunk + number of smaller elements
// in every other chunk: one block per (chunk a, chunk b) pair stages chunk b
// in shared memory and adds, for each element of a, its lower bound in b.
struct RankLevel {
  int nch;          // chunks of this level
  int pair_begin;   // first (a, b) pair block of this level
};
template <int kChunk>
__global__ void __launch_bounds__(kChunk / 2) chunk_pair_rank_kernel(SortParams P, RankLevel R0,
                                                               RankLevel R1, RankLevel R2,
                                                               RankLevel R3,
                                                               int32_t* __restrict__ rank_all) {
  __shared__ uint64_t sk[kChunk];
  __shared__ uint32_t si[kChunk];
  const RankLevel RL[4] = {R0, R1, R2, R3};
  int l = 0;
  for (int k = 1; k < P.n_levels; ++k)
    if ((int)blockIdx.x >= RL[k].pair_begin) l = k;
  const SortLevel& L = P.lv[l];
  const int pr = blockIdx.x - RL[l].pair_begin;
  const int ca = pr / RL[l].nch, cb = pr - ca * RL[l].nch;
  const int na = min(kChunk, L.count - ca * kChunk);
  const int nb = min(kChunk, L.count - cb * kChunk);
  int32_t* rank = rank_all + L.chunk_begin * kChunk;  // this level's rank slots
  if (ca == cb) {
    for (int p = threadIdx.x; p < na; p += blockDim.x) atomicAdd(&rank[ca * kChunk + p], p);
    return;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    sk[i] = L.key[cb * kChunk + i];
    si[i] = L.val[cb * kChunk + i];
  }
  __syncthreads();
  for (int p = threadIdx.x; p < na; p += blockDim.x) {
    const uint64_t k = L.key[ca * kChunk + p];
    const uint32_t v = L.val[ca * kChunk + p];
    int lo = 0, hi = nb;  // first element of b that is >= (k, v)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lex_less(sk[mid], si[mid], k, v)) lo = mid + 1; else hi = mid;
    }
    if (lo) atomicAdd(&rank[ca * kChunk + p], lo);
  }
}

template <int kChunk>
__global__ void rank_scatter_kernel(SortParams P, const int32_t* __restrict__ rank_all) {
  const int l = sort_level_of(P, blockIdx.x / (kChunk / 256));
  const SortLevel& L = P.lv[l];
  const int64_t i = (int64_t)(blockIdx.x - L.chunk_begin * (kChunk / 256)) * 256 + threadIdx.x;
  if (i >= L.count) return;
  L.out[rank_all[L.chunk_begin * kChunk + i]] = L.val[i];
}

// Large sets: the chunk-sorted runs (chunk_sort_kernel) merged pairwise,
// ceil(log2(chunks)) passes.  A block writes kMergeTile consecutive outputs
// of one run pair (runs are >= kChunk = kMergeTile long, so a tile never
// straddles pairs): two merge-path searches in global memory give its input
// spans, which are staged in shared memory with coalesced loads; each thread
// then merges kMergeIpt outputs from shared memory (a second merge-path
// search there) and the tile leaves as coalesced stores.  Keys are unique
// (key, window) pairs, so the order is total and no stability is needed.
constexpr int kMergeIpt = 8;
constexpr int kMergeTile = 256 * kMergeIpt;
static_assert(kMergeTile == kChunk, "merge tiles must divide the run width");

__device__ __forceinline__ int64_t merge_path(const uint64_t* __restrict__ ka, const uint32_t* __restrict__ va,
                                              int64_t na, const uint64_t* __restrict__ kb,
                                              const uint32_t* __restrict__ vb, int64_t nb, int64_t d) {
  int64_t lo = max((int64_t)0, d - nb), hi = min(d, na);
  while (lo < hi) {  // first x with !(a[x] < b[d - x - 1])
    const int64_t x = (lo + hi) >> 1;
    const int64_t y = d - x - 1;
    if (lex_less(ka[x], va[x], kb[y], vb[y])) lo = x + 1;
    else hi = x;
  }
  return lo;
}

// The same split by a warp: 32 probes per round (ballot of the monotone
// predicate a[x] < b[d - x - 1]), so a run of 2^21 takes 5 dependent rounds
// of loads instead of 21.
__device__ __forceinline__ int64_t merge_path_warp(const uint64_t* __restrict__ ka,
                                                   const uint32_t* __restrict__ va, int64_t na,
                                                   const uint64_t* __restrict__ kb,
                                                   const uint32_t* __restrict__ vb, int64_t nb,
                                                   int64_t d) {
  const int lane = threadIdx.x & 31;
  int64_t lo = max((int64_t)0, d - nb), hi = min(d, na);  // answer in [lo, hi]
  while (lo < hi) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t x = lo + lane * step;
    bool p = false;
    if (x < hi) {
      const int64_t y = d - x - 1;
      p = lex_less(ka[x], va[x], kb[y], vb[y]);
    }
    const int c = __popc(__ballot_sync(0xffffffffu, p));  // true lanes form a prefix
    if (c == 0) {
      hi = lo;
    } else {
      const int64_t last = lo + (int64_t)(c - 1) * step;
      lo = last + 1;
      hi = min(hi, last + step);
    }
  }
  return lo;
}

__global__ void __launch_bounds__(256)
merge_pass_kernel(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                  uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n,
                  int64_t width) {
  __shared__ uint64_t sk[kMergeTile];
  __shared__ uint32_t sv[kMergeTile];
  __shared__ int64_t split[2];
  const int64_t o0 = (int64_t)blockIdx.x * kMergeTile;
  const int64_t a0 = o0 / (2 * width) * (2 * width);
  const int64_t na = min(width, n - a0);
  const int64_t b0 = a0 + na;
  const int64_t nb = max((int64_t)0, min(width, n - b0));
  const int64_t d0 = o0 - a0;
  const int64_t d1 = min(d0 + kMergeTile, na + nb);
  if (threadIdx.x < 64) {  // warp 0: the tile's start split, warp 1: its end
    const int64_t d = threadIdx.x < 32 ? d0 : d1;
    const int64_t x = merge_path_warp(kin + a0, vin + a0, na, kin + b0, vin + b0, nb, d);
    if ((threadIdx.x & 31) == 0) split[threadIdx.x >> 5] = x;
  }
  __syncthreads();
  const int64_t ia0 = split[0], ia1 = split[1];
  const int64_t ib0 = d0 - ia0, ib1 = d1 - ia1;
  const int la = (int)(ia1 - ia0), lb = (int)(ib1 - ib0), len = la + lb;
  // stage: [0, la) = run a's span, [la, len) = run b's span
  for (int i = threadIdx.x; i < len; i += 256) {
    const int64_t g = i < la ? a0 + ia0 + i : b0 + ib0 + (i - la);
    sk[i] = kin[g];
    sv[i] = vin[g];
  }
  __syncthreads();
  const int t0 = threadIdx.x * kMergeIpt;
  uint64_t ok[kMergeIpt];
  uint32_t ov[kMergeIpt];
  int cnt = 0;
  if (t0 < len) {
    int ia = (int)merge_path(sk, sv, la, sk + la, sv + la, lb, t0);
    int ib = t0 - ia;
    cnt = min(kMergeIpt, len - t0);
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k) {
      if (k < cnt) {
        const bool take_a = ib >= lb || (ia < la && lex_less(sk[ia], sv[ia], sk[la + ib], sv[la + ib]));
        const int src = take_a ? ia : la + ib;
        ok[k] = sk[src];
        ov[k] = sv[src];
        ia += take_a;
        ib += !take_a;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kMergeIpt; ++k)
    if (k < cnt) {
      sk[t0 + k] = ok[k];
      sv[t0 + k] = ov[k];
    }
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += 256) {
    kout[o0 + i] = sk[i];
    vout[o0 + i] = sv[i];
  }
}

// Survivors of all levels in one launch.  A survivor's 2B x 2B window is
// handled by B lanes, lane = output row: its two input rows are read as
// aligned 16-byte blocks (funnel-shifted into place), horizontal pixel pairs
// are summed as packed 16-bit lanes over both rows, and the lane emits one
// output row (floor 2x2 mean, image.py:125-130).  Then per survivor:
// coordinates, entropy, exact sum / sum of squares, mean and centred norm
// (pool.py:138-152).
struct SurvLevel {
  const uint32_t* order;
  const double* ent_all;
  int64_t count;
  int B, nx, stride;
  int64_t warp_begin;
  uint32_t* xy;
  double* ent;
  uint8_t* tiles;
  int32_t* sum;
  int64_t* sumsq;
  double* mean;
  double* cnorm;
};
struct SurvParams {
  SurvLevel lv[4];
  int64_t total_warps;
  int* nsel_reset;  // the survivor counters, zeroed for the next pool build (read already)
};

// One window row: the 16-byte aligned blocks that cover bytes [a, a + D) of
// the image (a block is loaded only when it starts inside the image, so no
// access leaves the image's pages), then the NW + 1 words starting at the
// word of byte a; sh = bit offset of byte a inside that first word.
template <int D>
__device__ __forceinline__ void load_row_words(const uint8_t* __restrict__ img, int64_t img_bytes,
                                               int64_t a, uint32_t (&raw)[D / 4 + 1], int& sh) {
  constexpr int NW = D / 4, NL = (D + 30) / 16;
  const uintptr_t abs = reinterpret_cast<uintptr_t>(img + a);
  const uintptr_t base = abs & ~static_cast<uintptr_t>(15);
  const uintptr_t end = reinterpret_cast<uintptr_t>(img + img_bytes);
  const int off = (int)(abs - base);
  uint32_t wv[4 * NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    uint4 b = make_uint4(0, 0, 0, 0);
    if (base + 16 * k < end) b = __ldg(reinterpret_cast<const uint4*>(base + 16 * k));
    wv[4 * k] = b.x;
    wv[4 * k + 1] = b.y;
    wv[4 * k + 2] = b.z;
    wv[4 * k + 3] = b.w;
  }
  const int q4 = off >> 2;
#pragma unroll
  for (int j = 0; j <= NW; ++j) {
    uint32_t r = wv[j];
    r = q4 == 1 ? wv[j + 1] : r;
    r = q4 == 2 ? wv[j + 2] : r;
    r = q4 == 3 ? wv[j + 3] : r;
    raw[j] = r;
  }
  sh = (off & 3) * 8;
}

// lane = (survivor, decimated row): B = D / 2 lanes per survivor, PER = 32 / B
// survivors per warp.  Each lane loads its two window rows (two or three
// 16-byte loads each, from L2: the image is resident), forms the horizontal
// pair sums as packed 16-bit lanes, adds the two rows and emits one row of
// the floor 2x2 mean (pool.py:138-152 / image.py:116-130).
template <int D>
__device__ __forceinline__ void survivor_rows(const SurvLevel& L, const uint8_t* __restrict__ img,
                                              int width, int64_t img_bytes, int64_t warp_in_level,
                                              int lane, uint32_t* __restrict__ xy_s) {
  constexpr int B = D / 2, n = B * B, PER = 32 / B, NW = D / 4;
  const int grp = lane / B, row = lane % B;
  const int64_t sv = warp_in_level * PER + grp;
  const bool valid = sv < L.count;
  uint32_t w = 0;
  int wx = 0, wy = 0;
  int s1 = 0, s2 = 0;
  uint32_t outw[NW > 1 ? NW / 2 : 1];
  if (valid) {
    w = __ldg(L.order + sv);
    wy = w / L.nx;
    wx = w - wy * L.nx;
    const int64_t a = (int64_t)(wy * L.stride + 2 * row) * width + wx * L.stride;
    uint32_t r0[NW + 1], r1[NW + 1];
    int sh;
    load_row_words<D>(img, img_bytes, a, r0, sh);
    load_row_words<D>(img, img_bytes, a + width, r1, sh);
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const uint32_t u = __funnelshift_r(r0[k], r0[k + 1], sh);
      const uint32_t v = __funnelshift_r(r1[k], r1[k + 1], sh);
      // [b0+b1 | b2+b3] of both rows, then floor(sum / 4): two output pixels
      const uint32_t t = (u & 0x00ff00ffu) + ((u >> 8) & 0x00ff00ffu) + (v & 0x00ff00ffu) +
                         ((v >> 8) & 0x00ff00ffu);
      const uint32_t q = (t >> 2) & 0x00ff00ffu;
      const int v0 = (int)(q & 0xffu), v1 = (int)(q >> 16);
      s1 += v0 + v1;
      s2 += v0 * v0 + v1 * v1;
      if (k & 1) outw[k >> 1] = __byte_perm(outw[k >> 1], q, 0x6420);
      else outw[k >> 1] = q;
    }
    uint8_t* dst = L.tiles + sv * n + row * B;
    if constexpr (B == 16) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    } else if constexpr (B == 8) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(outw[0], outw[1]);
    } else if constexpr (B == 4) {
      *reinterpret_cast<uint32_t*>(dst) = outw[0];
    } else {
      *reinterpret_cast<uint16_t*>(dst) = (uint16_t)(outw[0] | (outw[0] >> 8));
    }
  }
#pragma unroll
  for (int o = B >> 1; o; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (valid && row == 0) {
    // staged: the block writes its survivors' origins as one coalesced run
    xy_s[(threadIdx.x >> 5) * PER + grp] = (uint32_t)(wx * L.stride) | ((uint32_t)(wy * L.stride) << 16);
    L.ent[sv] = L.ent_all[w];
    L.sum[sv] = s1;
    L.sumsq[sv] = s2;
    // mean = s1 / n; cnorm = s2 - s1*s1/n with Python float semantics
    // (pool.py:144-151).  n is a power of two and s1^2 < 2^53, so the
    // divisions are exact scalings: a multiplication by 1/n gives the same bits.
    constexpr double inv_n = 1.0 / n;
    L.mean[sv] = (double)s1 * inv_n;
    L.cnorm[sv] = __dsub_rn((double)s2, (double)((long long)s1 * s1) * inv_n);
  }
}

__global__ void __launch_bounds__(256) survivors_all_kernel(const uint8_t* __restrict__ img,
                                                            int width, int64_t img_bytes,
                                                            SurvParams P) {
  if (blockIdx.x == 0 && threadIdx.x < 4 && P.nsel_reset) P.nsel_reset[threadIdx.x] = 0;
  __shared__ uint32_t xy_s[8 * 16];  // 8 warps x up to 16 survivors per warp
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // levels start on block boundaries (warp_begin is a multiple of 8)
  int l = 0;
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if ((int64_t)blockIdx.x * 8 >= P.lv[k].warp_begin) l = k;
  // a by-value copy selected with constant indices: the fields are then read
  // with immediate constant-bank offsets, not an indexed load per field
  SurvLevel L;
  switch (l) {
    case 0: L = P.lv[0]; break;
    case 1: L = P.lv[1]; break;
    case 2: L = P.lv[2]; break;
    default: L = P.lv[3]; break;
  }
  const int64_t wl = gw - L.warp_begin;
  const int per = 32 / L.B;
  const int64_t level_warps = (L.count + per - 1) / per;
  if (wl < level_warps) {
    switch (L.B) {
      case 16: survivor_rows<32>(L, img, width, img_bytes, wl, lane, xy_s); break;
      case 8: survivor_rows<16>(L, img, width, img_bytes, wl, lane, xy_s); break;
      case 4: survivor_rows<8>(L, img, width, img_bytes, wl, lane, xy_s); break;
      default: survivor_rows<4>(L, img, width, img_bytes, wl, lane, xy_s); break;
    }
  }
  __syncthreads();
  const int64_t sv0 = ((int64_t)blockIdx.x * 8 - L.warp_begin) * per;
  const int64_t nblk = min((int64_t)8 * per, L.count - sv0);
  if ((int64_t)threadIdx.x < nblk) L.xy[sv0 + threadIdx.x] = xy_s[threadIdx.x];
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

__global__ void gather_all_keys_kernel(const double* __restrict__ ent, int64_t n,
                                       uint64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = entropy_key(ent[i]);
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

// Phase 1 of the pool build: every lattice window's entropy, all levels in
// two launches.  row_lo / row_hi (optional, per level) restrict the pass to
// window rows [row_lo, row_hi): a rank of a range-sharded encode computes its
// slice, and the slices are all-gathered before phase 2.
// Without a threshold a level's ent / key / val are written at the window
// index; with one, ent at the window index and the survivors (ent > tau)
// appended to key / val with a device counter.
//
// entropy_setup: one context's checks, level geometry, window buffers and
// survivor counters -> its four EntLevel entries (in stream order on c).
static int entropy_setup(Ctx* c, const int32_t strides[4], const int64_t caps[4],
                         const double taus[4], const int32_t use_tau[4], const int32_t* row_lo,
                         const int32_t* row_hi, EntLevel E[4]) {
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  for (int li = 0; li < kLevels; ++li) {
    if (strides[li] < 1) return set_error(c, FC_ERR_ARG, "strides must be 4 positive integers");
    if (caps[li] < 1) return set_error(c, FC_ERR_ARG, "caps must be >= 1");
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
  for (int li = 0; li < kLevels; ++li) {
    c->pool_caps[li] = caps[li];
    c->pool_use_tau[li] = use_tau[li];
  }
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
    c->pool_nx[li] = nx;
    c->pool_ny[li] = ny;
    const int64_t nwin = (int64_t)nx * ny;
    if (nwin >= (1ll << 31)) return set_error(c, FC_ERR_ARG, "too many lattice windows");
    FC_CUDA(c, L.win_ent.reserve(nwin * 8));
    FC_CUDA(c, L.win_key.reserve(nwin * 8 + 8 * 1032));
    FC_CUDA(c, L.win_key2.reserve(nwin * 8 + 8 * 1032));
    FC_CUDA(c, L.win_val.reserve(nwin * 4 + 4 * 1032));
    FC_CUDA(c, L.win_val2.reserve(nwin * 4 + 4 * 1032));
    EntLevel& e = E[li];
    e = EntLevel{};
    e.img = c->img_ptr;
    e.width = c->width;
    e.D = D;
    e.stride = L.stride;
    e.nx = nx;
    e.ny = ny;
    e.y_lo = row_lo ? std::min(std::max(row_lo[li], 0), ny) : 0;
    e.y_hi = row_hi ? std::min(std::max(row_hi[li], e.y_lo), ny) : ny;
    e.strips_x = (nx + 31) / 32;
    e.lut_off = ent_lut_off(D);
    e.mode = use_tau[li] ? 1 : 0;
    e.tau = use_tau[li] ? taus[li] : 0.0;
    e.ent = L.win_ent.as<double>();
    e.key = L.win_key.as<uint64_t>();
    e.val = L.win_val.as<uint32_t>();
    e.sel_count = d_nsel + li;
  }
  // the survivor counters are zero here: cleared once at allocation, then by
  // the previous build's survivors kernel after the host read them
  if (!c->nsel_clean) FC_CUDA(c, cudaMemsetAsync(d_nsel, 0, 4 * kLevels, c->stream));
  c->nsel_clean = false;
  if (!c->pool_ev[0])
    for (auto& e : c->pool_ev) FC_CUDA(c, cudaEventCreate(&e));
  FC_CUDA(c, cudaEventRecord(c->pool_ev[0], c->stream));
  return FC_OK;
}

// The levels of one or more contexts in two launches on lc's stream: u16
// histograms for the 32x32 / 16x16 windows, u8 for the 8x8 / 4x4 ones (half
// the shared memory per warp, twice the warps).  Rows per task: the smallest
// count whose tasks all fit in one wave of resident warps (every task costs
// about the same per row, so the kernel time is the longest task; a second
// partial wave would double it).
template <int CAP>
static int entropy_launch(Ctx* lc, const EntLevel* lv, int n, const double* const lut[4]) {
  EntParamsT<CAP> PL[2];  // launch parameters (copied at launch; up to 2 x 15 KB of stack)
  for (auto& Q : PL) {
    Q.n_levels = 0;
    Q.total_tasks = 0;
    for (auto& l : Q.lut) l = nullptr;
  }
  for (int i = 0; i < n; ++i) {
    const int k = lv[i].D >= 16 ? 0 : 1;
    EntParamsT<CAP>& Q = PL[k];
    if (Q.n_levels == CAP) return set_error(lc, FC_ERR_ARG, "too many levels for one entropy launch");
    Q.lv[Q.n_levels++] = lv[i];
    const int slot = lut_slot(lv[i].D * lv[i].D);
    Q.lut[slot] = lut[slot];
  }
  for (int k = 0; k < 2; ++k) {
    EntParamsT<CAP>& Q = PL[k];
    if (Q.n_levels == 0) continue;
    const int warps = k == 0 ? ent_warps<2>() : ent_warps<4>();
    const int64_t resident = (int64_t)lc->sm_count * kEntBlocksPerSm * warps;
    int rows = 4;
    for (;; ++rows) {
      int64_t t = 0;
      for (int i = 0; i < Q.n_levels; ++i)
        t += (int64_t)Q.lv[i].strips_x * ((Q.lv[i].y_hi - Q.lv[i].y_lo + rows - 1) / rows);
      if (t <= resident || rows >= 1 << 20) break;
    }
    int nt = 0;
    for (int i = 0; i < Q.n_levels; ++i) {
      Q.lv[i].rows = rows;
      Q.lv[i].task_begin = nt;
      nt += Q.lv[i].strips_x * ((Q.lv[i].y_hi - Q.lv[i].y_lo + rows - 1) / rows);
    }
    Q.total_tasks = nt;
  }
  trace_mark(lc, "pool_begin");
  bool& attr_set = CAP <= 4 ? lc->ent_attr_set : lc->ent_attr_batch;
  if (!attr_set) {
    FC_CUDA(lc, cudaFuncSetAttribute(entropy_all_kernel<2, CAP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, ent_smem<2>()));
    FC_CUDA(lc, cudaFuncSetAttribute(entropy_all_kernel<4, CAP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, ent_smem<4>()));
    attr_set = true;
  }
  for (int k = 0; k < 2; ++k) {
    const EntParamsT<CAP>& Q = PL[k];
    if (Q.n_levels == 0 || Q.total_tasks == 0) continue;
    const int warps = k == 0 ? ent_warps<2>() : ent_warps<4>();
    const int blocks = std::max(
        1, std::min((Q.total_tasks + warps - 1) / warps, lc->sm_count * kEntBlocksPerSm));
    if (k == 0)
      entropy_all_kernel<2, CAP><<<blocks, warps * 32, ent_smem<2>(), lc->stream>>>(Q);
    else
      entropy_all_kernel<4, CAP><<<blocks, warps * 32, ent_smem<4>(), lc->stream>>>(Q);
    FC_CUDA(lc, cudaGetLastError());
    lc->total_launches += 1;
  }
  return FC_OK;
}

int pool_entropy(Ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
                 const int32_t use_tau[4], const int32_t* row_lo, const int32_t* row_hi) {
  EntLevel E[4];
  FC_TRY(entropy_setup(c, strides, caps, taus, use_tau, row_lo, row_hi, E));
  const double* lut[4];
  for (int t = 0; t < 4; ++t) lut[t] = c->lut_set[t] ? c->lut[t].as<double>() : nullptr;
  FC_TRY(entropy_launch<4>(c, E, kLevels, lut));
  FC_CUDA(c, cudaEventRecord(c->pool_ev[1], c->stream));
  return FC_OK;
}

// Phase 1 for a batch of contexts (independent images of one size): their
// levels share the two launches, on the first context's stream, ordered after
// every context's pending work and before any of their later work.
int pool_entropy_batch(Ctx** cs, int n, const int32_t strides[4], const int64_t caps[4],
                       const double taus[4], const int32_t use_tau[4]) {
  if (n < 1) return FC_OK;
  Ctx* lc = cs[0];
  if (n * kLevels > 2 * kEntBatchLevels)
    return set_error(lc, FC_ERR_ARG, "too many contexts for one entropy launch");
  std::vector<EntLevel> all((size_t)n * kLevels);
  for (int i = 0; i < n; ++i) {
    Ctx* c = cs[i];
    if (c->device != lc->device) return set_error(lc, FC_ERR_ARG, "contexts on different devices");
    if (c->width != lc->width || c->height != lc->height)
      return set_error(lc, FC_ERR_ARG, "batch images must share one size");
    FC_TRY(entropy_setup(c, strides, caps, taus, use_tau, nullptr, nullptr, &all[(size_t)i * kLevels]));
    if (i > 0) {  // lc's stream waits for context i's buffers and counters
      FC_CUDA(c, cudaEventRecord(c->pool_ev[0], c->stream));
      FC_CUDA(lc, cudaStreamWaitEvent(lc->stream, c->pool_ev[0], 0));
    }
  }
  const double* lut[4];
  for (int t = 0; t < 4; ++t) lut[t] = lc->lut_set[t] ? lc->lut[t].as<double>() : nullptr;
  FC_TRY(entropy_launch<kEntBatchLevels>(lc, all.data(), (int)all.size(), lut));
  FC_CUDA(lc, cudaEventRecord(lc->pool_ev[1], lc->stream));
  for (int i = 1; i < n; ++i) {  // every context's later work after the launches
    FC_CUDA(cs[i], cudaStreamWaitEvent(cs[i]->stream, lc->pool_ev[1], 0));
    FC_CUDA(cs[i], cudaEventRecord(cs[i]->pool_ev[1], cs[i]->stream));
  }
  return FC_OK;
}

// Phase 2: ranking, truncation and the survivors' tiles / moments.  sel:
// per-level threshold-survivor counts known to the host (after an all-gather
// of the slices), or nullptr: read back the device counters (the one
// synchronisation of the pool build).  On return the pool sizes are known;
// the survivor data is produced in stream order.
int pool_rank(Ctx* c, const int64_t* sel, int64_t out_sizes[4]) {
  const int64_t* caps = c->pool_caps;
  const int32_t* use_tau = c->pool_use_tau;
  const int* nx_l = c->pool_nx;
  const int* ny_l = c->pool_ny;
  int* d_nsel = reinterpret_cast<int*>(c->count_buf.ptr);
  int* h_nsel = c->pool_rb.as<int>();
  int any_tau = 0;
  for (int li = 0; li < kLevels; ++li) any_tau |= use_tau[li];
  // ---- caps without a threshold: every window is ranked (cap 1: argmin) ----
  // Sort jobs (key, window) ascending = entropy descending, raster ascending
  // (pool.py:171 argsort(-ent, kind="stable")): the window ids in rank order
  // land in win_val2 and the level keeps the first `count` of them.
  struct SortJob {
    Level* L;
    int64_t n;
  };
  SortJob jobs[kLevels];
  int n_jobs = 0;
  for (int li = 0; li < kLevels; ++li) {
    Level& L = c->lv[li];
    const int64_t nwin = (int64_t)nx_l[li] * ny_l[li];
    if (use_tau[li]) continue;
    if (caps[li] == 1) {
      FC_TRY(argmin_windows(c, L.win_key.as<uint64_t>(), nwin, L.win_key2.as<uint64_t>(),
                            L.win_val2.as<uint32_t>()));
      L.count = 1;
    } else {
      jobs[n_jobs++] = SortJob{&L, nwin};
      L.count = std::min<int64_t>(caps[li], nwin);
    }
  }
  if (any_tau && sel) {
    for (int li = 0; li < kLevels; ++li) h_nsel[li] = (int)sel[li];
  } else if (any_tau) {
    FC_CUDA(c, cudaMemcpyAsync(h_nsel, d_nsel, 4 * kLevels, cudaMemcpyDeviceToHost, c->stream));
    trace_mark(c, "pool_entropy_done");
    FC_TRY(sync_stream(c));
    trace_mark(c, "pool_sync");
  }
  // ---- threshold survivors (entropy > tau), then every ranked set ----
  for (int li = 0; li < kLevels; ++li) {
    if (!use_tau[li]) continue;
    Level& L = c->lv[li];
    const int64_t nwin = (int64_t)nx_l[li] * ny_l[li];
    const int nsel = h_nsel[li];
    if (nsel == 0) {
      // caps are >= 1 (pool.py:47-48): keep the single highest-entropy window;
      // the entropy kernel wrote no keys for this level, so rebuild them
      gather_all_keys_kernel<<<(unsigned)((nwin + 255) / 256), 256, 0, c->stream>>>(
          L.win_ent.as<double>(), nwin, L.win_key.as<uint64_t>());
      c->total_launches += 1;
      FC_TRY(argmin_windows(c, L.win_key.as<uint64_t>(), nwin, L.win_key2.as<uint64_t>(),
                            L.win_val2.as<uint32_t>()));
      L.count = 1;
      continue;
    }
    // every survivor is ranked, then the level keeps the first cap of them
    // (pool.py:171 argsort(-ent, stable)[:cap] over the threshold set)
    L.count = std::min<int64_t>(nsel, caps[li]);
    jobs[n_jobs++] = SortJob{&L, nsel};
  }
  {
    // small sets: chunk sorts + pairwise chunk ranks (one launch each for all
    // levels); large sets (more than kMaxChunks chunks): chunk sorts, then
    // merge passes
    int64_t max_small = 0;
    for (int j = 0; j < n_jobs; ++j)
      if (jobs[j].n <= (int64_t)kMaxChunks * kChunk) max_small = std::max(max_small, jobs[j].n);
    // 1024-element chunks while every small set fits kMaxChunks of them
    // (shorter block sorts; c2: -1% per step), else 2048 (FC_POOL_CHUNK forces one)
    const int chunk = c->pool_chunk == kChunk        ? kChunk
                      : c->pool_chunk == kChunkSmall ? kChunkSmall
                      : max_small <= kMaxChunks * kChunkSmall ? kChunkSmall
                                                              : kChunk;
    SortParams SP{}, SPL{};
    Level* large_lv[kLevels] = {};
    int chunks = 0, lchunks = 0;
    for (int j = 0; j < n_jobs; ++j) {
      Level& L = *jobs[j].L;
      const int64_t n = jobs[j].n;
      if (n <= (int64_t)kMaxChunks * chunk) {
        SortLevel& S = SP.lv[SP.n_levels++];
        S.key = L.win_key.as<uint64_t>();
        S.val = L.win_val.as<uint32_t>();
        S.out = L.win_val2.as<uint32_t>();
        S.count = (int)n;
        S.chunk_begin = chunks;
        chunks += (int)((n + chunk - 1) / chunk);
      } else {
        large_lv[SPL.n_levels] = &L;
        SortLevel& S = SPL.lv[SPL.n_levels++];
        S.key = L.win_key.as<uint64_t>();
        S.val = L.win_val.as<uint32_t>();
        S.out = L.win_val2.as<uint32_t>();
        S.count = (int)n;
        S.chunk_begin = lchunks;
        lchunks += (int)((n + kChunk - 1) / kChunk);
      }
    }
    SP.total_chunks = chunks;
    SPL.total_chunks = lchunks;
    if (chunks > 0) {
      RankLevel RL[4] = {};
      int pairs = 0;
      for (int k = 0; k < SP.n_levels; ++k) {
        RL[k].nch = (SP.lv[k].count + chunk - 1) / chunk;
        RL[k].pair_begin = pairs;
        pairs += RL[k].nch * RL[k].nch;
      }
      for (int k = SP.n_levels; k < 4; ++k) RL[k].pair_begin = 1 << 30;
      FC_CUDA(c, c->pool_rank.reserve((size_t)chunks * chunk * 4));
      int32_t* rank = c->pool_rank.as<int32_t>();
      if (chunk == kChunkSmall) {
        chunk_sort_kernel<kChunkSmall><<<chunks, kChunkSmall / 2, 0, c->stream>>>(SP, rank);
        chunk_pair_rank_kernel<kChunkSmall><<<pairs, kChunkSmall / 2, 0, c->stream>>>(
            SP, RL[0], RL[1], RL[2], RL[3], rank);
        rank_scatter_kernel<kChunkSmall>
            <<<chunks * (kChunkSmall / 256), 256, 0, c->stream>>>(SP, rank);
      } else {
        chunk_sort_kernel<kChunk><<<chunks, kChunk / 2, 0, c->stream>>>(SP, rank);
        chunk_pair_rank_kernel<kChunk><<<pairs, kChunk / 2, 0, c->stream>>>(SP, RL[0], RL[1], RL[2],
                                                                           RL[3], rank);
        rank_scatter_kernel<kChunk><<<chunks * (kChunk / 256), 256, 0, c->stream>>>(SP, rank);
      }
      FC_CUDA(c, cudaGetLastError());
      c->total_launches += 3;
    }
    if (lchunks > 0) {
      chunk_sort_kernel<kChunk><<<lchunks, kChunk / 2, 0, c->stream>>>(SPL, nullptr);
      c->total_launches += 1;
      for (int k = 0; k < SPL.n_levels; ++k) {
        const SortLevel& S = SPL.lv[k];
        Level& L = *large_lv[k];
        uint64_t* kb[2] = {L.win_key.as<uint64_t>(), L.win_key2.as<uint64_t>()};
        uint32_t* vb[2] = {L.win_val.as<uint32_t>(), L.win_val2.as<uint32_t>()};
        int cur = 0;
        const int64_t n = S.count;
        const unsigned grid = (unsigned)((n + kMergeTile - 1) / kMergeTile);
        for (int64_t width = kChunk; width < n; width *= 2, cur ^= 1) {
          merge_pass_kernel<<<grid, 256, 0, c->stream>>>(kb[cur], vb[cur], kb[cur ^ 1], vb[cur ^ 1],
                                                         n, width);
          c->total_launches += 1;
        }
        if (cur == 0)  // the ranked ids must end in win_val2
          FC_CUDA(c, cudaMemcpyAsync(vb[1], vb[0], (size_t)n * 4, cudaMemcpyDeviceToDevice, c->stream));
      }
      FC_CUDA(c, cudaGetLastError());
    }
  }
  SurvParams SV{};
  int64_t swarps = 0;
  // pool origins go straight to pinned host memory (the stream header needs
  // them on the host; no copy nodes later)
  {
    int64_t total = 0;
    for (int li = 0; li < kLevels; ++li) {
      c->coords_off[li] = total;
      total += c->lv[li].count;
    }
    FC_CUDA(c, c->coords_pinned.reserve(total * 4 + 16));
    c->coords_valid = true;  // valid once the stream has passed the survivors kernel
  }
  for (int li = 0; li < kLevels; ++li) {
    Level& L = c->lv[li];
    const int64_t E = L.count;
    FC_TRY(alloc_level(c, L, E));
    SurvLevel& V = SV.lv[li];
    V.order = L.win_val2.as<uint32_t>();
    V.ent_all = L.win_ent.as<double>();
    V.count = E;
    V.B = L.side;
    V.nx = nx_l[li];
    V.stride = L.stride;
    V.warp_begin = swarps;
    V.xy = c->coords_pinned.as<uint32_t>() + c->coords_off[li];
    V.ent = L.ent.as<double>();
    V.tiles = L.tiles.as<uint8_t>();
    V.sum = L.sum.as<int32_t>();
    V.sumsq = L.sumsq.as<int64_t>();
    V.mean = L.mean.as<double>();
    V.cnorm = L.cnorm.as<double>();
    const int per = 32 / L.side;  // survivors per warp (one lane per decimated row)
    swarps += ((E + per - 1) / per + 7) / 8 * 8;  // levels start on block boundaries
    out_sizes[li] = E;
  }
  SV.total_warps = swarps;
  SV.nsel_reset = d_nsel;
  if (swarps > 0) {
    survivors_all_kernel<<<(unsigned)((swarps * 32 + 255) / 256), 256, 0, c->stream>>>(
        c->img_ptr, c->width, (int64_t)c->width * c->height, SV);
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
    c->nsel_clean = true;
  }
  FC_CUDA(c, cudaEventRecord(c->pool_ev[2], c->stream));
  c->pool_timed = true;
  trace_mark(c, "pool_launched");
  return FC_OK;
}

int pool_build(Ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
               const int32_t use_tau[4], int64_t out_sizes[4]) {
  FC_TRY(pool_entropy(c, strides, caps, taus, use_tau, nullptr, nullptr));
  return pool_rank(c, nullptr, out_sizes);
}

// After pool_entropy over a slice: the level's window buffers (device) and
// its local threshold-survivor count (one synchronisation).
int pool_window_buffers(Ctx* c, int li, void** key, void** val, void** ent, int64_t* nx,
                        int64_t* ny, int64_t* local_sel) {
  Level& L = c->lv[li];
  if (key) *key = L.win_key.ptr;
  if (val) *val = L.win_val.ptr;
  if (ent) *ent = L.win_ent.ptr;
  if (nx) *nx = c->pool_nx[li];
  if (ny) *ny = c->pool_ny[li];
  if (local_sel) {
    int v = 0;
    FC_CUDA(c, cudaMemcpyAsync(&v, reinterpret_cast<int*>(c->count_buf.ptr) + li, 4,
                               cudaMemcpyDeviceToHost, c->stream));
    FC_TRY(sync_stream(c));
    *local_sel = v;
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
