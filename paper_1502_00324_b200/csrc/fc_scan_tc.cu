// tcgen05 int8 contraction for the exhaustive range-domain search (proposed
// mode, range sides 16 / 8 / 4).  Replaces the inner loops of
// _scan.py:29-61 for every (range, domain, isometry, s) candidate.
//
// Algebra (range m with offset o = rint(rmean), candidate column c = (e, si)
// with base operand q = rint(s*(d - dmean)), isometry iso applied to the range
// as a pixel permutation r_iso; Q1 = sum q, Q2 = sum q^2 = 2*hq + par):
//     err = sum_k (q_k + o - r_iso,k)^2                 (no clamping)
//         = key2 + R_m,   key2 = 2*kh + par_c,   R_m = sum (r - o)^2,
//     kh  = <-q_c, r_iso> + hq_c + o * Q1_c .
// All of kh comes out of ONE tensor-core contraction: the K dimension holds
// the -q planes against the permuted range (u8 x s8) plus an extra K block in
// which every A row carries constant weights (255..., 1, 1) and its own
// offset (o, o), and every B column carries hq in base-255 digits (each
// <= 127) and Q1 split into two s8 halves.
//
// Ordering without rescans: par = Q2 & 1 = Q1 & 1 (q^2 == q mod 2), so the
// columns are laid out in two groups, even-Q1 then odd-Q1, each in ascending
// candidate order and padded to whole 256-column tiles.  Inside a tile key2 =
// 2*kh + par_tile is a monotone function of kh; key2 values of different
// groups never tie.  Tiles are scanned in decreasing column order, so inside a
// group a later-visited (smaller) column wins ties.  Each TMEM row (range,
// isometry) keeps a running (key2, column) with ONE VIMNMX3 per two
// accumulator elements and locates the first argmin column of a 64-column
// block only when the block improves (or ties) the row.  The final packed key
// (err << 32) | c per range is reduced with shuffles and atomicMin, giving the
// reference's lexicographically first minimum independent of scheduling.
//
// Clamping: the GEMM error is exact unless some pixel of q + o leaves
// [0, 255]; it is then an UPPER bound of the true error for the SAME
// candidate index, so keeping it in the argmin is harmless as long as every
// clamp-active (range, column) pair is ALSO evaluated exactly.  The host
// buckets ranges by o and launches the exact CUDA-core kernel on the columns
// whose qmin < -o or qmax > 255 - o (prefixes of two sorted column lists).
//
// Kernel layout: persistent, one CTA per SM, 20 warps:
//   warp 0  producer: cp.async.bulk (TMA engine) of the A row tiles and the
//           B column tiles + their column map into a STAGES-deep ring
//   warp 1  MMA issuer (warp-uniform, elect.sync inside the asm):
//           tcgen05.mma.kind::i8, M=128, N=256, K=32 per instruction, into one
//           of two TMEM accumulators (2 x 256 columns = all 512 TMEM columns)
//   warp 2  TMEM allocator
//   warps 4..19 epilogue, 4 per TMEM sub-partition (one per 64-column
//           quarter), all draining each accumulator in turn:
//           tcgen05.ld 32x32b + VIMNMX3 running minimum, per-range atomicMin
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "fc_internal.cuh"
#include "fc_tc_ptx.cuh"

namespace fcb {
namespace {

constexpr int kTileN = 256;      // columns per B stage tile
constexpr int kTileM = 128;      // rows per row tile = 16 ranges x 8 isometries
constexpr int kAccN = 128;       // columns per MMA / TMEM accumulator (half a B tile)
constexpr int kNumAcc = 4;       // TMEM accumulators (4 x 128 columns = all 512)
constexpr int kIssuers = 4;      // MMA warps, one per accumulator
constexpr int kEpiBase = kIssuers;  // first epilogue warp (warps 0-3: MMA issuers, warp 0 also the producer)
constexpr int kEpiWarps = 16;    // two groups of 8 (one column half each), 4 per TMEM sub-partition
constexpr int kThreads = (kEpiBase + kEpiWarps) * 32;
// Accumulator release: named barriers 3..6, one per accumulator; the 8 warps
// of its epilogue group arrive (bar.arrive, non-blocking), its issuer warp
// waits (bar.sync: blocked without issuing, where an mbarrier try_wait loop
// took issue slots from the epilogue warps of its sub-partition).
constexpr uint32_t kReleaseBar = 3;
constexpr uint32_t kReleaseThreads = (kEpiWarps / 2 + 1) * 32;
constexpr int kSmemBudget = 227 * 1024;  // the opt-in maximum per block
constexpr int kNone = 0x7fffffff;

// Unit decomposition of one launch, computed on the device from the range
// count (level_plan_kernel) so the host never waits for it.  The work is the
// (row group g, column tile t) pairs, split into segments (g, tiles t1-1 down
// to t0), each costing one A load and one column resolution:
//  * mode 0 (B operand fits L2): pairs in the linear order p = g * ntiles + j
//    (j-th tile of group g counted from the LAST tile); CTA b takes the
//    contiguous share [P*b/grid, P*(b+1)/grid), i.e. a few segments, so every
//    CTA gets the same number of tile MMAs to within one pair;
//  * mode 1 (B larger than L2): units (g, span of ct tiles), u = span * n_rg + g,
//    dealt round-robin, so the CTAs work on the same span at the same time
//    and B streams from HBM about once per span (ct minimises the makespan).
struct TcPlan {
  int M;           // ranges
  int n_rgroups;   // groups of RG row tiles
  int n_pairs;     // n_rgroups * ntiles
  int rows_pad;    // n_rgroups * RG * 128
  int ntiles;      // B tiles of the level (TcDims)
  int mode;        // 0: contiguous pair shares, 1: round-robin span units
  int ct;          // mode 1: tiles per span
  int n_units;     // mode 1: spans * n_rgroups
};

__device__ __forceinline__ void cta_share(int P, int& p0, int& p1) {
  p0 = (int)((long long)P * blockIdx.x / gridDim.x);
  p1 = (int)((long long)P * (blockIdx.x + 1) / gridDim.x);
}

// Next segment of the share: row group g, tiles t1-1 down to t0.
__device__ __forceinline__ bool next_seg(int& p, int p1, int ntiles, int& g, int& t0, int& t1) {
  if (p >= p1) return false;
  g = p / ntiles;
  const int gb = g * ntiles;
  const int pe = min(p1, gb + ntiles);
  t1 = ntiles - (p - gb);
  t0 = ntiles - (pe - gb);
  p = pe;
  return true;
}

// The CTA's segments in either mode (every role walks the same sequence).
struct SegIter {
  int mode, ntiles, n_rg, ct, n_units, p, p1;
  __device__ __forceinline__ explicit SegIter(const TcPlan& pl)
      : mode(pl.mode), ntiles(pl.ntiles), n_rg(pl.n_rgroups), ct(pl.ct), n_units(pl.n_units) {
    if (mode == 0) {
      cta_share(pl.n_pairs, p, p1);
    } else {
      p = blockIdx.x;
      p1 = n_units;
    }
  }
  __device__ __forceinline__ bool next(int& g, int& t0, int& t1) {
    if (mode == 0) return next_seg(p, p1, ntiles, g, t0, t1);
    if (p >= n_units) return false;
    g = p % n_rg;
    t0 = (p / n_rg) * ct;
    t1 = min(ntiles, t0 + ct);
    p += gridDim.x;
    return true;
  }
};

// Clamp corrections: a warp handles fix_rpu ranges x fix_cols columns per
// unit (n = 256: one column per lane, the few pairs of B = 16 need
// parallelism).  Proposed mode batches the ranges of a unit (they share the
// job's offset, so a column's clipped pixels are formed once per unit);
// baseline mode forms the offset per (range, column): one range per unit.
__host__ __device__ constexpr int fix_cpl(int n, bool batched) {
  return n >= 256 ? 1 : (batched && n == 64) ? 2 : 4;
}
__host__ __device__ constexpr int fix_cols(int n, bool batched) { return 32 * fix_cpl(n, batched); }
__host__ __device__ constexpr int fix_rpu(int n, bool batched) {
  return (!batched || n >= 256) ? 1 : n == 64 ? 8 : 16;
}

// Clamp-correction plan (FixPlan) of one level.
struct FixPlan {
  int n_jobs;
  int rpu;                // ranges per unit (proposed mode batches a job's ranges)
  long long total_units;  // (range, columns-per-unit chunk) units; prefix[] counts them too
  long long fix_pairs;
  unsigned long long next_unit;  // work counter of the corrections fused into tc_scan_kernel
};

// Clamp corrections: one warp per unit = one range x CPL*32 consecutive
// columns of a job (job j: ranges sorted_ranges[r_off, r_off + r_cnt) x the
// first col_cnt columns of reach list `list`), CPL columns per lane.  The
// exact error of all 8 isometries follows _scan.py:47-55 (clip(q + o) - r,
// squared, summed): a column's clipped pixels are packed to bytes once per
// 16-pixel chunk and compared with the range's isometry rows, read straight
// from the A operand (its first n bytes of K are r[inv_iso[k]]; warp-uniform
// broadcast loads, shared by the lane's columns).  Minimum over the lane's
// columns, then the warp (err, then candidate index), one atomicMin per unit.
struct FixArgs {
  const int16_t* qbase;
  const uint8_t* a_tiles;
  const int32_t* roff;
  const int4* jobs;
  const long long* prefix;     // unit prefix per job (global; copied to smem by the kernel)
  FixPlan* fplan;
  const int32_t* sorted_ranges;
  const int32_t* list_low;
  const int32_t* list_high;
  unsigned long long* keys;
  int S, kpad, n;
  // baseline mode: the offset depends on (range, column), formed as the
  // reference does from the exact means (roff then holds the range bucket)
  int baseline;
  const double* rmean;
  const double* dmean;
  const double* svals;
};

template <int N, int CPL>
__device__ __forceinline__ void fix_unit(const FixArgs& F, const long long* __restrict__ pre,
                                         int n_jobs, long long u, int lane, uint4* __restrict__ a_s) {
  constexpr int kCols = 32 * CPL;
  int lo = 0, hi = n_jobs - 1;  // last job with prefix <= u (warp-uniform)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int4 job = F.jobs[lo];  // {list, r_off, r_cnt, col_cnt}
  const long long local = u - pre[lo];
  const unsigned ncc = (unsigned)(job.w + kCols - 1) / kCols;
  const unsigned ri = local < 0x7fffffffll ? (unsigned)local / ncc : (unsigned)(local / ncc);
  const int c0 = (int)((unsigned)(local - (long long)ri * ncc) * (unsigned)kCols);
  const int m = F.sorted_ranges[job.y + ri];
  const int32_t* list = job.x ? F.list_high : F.list_low;
  int col[CPL];
  bool valid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ci = c0 + c * 32 + lane;
    valid[c] = ci < job.w;
    col[c] = valid[c] ? list[ci] : list[c0];  // padding lanes repeat a real column
  }
  unsigned o2c[CPL];
  if (F.baseline) {
    const double rm = F.rmean[m];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int e = col[c] / F.S, si = col[c] - e * F.S;
      const unsigned o = (unsigned)baseline_offset(rm, F.svals[si], F.dmean[e]);
      o2c[c] = o | (o << 16);
    }
  } else {
    const unsigned o = (unsigned)F.roff[m];
#pragma unroll
    for (int c = 0; c < CPL; ++c) o2c[c] = o | (o << 16);
  }
  const int64_t row0 = (int64_t)m * 8;  // the range's 8 isometry rows: one 8-row core block
  const uint8_t* abase = F.a_tiles + (row0 >> 7) * ((int64_t)kTileM * F.kpad) +
                         ((int)(row0 & 127) >> 3) * 128;
  // the rows are staged in shared memory first (all loads in flight at once)
  __syncwarp();
  for (int i = lane; i < 8 * (N / 16); i += 32)
    a_s[i] = __ldg(reinterpret_cast<const uint4*>(abase + (i >> 3) * (kTileM * 16) + (i & 7) * 16));
  __syncwarp();
  unsigned acc[CPL][8];
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int iso = 0; iso < 8; ++iso) acc[c][iso] = 0u;
#pragma unroll 2
  for (int kc = 0; kc < N / 16; ++kc) {
    uint4 r4[8];
#pragma unroll
    for (int iso = 0; iso < 8; ++iso) r4[iso] = a_s[kc * 8 + iso];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int16_t* qc = F.qbase + (int64_t)col[c] * N + kc * 16;
      const uint4 qa = __ldg(reinterpret_cast<const uint4*>(qc));
      const uint4 qb = __ldg(reinterpret_cast<const uint4*>(qc + 8));
      const unsigned qw[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      unsigned x4[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        // clip(q + o, 0, 255) on int16 pairs, then packed to 4 bytes
        const unsigned lo2 = __vmins2(__vmaxs2(__vadd2(qw[2 * w], o2c[c]), 0u), 0x00ff00ffu);
        const unsigned hi2 = __vmins2(__vmaxs2(__vadd2(qw[2 * w + 1], o2c[c]), 0u), 0x00ff00ffu);
        x4[w] = __byte_perm(lo2, hi2, 0x6420);
      }
#pragma unroll
      for (int iso = 0; iso < 8; ++iso) {
        unsigned a = acc[c][iso], d;
        d = __vabsdiffu4(x4[0], r4[iso].x); a = __dp4a(d, d, a);
        d = __vabsdiffu4(x4[1], r4[iso].y); a = __dp4a(d, d, a);
        d = __vabsdiffu4(x4[2], r4[iso].z); a = __dp4a(d, d, a);
        d = __vabsdiffu4(x4[3], r4[iso].w); a = __dp4a(d, d, a);
        acc[c][iso] = a;
      }
    }
  }
  unsigned long long best = ~0ull;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    // err <= 256 * 255^2 < 2^24: (err << 3 | iso) orders by err, then iso
    unsigned k = acc[c][0] << 3;
#pragma unroll
    for (int iso = 1; iso < 8; ++iso) k = min(k, (acc[c][iso] << 3) | (unsigned)iso);
    // candidate index (e * 8 + iso) * S + si with e * S = col - si
    const int S = F.S;
    const int si = S == 1 ? 0 : (S == 2 ? (col[c] & 1) : col[c] % S);
    const unsigned cidx = (unsigned)(8 * (col[c] - si) + (int)(k & 7) * S + si);
    const unsigned long long key = ((unsigned long long)(k >> 3) << 32) | cidx;
    if (valid[c] && key < best) best = key;
  }
  const unsigned err = (unsigned)(best >> 32);  // 0xffffffff: no valid column
  const unsigned werr = __reduce_min_sync(0xffffffffu, err);
  const unsigned widx = __reduce_min_sync(0xffffffffu, err == werr ? (unsigned)best : 0xffffffffu);
  if (lane == 0 && werr != 0xffffffffu)
    atomicMin(&F.keys[m], ((unsigned long long)werr << 32) | widx);
}

struct TcParams {
  const uint8_t* a_tiles;    // [rt_pad][128 * kpad]
  const int4* row_meta;      // [rt_pad * 128] {o, R, m, unused}
  const int8_t* b_tiles;     // [ntiles][256 * kpad]
  const int32_t* colmap;     // [ntiles * 256] slot -> column (-1 = padding)
  const int2* tile_info;     // [ntiles] {parity of the tile's group, valid slots}
  unsigned long long* keys;  // [M]
  int S;
  int kpad;
  int rg;          // row tiles per unit (A resident in smem)
  int stages;      // B ring depth (in K chunks)
  int kc;          // K bytes per ring stage: kpad, or a divisor of it for long K
  int base;        // baseline mode: u8 x u8 contraction, errors formed in the epilogue
  int real;        // real-valued slope search (s-histogram analysis): u8 x u8, fp64 epilogue
  int shift;       // log2(B*B)
  const int4* bconst;  // baseline: per slot {W', 2 Q1, Q2, tie mask} (qprep_level);
                       // real: per slot {D1, flat, rcp(cnorm) / n^2 as two words}
  const double* cnorm;             // real: centered norm per entry
  unsigned long long* real_out;    // real: per range {err bits, e * 8 + iso}, 128-bit CAS-min
  const TcPlan* plan;
  FixArgs fix;
  unsigned long long* tspan;  // optional {start, end} slots (global ns)
};

__host__ __device__ inline uint32_t a_bytes(const TcParams& p) { return p.rg * kTileM * p.kpad; }
__host__ __device__ inline uint32_t b_bytes(const TcParams& p) { return kTileN * p.kpad; }
__host__ __device__ inline uint32_t stage_bytes(const TcParams& p) { return kTileN * p.kc; }
// per epilogue thread and resident row tile: {best key2, tile * 8 + 8-column group}
// (real mode: {best err, screening threshold} as two doubles)
__host__ __device__ inline uint32_t best_offset(const TcParams& p) {
  return a_bytes(p) + p.stages * stage_bytes(p);
}
// baseline mode: each thread's range sum R1 per resident row tile; real mode:
// {rnorm, R1} doubles then the best column; then two double-buffered
// 256-column constant tables (one per epilogue group)
__host__ __device__ inline uint32_t r1_offset(const TcParams& p) {
  return best_offset(p) + p.rg * kEpiWarps * 32 * (p.real ? 16 : 8);
}
__host__ __device__ inline uint32_t const_offset(const TcParams& p) {
  return r1_offset(p) + (p.base ? p.rg * kEpiWarps * 32 * 4 : p.real ? p.rg * kEpiWarps * 32 * 20 : 0);
}
// column constants: baseline, per epilogue group, 2 tiles x 256 x int4;
// real mode, per epilogue warp, 2 tiles x its 128 columns x {D1, sqrt(cnorm)}
__host__ __device__ inline uint32_t bar_offset(const TcParams& p) {
  return const_offset(p) + (p.real ? kEpiWarps * 2 * 128 * 8 : p.base ? 2 * 2 * kTileN * 16 : 0);
}
__host__ __device__ inline uint32_t smem_bytes(const TcParams& p) {
  const uint32_t raw = bar_offset(p) + (2 * p.stages + 2 * kNumAcc + 2) * 8 + 16;
  return raw < 116 * 1024 ? 116 * 1024 : raw;  // one CTA (owning all 512 TMEM columns) per SM
}

// Minimum of 8 consecutive values v[o..o+7]: 3 VIMNMX3 + 1 VIMNMX.
template <int O>
__device__ __forceinline__ int min8(const int (&v)[32]) {
  return __vimin3_s32(__vimin3_s32(v[O], v[O + 1], v[O + 2]), __vimin3_s32(v[O + 3], v[O + 4], v[O + 5]),
                      min(v[O + 6], v[O + 7]));
}

// u8 x s8 (proposed) / u8 x u8 (baseline) four-way dot product accumulate
// (the MMA's kind::i8 arithmetic).
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ int dp4a_uu(uint32_t a, uint32_t b, int c) {
  int d;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Baseline mode: the candidate's error minus the range's R2 from the
// contraction value acc = <q, r_iso> (_scan.py:38-55 without clamping):
//   o = clip(rint(rmean - s * dmean), 0, 255) from R1 and the column's W' /
//       tie mask (see qprep_level: exact integer form of the fp64 rounding),
//   e = Q2 + o (2 Q1 + n o - 2 R1) - 2 acc      (+ R2 = sum (q + o - r)^2).
// Clamp-active pairs make this an upper bound of the true error; they are
// corrected exactly by fix_pairs_kernel like in proposed mode.
__device__ __forceinline__ int base_err(int acc, int4 k, int R1, int X, int shift, int hn1) {
  int t = R1 + k.x;
  t += ((t - hn1) >> shift) & 1 & k.w;  // round half to even when V is integral
  const int o = max(t >> shift, 0);
  return o * (k.y - X + (o << shift)) + k.z - 2 * acc;
}

// Row state: best2 = 2*kh + par of the row's best so far and where it lies
// (tile, 8-column group of this thread's 64-column slice); the exact column
// inside the group is resolved once per segment by recomputing its 8 dot
// products.  Tiles are visited in DECREASING column order (the entropy-ranked
// pool puts the usually-better low-entropy domains last, so scanning backwards
// finds them first and the running minimum rarely changes); an equal key2 at a
// smaller column must then win, so a block updates iff 2*m + par <= best2
// <=>  m < ((best2 - par) >> 1) + 1.
// (32-bit: best2 <= 0x7fffffff and par in {0, 1} cannot overflow.)
__device__ __forceinline__ int improve_limit(int best2, int par) {
  return ((best2 - par) >> 1) + 1;
}

// (tile, row tile) pair counter H and column half h -> accumulator
// acc = 2 * (H & 1) + h: MMA warp acc issues it, epilogue group H & 1 drains
// both halves of its pairs.  Accumulator acc is used by every other pair, so
// its n-th use has phase parity n & 1 with n = H >> 1.

struct EpiCtx {
  uint32_t kB, bar_base, tmem_base;
  int RG, KPAD, warp, lane;
  TcPlan plan;
};

// Epilogue role (warps kEpiBase .. kEpiBase + 15): group gq (8 warps, two
// per TMEM sub-partition) takes the pairs with (H & 1) == gq, i.e. the
// accumulators 2 gq (column half 0) and 2 gq + 1 (half 1); each warp one
// 64-column slice of each half.  Per accumulator one wave of two
// tcgen05.ld x32, released right after the loads; the per-pair bookkeeping
// (row state, tile info, loop control) is shared by the two halves.
// BASE (baseline mode): the accumulator holds <q, r_iso>; every value becomes
// the candidate's error (base_err) from the row's range sum and the column's
// constants, which the group stages per tile in shared memory (one 16-byte
// load per thread, double buffered, one named barrier per tile).
template <bool BASE>
__device__ __forceinline__ void epilogue_role(const TcParams& p, uint8_t* smem, const EpiCtx& x) {
  const uint32_t kB = x.kB, bar_base = x.bar_base, tmem_base = x.tmem_base;
  const int RG = x.RG, KPAD = x.KPAD, warp = x.warp, lane = x.lane;
  const int e = warp - kEpiBase;
  const int gq = e >> 3;            // pair parity this group drains
  const int hq = (e >> 2) & 1;      // 64-column slice inside each half
  const int sp = warp & 3;          // TMEM sub-partition (lanes 32*sp .. 32*sp+31)
  const int row = sp * 32 + lane;
  const int S = p.S;
  const int slice = hq * 64;        // tile slot of this thread's slice in half 0 (+128: half 1)
  const uint32_t tm0 = tmem_base + ((uint32_t)(sp * 32) << 16) + (2 * gq) * kAccN + slice;
  const uint32_t tfull0 = bar_base + 8u * (2 * p.stages) + 8u * (2 * gq);
  // this thread's {best2, loc} per resident row tile, stride = 512 threads;
  // loc = tile << 4 | half << 3 | 8-column group
  const uint32_t bst = ptx::smem_u32(smem + best_offset(p)) + (e * 32 + lane) * 8;
  constexpr int kBS = kEpiWarps * 32;
  // baseline: range sums per row tile, the group's column-constant buffers
  const uint32_t r1s = ptx::smem_u32(smem + r1_offset(p)) + (e * 32 + lane) * 4;
  const int4* cbase = reinterpret_cast<const int4*>(smem + const_offset(p)) + gq * 2 * kTileN;
  const int gtid = (e & 7) * 32 + lane;  // thread index inside the group
  const int shift = p.shift, hn1 = (1 << (shift - 1)) - 1;
  uint32_t tcount = 0;
  int4 pre = make_int4(0, 0, 0, 0);
  uint32_t H = 0;
  int g, t0, t1;
  for (SegIter it(x.plan); it.next(g, t0, t1);) {
    for (int r = 0; r < RG; ++r) ptx::sts_v2(bst + r * (kBS * 8), make_int2(kNone, 0));
    if constexpr (BASE) {
      for (int r = 0; r < RG; ++r) {
        const int r1 = p.row_meta[(size_t)(g * RG + r) * kTileM + row].x;
        asm volatile("st.shared.s32 [%0], %1;" ::"r"(r1s + r * (kBS * 4)), "r"(r1) : "memory");
      }
      pre = p.bconst[(size_t)(t1 - 1) * kTileN + gtid];
    }
    // tiles in DECREASING order (see improve_limit); tile_info one tile ahead
    int2 tinfo_next = p.tile_info[t1 - 1];
    for (int t = t1 - 1; t >= t0; --t) {
      const int2 tinfo = tinfo_next;  // {parity, valid slots}
      if (t > t0) tinfo_next = p.tile_info[t - 1];
      const int4* cb = cbase;
      if constexpr (BASE) {
        int4* w = const_cast<int4*>(cbase) + (tcount & 1) * kTileN;
        ++tcount;
        w[gtid] = pre;
        ptx::named_bar_sync(1 + gq, kEpiWarps / 2 * 32);
        if (t > t0) pre = p.bconst[(size_t)(t - 1) * kTileN + gtid];
        cb = w;
      }
      // this group's pairs of the tile: Hr = Ht + r with (Hr & 1) == gq
      const uint32_t Ht = H;
      H += RG;
#pragma unroll 1
      for (int r = (gq ^ (int)(Ht & 1)) & 1; r < RG; r += 2) {
        const uint32_t bst_r = bst + r * (kBS * 8);
        const int2 bs = ptx::lds_v2(bst_r);
        int R1 = 0;
        if constexpr (BASE)
          asm volatile("ld.shared.s32 %0, [%1];" : "=r"(R1) : "r"(r1s + r * (kBS * 4)) : "memory");
        const uint32_t ph = ((Ht + r) >> 1) & 1;
        // half 0 vs earlier tiles: improve_limit (ties go to the later-visited,
        // smaller columns); half 1 vs half 0 of this tile: strictly smaller
        int lim = improve_limit(bs.x, tinfo.x);
        int best_m = kNone, best_loc = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          ptx::mbar_wait_sleep(tfull0 + 8u * h, ph);
          ptx::tc_fence_after();
          int va[32], vb[32];
          ptx::tmem_ld32(tm0 + h * kAccN, va);
          ptx::tmem_ld32(tm0 + h * kAccN + 32, vb);
          ptx::tmem_wait_ld();
          // every value is in registers: release the accumulator
          ptx::tc_fence_before();
          __syncwarp();
          ptx::named_bar_arrive(kReleaseBar + 2 * gq + h, kReleaseThreads);
          const int s0 = h * kAccN + slice;
          if constexpr (BASE) {
            const int X = 2 * R1;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              va[j] = base_err(va[j], cb[s0 + j], R1, X, shift, hn1);
              vb[j] = base_err(vb[j], cb[s0 + 32 + j], R1, X, shift, hn1);
            }
          }
          if (tinfo.y < kTileN) {  // mask padding slots (last tile of a group)
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (s0 + j >= tinfo.y) va[j] = kNone;
              if (s0 + 32 + j >= tinfo.y) vb[j] = kNone;
            }
          }
          int gm[8];
          gm[0] = min8<0>(va);
          gm[1] = min8<8>(va);
          gm[2] = min8<16>(va);
          gm[3] = min8<24>(va);
          gm[4] = min8<0>(vb);
          gm[5] = min8<8>(vb);
          gm[6] = min8<16>(vb);
          gm[7] = min8<24>(vb);
          const int m = min(__vimin3_s32(gm[0], gm[1], gm[2]),
                            __vimin3_s32(__vimin3_s32(gm[3], gm[4], gm[5]), gm[6], gm[7]));
          // the 8-column group is located only when some lane of the warp
          // improves (rare once the row minima settle): the first group
          // holding m (column order)
          const bool imp = m < lim;
          if (__any_sync(0xffffffffu, imp)) {
            int gi = 7;
#pragma unroll
            for (int k = 6; k >= 0; --k) gi = (gm[k] == m) ? k : gi;
            if (imp) {
              best_m = m;
              best_loc = (h << 3) + gi;
              lim = m;
            }
          }
        }
        if (best_m != kNone) ptx::sts_v2(bst_r, make_int2(2 * best_m + tinfo.x, (t << 4) + best_loc));
      }
    }
    // resolve each row's winning 8-column group: recompute its dot products
    // from the global copies of A and B (the shared A slot is already being
    // refilled for the next segment) and take the first column whose value
    // equals the recorded minimum.  Only the candidates at the minimal error
    // of their range (the 8 isometry rows = lanes 8k..8k+7) can win, so just
    // those are resolved, the range's 8 lanes computing the candidate group's
    // 8 dot products together (one L2 round trip per candidate, not 8 x K/16).
    const int chunks = KPAD / 16;
#pragma unroll 1
    for (int r = 0; r < RG; ++r) {
      unsigned long long key = ~0ull;
      const int2 bs = ptx::lds_v2(bst + r * (kBS * 8));
      const int4 rm = p.row_meta[(size_t)(g * RG + r) * kTileM + row];  // {o, R, m, -} | {R1, R2, m, 2 R1}
      const bool valid = bs.x != kNone && rm.z >= 0;
      // error = key2 + R (proposed: key2 = 2 kh + par) | key2 / 2 + R2 (baseline)
      const long long err = valid ? (BASE ? (long long)(bs.x >> 1) : (long long)bs.x) + rm.y : LLONG_MAX;
      long long gmin = err;
      gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, 1));
      gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, 2));
      gmin = min(gmin, __shfl_xor_sync(0xffffffffu, gmin, 4));
      const int gbase = lane & ~7;
      const int j = lane & 7;
      unsigned tied = (__ballot_sync(0xffffffffu, valid && err == gmin) >> gbase) & 0xffu;
      while (__any_sync(0xffffffffu, tied != 0)) {
        const int src = tied ? gbase + __ffs(tied) - 1 : lane;
        const int loc = __shfl_sync(0xffffffffu, bs.y, src);
        const int b2 = __shfl_sync(0xffffffffu, bs.x, src);
        const int R1s = __shfl_sync(0xffffffffu, rm.x, src);
        const int t = loc >> 4;
        const int slot0 = ((loc >> 3) & 1) * kAccN + slice + (loc & 7) * 8;
        int m = 0, kh = 0;
        if (tied) {
          m = (b2 - p.tile_info[t].x) >> 1;
          const int srow = sp * 32 + src;
          const uint8_t* arow = p.a_tiles + (size_t)(g * RG + r) * (kTileM * KPAD) +
                                (srow >> 3) * 128 + (srow & 7) * 16;
          const int8_t* bcol = p.b_tiles + (size_t)t * kB + (slot0 >> 3) * 128 + j * 16;
#pragma unroll 4
          for (int kc = 0; kc < chunks; ++kc) {
            const uint4 a4 = __ldg(reinterpret_cast<const uint4*>(arow + kc * (kTileM * 16)));
            const uint4 b4 = __ldg(reinterpret_cast<const uint4*>(bcol + kc * (kTileN * 16)));
            if constexpr (BASE) {
              kh = dp4a_uu(a4.x, b4.x, kh);
              kh = dp4a_uu(a4.y, b4.y, kh);
              kh = dp4a_uu(a4.z, b4.z, kh);
              kh = dp4a_uu(a4.w, b4.w, kh);
            } else {
              kh = dp4a_us(a4.x, b4.x, kh);
              kh = dp4a_us(a4.y, b4.y, kh);
              kh = dp4a_us(a4.z, b4.z, kh);
              kh = dp4a_us(a4.w, b4.w, kh);
            }
          }
          if constexpr (BASE)
            kh = base_err(kh, p.bconst[(size_t)t * kTileN + slot0 + j], R1s, 2 * R1s, shift, hn1);
        }
        const unsigned hits = (__ballot_sync(0xffffffffu, tied && kh == m) >> gbase) & 0xffu;
        if (tied) {
          const int col = p.colmap[(size_t)t * kTileN + slot0 + __ffs(hits) - 1];
          const int e_idx = col / S, si = col - e_idx * S;
          const unsigned long long k2 =
              ((unsigned long long)gmin << 32) |
              (unsigned long long)((e_idx * 8 + (src & 7)) * S + si);
          key = k2 < key ? k2 : key;
          tied &= tied - 1;
        }
      }
      unsigned long long w = __shfl_xor_sync(0xffffffffu, key, 1);
      key = w < key ? w : key;
      w = __shfl_xor_sync(0xffffffffu, key, 2);
      key = w < key ? w : key;
      w = __shfl_xor_sync(0xffffffffu, key, 4);
      key = w < key ? w : key;
      if ((lane & 7) == 0 && key != ~0ull) atomicMin(&p.keys[rm.z], key);
    }
  }
}

// Real-valued slope search (bench.py:117-139 _real_s_matches), the
// s-histogram analysis: the accumulator holds X = <d, r_iso> (u8 x u8, d the
// decimated domain), and per candidate
//   cross = (n X - D1 R1) / n,  gain = cross^2 / cnorm,  err = max(rnorm - gain, 0)
// with the first minimum of (err, e * 8 + iso) kept (gain = 0 for a flat
// domain).  Every product is an exact integer / n^2 (see fc_real.cu), so the
// fp64 steps below reproduce the reference bit for bit.  Screening: g =
// fl(fl(xn^2) * rcp / n^2) with xn = n X - D1 R1 equals fc_real.cu's
// fl(cross^2 * rcp); g < T = (rnorm - best) - 1e-13 (rnorm + |best|) implies
// that kernel's own rejection test (rnorm - g > best + 1e-14 (rnorm + g),
// rounding included), so only the rare candidates at or above T take its
// exact path.  Each row keeps {best err, T} and the best column in shared
// memory; at the end of a segment the 8 isometry rows of a range reduce
// lexicographically and merge into the range's 128-bit {err bits, index}
// record with a compare-and-swap loop (order independent).
__device__ __forceinline__ void real_cas_min(unsigned long long* slot, unsigned long long eb,
                                             unsigned long long idx) {
  unsigned long long olo = slot[1], ohi = slot[0];  // hint; the CAS re-reads
  for (;;) {
    if (ohi < eb || (ohi == eb && olo <= idx)) return;
    unsigned long long rlo, rhi;
    asm volatile(
        "{\n\t.reg .b128 d, c, v;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 v, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, v;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(rlo), "=l"(rhi)
        : "l"(ohi), "l"(olo), "l"(eb), "l"(idx), "l"(slot)
        : "memory");
    if (rlo == ohi && rhi == olo) return;  // swapped
    ohi = rlo;
    olo = rhi;
  }
}

__device__ __forceinline__ double real_threshold(double rn, double best) {
  return __dsub_rn(__dsub_rn(rn, best), __dmul_rn(1e-13, __dadd_rn(rn, fabs(best))));
}

// The screen's row factor: sT <= sqrt(T) (1 - 1e-5), 0 when T is not above
// 1e-30 (the MUFU reciprocal square root is within 3e-7 of the true value).
// With f = fl32(cross) and the column factor sqn <= sqrt(cnorm) (fp32,
// rounded down), |f| < fl(sT * sqn) gives |cross| < sqrt(T cnorm), so the
// candidate's gain cross^2 / cnorm is below T: it can neither win nor tie.
__device__ __forceinline__ float real_screen_factor(double rn, double best) {
  const float t = __double2float_rd(real_threshold(rn, best));
  return t > 1e-30f ? __fmul_rd(__fmul_rd(t, rsqrtf(t)), 0.99999f) : 0.0f;
}

constexpr int kRC = 16;  // accumulator columns per register chunk (one tcgen05.ld x16)

static_assert(kRC == 16, "the exact path's register select is written for 16 columns");

__device__ __forceinline__ void epilogue_real(const TcParams& p, uint8_t* smem, const EpiCtx& x) {
  const uint32_t bar_base = x.bar_base, tmem_base = x.tmem_base;
  const int RG = x.RG, KPAD = x.KPAD, warp = x.warp, lane = x.lane;
  const int e = warp - kEpiBase;
  const int gq = e >> 3, hq = (e >> 2) & 1, sp = warp & 3;
  const int row = sp * 32 + lane;
  const int slice = hq * 64;
  const uint32_t tm0 = tmem_base + ((uint32_t)(sp * 32) << 16) + (2 * gq) * kAccN + slice;
  const uint32_t tfull0 = bar_base + 8u * (2 * p.stages) + 8u * (2 * gq);
  constexpr int kBS = kEpiWarps * 32;
  const int tix = e * 32 + lane;
  double2* st_best = reinterpret_cast<double2*>(smem + best_offset(p)) + tix;  // {best, sT}
  double2* st_row = reinterpret_cast<double2*>(smem + r1_offset(p)) + tix;     // {rnorm, R1}
  int* st_col = reinterpret_cast<int*>(smem + r1_offset(p) + RG * kBS * 16) + tix;
  const int shift = p.shift, n = 1 << shift;
  const double ninv = 1.0 / (double)n;
  const uint32_t wbuf = ptx::smem_u32(smem + const_offset(p)) + e * 2048;
  uint32_t tcount = 0;
  uint32_t H = 0;
  int g, t0, t1;
  for (SegIter it(x.plan); it.next(g, t0, t1);) {
    for (int r = 0; r < RG; ++r) {
      const int4 rm = p.row_meta[(size_t)(g * RG + r) * kTileM + row];  // {R1, R2, m, 2 R1}
      const double rn = __dmul_rn((double)((long long)n * rm.y - (long long)rm.x * rm.x), ninv);
      st_row[r * kBS] = make_double2(rn, (double)rm.x);
      st_best[r * kBS] = make_double2(DBL_MAX, 0.0);
      st_col[r * kBS] = INT_MAX;
    }
    // the warp's column constants {D1, sqrt(cnorm)} as fp32 (real_prep_kernel's
    // layout) staged by cp.async one tile ahead into its own double buffer:
    // lane l copies 16 bytes (two columns) of each half; no cross-warp sync
    // (lanes 0-7 also pull the warp's cnorm lines of the tile into L1 for
    // the exact path)
    auto stage = [&](int tt, uint32_t buf) {
      const int2* src = reinterpret_cast<const int2*>(p.bconst) + (size_t)tt * kTileN + slice + 2 * lane;
      ptx::cp_async16(wbuf + buf * 1024u + lane * 16u, src);
      ptx::cp_async16(wbuf + buf * 1024u + 512u + lane * 16u, src + kAccN);
      ptx::cp_async_commit();
      if (lane < 8)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.cnorm + (size_t)tt * kTileN + (lane >> 2) * kAccN +
                                                      slice + (lane & 3) * 16));
    };
    stage(t1 - 1, tcount & 1);
    for (int t = t1 - 1; t >= t0; --t) {
      const int valid_slots = p.tile_info[t].y;
      const uint32_t buf = tcount & 1;
      ++tcount;
      ptx::cp_async_wait_all();
      __syncwarp();  // every lane's copies landed; every lane is done with the other buffer
      if (t > t0) stage(t - 1, buf ^ 1);
      // cf: this warp's 128 columns (half h at h * 64)
      const int2* cf = reinterpret_cast<const int2*>(smem + const_offset(p) + e * 2048 + buf * 1024);
      const uint32_t Ht = H;
      H += RG;
#pragma unroll 1
      for (int r = (gq ^ (int)(Ht & 1)) & 1; r < RG; r += 2) {
        const double2 rr = st_row[r * kBS];
        const double rn = rr.x;
        const int nR1 = -(int)rr.y;
        float mR1n = (float)(-rr.y * ninv);  // -R1 / n, exact
        double2 bt = st_best[r * kBS];
        int bcol = st_col[r * kBS];
        bool changed = false;
        const uint32_t ph = ((Ht + r) >> 1) & 1;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          ptx::mbar_wait_sleep(tfull0 + 8u * h, ph);
          ptx::tc_fence_after();
          // the half's 64 columns in chunks of kRC (the accumulator is
          // released after the last load); rn == 0 rows take the shortcut
#pragma unroll 1
          for (int c = 0; c < 64 / kRC; ++c) {
            int v[kRC];
            ptx::tmem_ld16(tm0 + h * kAccN + kRC * c, v);
            ptx::tmem_wait_ld();
            if (c == 64 / kRC - 1) {
              ptx::tc_fence_before();
              __syncwarp();
              ptx::named_bar_arrive(kReleaseBar + 2 * gq + h, kReleaseThreads);
            }
            const int s0 = h * kAccN + slice + kRC * c;
            if (rn == 0.0) {
              // a constant range: every candidate's error is max(0 - gain, 0) = 0,
              // so the first candidate of the slice in column order wins
              const int col = t * kTileN + s0;
              if (c == 0 && s0 < valid_slots && (bt.x > 0.0 || col < bcol)) {
                bt = make_double2(0.0, 0.0);
                bcol = col;
                changed = true;
              }
              continue;
            }
            const int nvalid = valid_slots - s0;
            const uint32_t vmask = nvalid >= kRC ? (1u << kRC) - 1 : nvalid <= 0 ? 0u : (1u << nvalid) - 1;
            float sT = (float)bt.y;
            const int l0 = h * 64 + kRC * c;  // the chunk's first column in the warp's constants
            const int4* cf4 = reinterpret_cast<const int4*>(cf + l0);
            // screen per candidate: f = fl32(X - D1 R1 / n) = fl32(cross) (one
            // FFMA: D1, R1 / n and X < 2^24 are exact in fp32), candidate unless
            // |f| < sT * sqn (see real_screen_factor; flat columns: sqn = inf,
            // f = 0, so they pass only when sT = 0, through the NaN product)
#define FC_REAL_F(D1F, X) __fmaf_rn(__int_as_float(D1F), mR1n, __int2float_rn(X))
#define FC_REAL_PASS(D1F, SQN, X) (!(fabsf(FC_REAL_F(D1F, X)) < __fmul_rn(sT, __int_as_float(SQN))))
            if (bt.x != DBL_MAX) {
              // one predicate-OR per candidate; the slices that pass build the
              // candidate mask below
              bool any = false;
#pragma unroll
              for (int q = 0; q < kRC / 2; ++q) {
                const int4 k = cf4[q];
                any |= FC_REAL_PASS(k.x, k.y, v[2 * q]);
                any |= FC_REAL_PASS(k.z, k.w, v[2 * q + 1]);
              }
              if (!any) continue;
            } else {
              // first slice of a segment (no best yet): a = |f| / sqn is within
              // 3e-7 of sqrt(gain); its maximum over the slice (tracked as a
              // pair, no division per candidate) sets the row factor, so only
              // candidates near the slice's best gain pass -- any other has a
              // gain smaller by more than 1e-4 relative and 1e-12 rnorm, so a
              // larger fp64 error -- plus every candidate whose gain may reach
              // rnorm (error clamped to 0: ties by column)
              float fm = 0.0f, sm = 1.0f;
#pragma unroll
              for (int q = 0; q < kRC; ++q) {
                // (a memory clobber every 4 candidates keeps the constant loads
                // from being hoisted all at once)
                if ((q & 3) == 0) asm volatile("" : : : "memory");
                const int2 k = cf[l0 + q];
                const float a = fabsf(FC_REAL_F(k.x, v[q])), nq = __int_as_float(k.y);
                const bool take = ((vmask >> q) & 1u) && __fmul_rn(a, sm) > __fmul_rn(fm, nq);
                fm = take ? a : fm;
                sm = take ? nq : sm;
              }
              const float amax = __fdividef(fm, sm);
              const float rn32 = __double2float_rd(rn);
              sT = fminf(fminf(__fmul_rn(amax, 0.99994f), amax - __fdividef(2e-12f * rn32, amax)),
                         __fmul_rn(__fmul_rn(rn32, rsqrtf(rn32)), 0.999998f));
            }
            // the mask pass recomputes f from opaque copies of its inputs:
            // common subexpressions with the pass above would keep 64 values
            // live across it (spilled)
            asm volatile("" : "+f"(mR1n), "+f"(sT) : : "memory");
#pragma unroll
            for (int j = 0; j < kRC; ++j) asm volatile("" : "+r"(v[j]));
            uint32_t mask = 0u;
#pragma unroll
            for (int q = 0; q < kRC / 2; ++q) {
              const int4 k = cf4[q];
              mask |= ((uint32_t)FC_REAL_PASS(k.x, k.y, v[2 * q]) << (2 * q)) |
                      ((uint32_t)FC_REAL_PASS(k.z, k.w, v[2 * q + 1]) << (2 * q + 1));
            }
#undef FC_REAL_PASS
#undef FC_REAL_F
            mask &= vmask;
            if (mask == 0u) continue;
            // exact path (rare): X selected from the chunk, then fc_real.cu's steps
            while (mask) {
              const int j = __ffs(mask) - 1;
              mask &= mask - 1;
              int w[kRC / 2];
#pragma unroll
              for (int i = 0; i < kRC / 2; ++i) w[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
              for (int i = 0; i < kRC / 4; ++i) w[i] = (j & 2) ? w[2 * i + 1] : w[2 * i];
#pragma unroll
              for (int i = 0; i < kRC / 8; ++i) w[i] = (j & 4) ? w[2 * i + 1] : w[2 * i];
              const int X = (j & 8) ? w[1] : w[0];
              const int slot = s0 + j;
              const int col = t * kTileN + slot;  // real mode: slots are columns in order
              const double norm = p.cnorm[col];  // prefetched into L1 with the tile's constants
              const double xd = (double)((int)__int_as_float(cf[l0 + j].x) * nR1 + (X << shift));
              const double cross = __dmul_rn(xd, ninv);
              const double cc = __dmul_rn(cross, cross);
              const double gain = norm == 0.0 ? 0.0 : __ddiv_rn(cc, norm);
              const double err = fmax(__dsub_rn(rn, gain), 0.0);
              if (err < bt.x || (err == bt.x && col < bcol)) {
                bt.x = err;
                bt.y = (double)real_screen_factor(rn, err);
                bcol = col;
                changed = true;
              }
            }
          }
        }
        if (changed) {
          st_best[r * kBS] = bt;
          st_col[r * kBS] = bcol;
        }
      }
    }
    // per range: the 8 isometry rows (lanes 8k..8k+7) reduce on (err, e * 8 + iso)
#pragma unroll 1
    for (int r = 0; r < RG; ++r) {
      const int4 rm = p.row_meta[(size_t)(g * RG + r) * kTileM + row];
      const double be = st_best[r * kBS].x;
      const int bcol = st_col[r * kBS];
      unsigned long long eb = (bcol != INT_MAX && rm.z >= 0) ? (unsigned long long)__double_as_longlong(be)
                                                             : ~0ull;
      unsigned long long ix = bcol != INT_MAX ? (unsigned long long)bcol * 8 + (lane & 7) : ~0ull;
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const unsigned long long oe = __shfl_xor_sync(0xffffffffu, eb, o);
        const unsigned long long oi = __shfl_xor_sync(0xffffffffu, ix, o);
        if (oe < eb || (oe == eb && oi < ix)) {
          eb = oe;
          ix = oi;
        }
      }
      if ((lane & 7) == 0 && eb != ~0ull) real_cas_min(p.real_out + 2 * (size_t)rm.z, eb, ix);
    }
  }
}

// Work order (all roles derive it identically): the CTA's share of
// (row group, tile) pairs as segments (cta_share / next_seg; one A load and
// one column resolution per segment); inside a segment: tiles t descending,
// row tiles r; the pair counter H and the column half h select accumulator
// 2 * (H & 1) + h, issued by MMA warp acc and drained by epilogue group
// H & 1.
// CHUNK: the B ring holds K chunks of a tile (long K); a separate
// instantiation, so the whole-tile issue loop keeps its code (the branch
// cost c5 1-3%).
template <int MODE, bool CHUNK>  // MODE 0 proposed, 1 baseline, 2 real-valued slope search
__global__ void __launch_bounds__(kThreads, 1) tc_scan_kernel(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int KPAD = p.kpad, RG = p.rg, STAGES = p.stages;
  const int NC = CHUNK ? KPAD / p.kc : 1;  // ring stages (K chunks) per B tile
  const uint32_t kA = a_bytes(p), kB = b_bytes(p), kStage = stage_bytes(p);
  uint8_t* sA = smem;
  uint8_t* sStage = smem + kA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bar_offset(p));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * kNumAcc + 2);
  const uint32_t bar_base = ptx::smem_u32(bars);
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + b); };
  const uint32_t afull_bar = bar_base + 8u * (2 * STAGES + 2 * kNumAcc);
  const uint32_t aempty_bar = afull_bar + 8u;

  // warp index through a shuffle: ptxas then treats every role branch and
  // the issuers' descriptors as warp-uniform (uniform datapath, no per-MMA
  // R2UR.BROADCAST / divergence checks -- the issue loop halves)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 1);
      ptx::mbar_init(empty_bar(s), kIssuers);  // one commit per MMA warp and tile
    }
    for (int b = 0; b < kNumAcc; ++b) {
      ptx::mbar_init(tfull_bar(b), 1);
    }
    ptx::mbar_init(afull_bar, 1);
    ptx::mbar_init(aempty_bar, kIssuers);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (p.tspan && threadIdx.x == 0) atomicMin(&p.tspan[0], global_ns());

  const TcPlan plan = *p.plan;
  int g, t0, t1;

  if (warp < kIssuers) {
    // ---------------- MMA issuers: warp i owns accumulator i ----------------
    // Four issuing warps keep four 128-column accumulators in flight: the
    // issuing thread's own latency (descriptor set-up, barrier waits, commits)
    // and the commit -> epilogue -> release round trip are both longer than
    // one accumulator's MMA work, so one issuer over two 256-column
    // accumulators left the tensor pipe idle ~40% of the time.  Warp 0 also
    // drives the TMA engine (bulk copies of the A row group per segment and
    // of the B tiles STAGES - 1 ahead, each right after its own MMAs for a
    // tile, so a wait for a ring slot overlaps MMAs already issued); 20 warps
    // = 5 per SM sub-partition keeps the 96-register budget.
    const int i = warp;
    const int my_h = i & 1, my_par = i >> 1;
    // u8 A x s8 B (proposed: -q planes) or u8 x u8 (baseline: q = rint(s d))
    constexpr uint32_t kIdesc = MODE ? ptx::idesc_i8u(kTileM, kAccN) : ptx::idesc_i8(kTileM, kAccN);
    const int ksteps = KPAD / 32;
    // descriptor start-address field is addr >> 4: stepping K by 32 bytes
    // (two 16-byte core-matrix chunks) adds 2*LBO >> 4; column half h starts
    // h * 128 / 8 core matrices (128 B each) into the B tile
    constexpr uint64_t kAStep = (2 * kTileM * 16) >> 4;
    constexpr uint64_t kBStep = (2 * kTileN * 16) >> 4;
    const uint32_t a_base = ptx::smem_u32(sA);
    const uint32_t b_half = (uint32_t)my_h * (kAccN / 8) * 128;
    const uint32_t d = tmem_base + i * kAccN;
    const uint32_t tfull_i = tfull_bar(i);
    // producer state (warp 0): its own walk over the same tile sequence
    // A long K is split into NC chunk stages (contiguous in the K-major
    // tile), so the ring holds several chunks of the next tiles instead of
    // one whole tile (B = 16: 288 K bytes = 72 KB per tile, 2 whole-tile
    // stages starved the tensor pipe)
    SegIter pit(plan);
    int pg = 0, pt0 = 0, pt = -1, pc = 0;
    uint32_t PL = 0;
    auto produce_b = [&]() {
      if (pt < pt0) {
        int pt1;
        if (!pit.next(pg, pt0, pt1)) return;
        pt = pt1 - 1;
      }
      const int s = PL % STAGES;
      ptx::mbar_wait(empty_bar(s), ((PL / STAGES) & 1) ^ 1);
      if (lane == 0) {
        ptx::mbar_expect_tx(full_bar(s), kStage);
        ptx::bulk_g2s(ptx::smem_u32(sStage + s * kStage),
                      p.b_tiles + (size_t)pt * kB + (size_t)pc * kStage, kStage, full_bar(s));
      }
      __syncwarp();
      if (++pc == NC) {
        pc = 0;
        --pt;
      }
      ++PL;
    };
    if (i == 0)
      for (int k = 0; k < STAGES - 1; ++k) produce_b();
    uint32_t L = 0, H = 0, U = 0, uses = 0;
    for (SegIter it(plan); it.next(g, t0, t1); ++U) {
      if (i == 0) {
        // the single A slot: refilled once every MMA of the previous segment completed
        ptx::mbar_wait(aempty_bar, (U & 1) ^ 1);
        if (lane == 0) {
          ptx::mbar_expect_tx(afull_bar, kA);
          ptx::bulk_g2s(ptx::smem_u32(sA), p.a_tiles + (size_t)g * kA, kA, afull_bar);
        }
        __syncwarp();
      }
      ptx::mbar_wait(afull_bar, U & 1);
      ptx::tc_fence_after();
      for (int t = t1 - 1; t >= t0; --t, L += (CHUNK ? NC : 1)) {
        // this issuer's pairs of the tile: Hr = Ht + r with (Hr & 1) == my_par
        const uint32_t Ht = H;
        H += RG;
        const int r_first = (my_par ^ (int)(Ht & 1)) & 1;
        if constexpr (!CHUNK) {
          const int s = L % STAGES;
          ptx::mbar_wait_sleep(full_bar(s), (L / STAGES) & 1);
          ptx::tc_fence_after();
          const uint64_t bd0 = ptx::umma_desc(ptx::smem_u32(sStage + s * kStage) + b_half, kTileN * 16, 128);
          for (int r = r_first; r < RG; r += 2) {
            const uint64_t ad0 = ptx::umma_desc(a_base + r * (kTileM * KPAD), kTileM * 16, 128);
            // the epilogue's release is a hardware named barrier: the issuer
            // blocks without taking issue slots from the epilogue warps
            if (uses++ > 0) ptx::named_bar_sync(kReleaseBar + i, kReleaseThreads);
            ptx::tc_fence_after();
            ptx::umma_i8_elect(d, ad0, bd0, kIdesc, 0u);
            for (int ks = 1; ks < ksteps; ++ks)
              ptx::umma_i8_elect(d, ad0 + ks * kAStep, bd0 + ks * kBStep, kIdesc, 1u);
            ptx::umma_commit_elect(tfull_i);
          }
          ptx::umma_commit_elect(empty_bar(s));
          if (i == 0) produce_b();
        } else {
          // chunked K: every pair walks the tile's NC stages; a stage is
          // waited for by the first pair and released after the last one
          const int csteps = ksteps / NC;
          if (r_first >= RG) {
            // no pair of this issuer in the tile (RG == 1): release its stages
            for (int c = 0; c < NC; ++c) {
              const uint32_t Lc = L + c;
              ptx::mbar_wait_sleep(full_bar(Lc % STAGES), (Lc / STAGES) & 1);
              ptx::umma_commit_elect(empty_bar(Lc % STAGES));
              if (i == 0) produce_b();
            }
          }
          for (int r = r_first; r < RG; r += 2) {
            const uint64_t ad0 = ptx::umma_desc(a_base + r * (kTileM * KPAD), kTileM * 16, 128);
            if (uses++ > 0) ptx::named_bar_sync(kReleaseBar + i, kReleaseThreads);
            const bool last = r + 2 >= RG;
            for (int c = 0; c < NC; ++c) {
              const uint32_t Lc = L + c;
              const int s = Lc % STAGES;
              if (r == r_first) ptx::mbar_wait_sleep(full_bar(s), (Lc / STAGES) & 1);
              ptx::tc_fence_after();
              const uint64_t bd = ptx::umma_desc(ptx::smem_u32(sStage + s * kStage) + b_half, kTileN * 16, 128);
              const uint64_t ad = ad0 + (uint64_t)(c * csteps) * kAStep;
              ptx::umma_i8_elect(d, ad, bd, kIdesc, c > 0 ? 1u : 0u);
              for (int ks = 1; ks < csteps; ++ks)
                ptx::umma_i8_elect(d, ad + ks * kAStep, bd + ks * kBStep, kIdesc, 1u);
              if (last) {
                ptx::umma_commit_elect(empty_bar(s));
                if (i == 0) produce_b();
              }
            }
            ptx::umma_commit_elect(tfull_i);
          }
        }
      }
      ptx::umma_commit_elect(aempty_bar);
    }
    // consume the epilogue's last release of this accumulator
    if (uses > 0) ptx::named_bar_sync(kReleaseBar + i, kReleaseThreads);
  } else if (warp >= kEpiBase) {
    // ---------------- epilogue: two groups of 8 warps, one column half each ----------------
    const EpiCtx x{kB, bar_base, tmem_base, RG, KPAD, warp, lane, plan};
    if constexpr (MODE == 2) epilogue_real(p, smem, x);
    else epilogue_role<MODE == 1>(p, smem, x);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem_base, 512);
  if (p.tspan && threadIdx.x == 0) atomicMax(&p.tspan[1], global_ns());
}

// ---------------------------------------------------------------------------
// operand preparation
// ---------------------------------------------------------------------------

// Parity-group sizes of a level's columns (computed on the device).
struct TcDims {
  long long n_even, n_odd;  // columns with even / odd Q1
  long long ntiles;         // ceil(n_even / 256) + ceil(n_odd / 256)
  long long odd_base;       // first slot of the odd group
  long long n_pad;          // padding slots (last tile of each group)
  long long pad[3];
};
static_assert(sizeof(TcDims) == kUpDimsBytes, "table image layout");

// One block of 1024 threads: the level's table image from the operand
// statistics histogram (qprep / parity_slot): counting-sort cursors for the
// clamp-reach lists (qmin ascending | qmax descending), the reach counts
// low[o] = #{qmin < -o}, high[o] = #{qmax > 255 - o}, the group sizes and the
// per-tile {parity, valid slots} table for every tile below the bound.
__global__ void __launch_bounds__(1024)
tc_tables_kernel(const unsigned* __restrict__ hist, int64_t ncols, int64_t ntiles_max,
                 uint8_t* __restrict__ tab) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int lo_ex[1025], hi_ex[1025];
  const int v = threadIdx.x;
  int32_t* cur = reinterpret_cast<int32_t*>(tab);
  auto* rc = reinterpret_cast<long long*>(tab + kUpCursorBytes);
  auto* dims = reinterpret_cast<TcDims*>(tab + kUpCursorBytes + kUpReachBytes);
  int2* tinfo = reinterpret_cast<int2*>(tab + kUpCursorBytes + kUpReachBytes + kUpDimsBytes);
  int lo, hi;
  Scan(tmp).ExclusiveSum((int)hist[v], lo);             // sum of hmin[u], u < v
  __syncthreads();
  Scan(tmp).ExclusiveSum((int)hist[1024 + 1023 - v], hi);  // sum of hmax[u], u > 1023 - v
  cur[v] = lo;
  cur[1024 + (1023 - v)] = hi;
  lo_ex[v] = lo;
  hi_ex[1023 - v] = hi;
  __syncthreads();
  if (v < 256) {
    rc[v] = lo_ex[512 - v];        // q < -o       <=> bin < 512 - o
    rc[256 + v] = hi_ex[767 - v];  // q > 255 - o  <=> bin > 767 - o
  }
  const long long n_odd = hist[2049];
  const long long n_even = ncols - n_odd;
  const long long te = (n_even + kTileN - 1) / kTileN, to = (n_odd + kTileN - 1) / kTileN;
  if (v == 0) {
    TcDims d{};
    d.n_even = n_even;
    d.n_odd = n_odd;
    d.ntiles = te + to;
    d.odd_base = te * kTileN;
    d.n_pad = (te + to) * kTileN - ncols;
    *dims = d;
  }
  for (long long t = v; t < ntiles_max; t += 1024) {
    int2 ti = make_int2(0, 0);
    if (t < te) ti = make_int2(0, (int)(n_even - t * kTileN < kTileN ? n_even - t * kTileN : kTileN));
    else if (t < te + to) ti = make_int2(1, (int)(n_odd - (t - te) * kTileN < kTileN ? n_odd - (t - te) * kTileN : kTileN));
    tinfo[t] = ti;
  }
}

// Per column: Q1, Q2, qmin, qmax; sort keys for the clamp-reach lists; odd-Q1
// flags for the parity grouping; histograms of qmin / qmax; max of Q2.
// B operand in grouped slot order, K-major canonical UMMA layout per tile:
// k in [0, kbase): -q planes;  then m digits of hq (weight 255), 2 remainder
// slots (weight 1), 2 halves of Q1 (weight o);  zero up to kpad.
// slot = even/odd group base + rank of the column inside its parity group.
// One thread per column (then per padding slot), looping over the 16-byte K
// chunks: it reads its column's q as whole lines, and for every chunk a warp
// writes 32 consecutive slots (512 contiguous bytes within a parity group).
__device__ __forceinline__ uint32_t extra_word(int k0, int kbase, int m, int Q, int r1, int R,
                                               int q1a, int Q1) {
  uint32_t word = 0;
#pragma unroll
  for (int bb = 0; bb < 4; ++bb) {
    const int sl = k0 + bb - kbase;
    int v = sl < m ? min(max(Q - 127 * sl, 0), 127) : 0;
    v = sl == m ? r1 : v;
    v = sl == m + 1 ? R - r1 : v;
    v = sl == m + 2 ? q1a : v;
    v = sl == m + 3 ? Q1 - q1a : v;
    word |= (uint32_t)(v & 0xff) << (8 * bb);
  }
  return word;
}

__global__ void __launch_bounds__(256) build_b_kernel(
    const int16_t* __restrict__ qbase, int n, int kpad, int planes, int m_digits, int baseline,
    int64_t ncols, const int4* __restrict__ stats, const int32_t* __restrict__ odd_prefix,
    const TcDims* __restrict__ dims, int8_t* __restrict__ b_tiles, int32_t* __restrict__ colmap) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int chunks = kpad / 16;
  int64_t slot;
  int4 st = make_int4(0, 0, 0, 0);
  const int16_t* q = nullptr;
  if (j >= ncols) {
    // padding slots of the last tile of each parity group: zero operand, no column
    const int64_t p = j - ncols;
    const int64_t n_even = dims->n_even;
    if (p >= dims->n_pad) return;
    const int64_t pad_even = ((n_even + kTileN - 1) / kTileN) * kTileN - n_even;
    slot = p < pad_even ? n_even + p : dims->odd_base + dims->n_odd + (p - pad_even);
  } else {
    st = __ldg(stats + j);
    const int64_t oddp = __ldg(odd_prefix + j);
    slot = (!baseline && (st.y & 1)) ? dims->odd_base + oddp : j - oddp;
    q = qbase + j * n;
  }
  const int64_t tile = slot / kTileN;
  const int cc = (int)(slot - tile * kTileN);
  int8_t* dst = b_tiles + tile * ((int64_t)kTileN * kpad) + (cc >> 3) * 128 + (cc & 7) * 16;
  colmap[slot] = q ? (int32_t)j : -1;
  const int kbase = planes * n;
  const int hq = st.y >> 1;
  const int Q = hq / 255, R = hq - Q * 255;
  const int r1 = min(R, 127);
  const int q1a = min(max(st.x, -127), 127);
  for (int kc = 0; kc < chunks; ++kc) {
    uint4 out = make_uint4(0, 0, 0, 0);
    if (q == nullptr) {
    } else if (baseline) {
      // u8 q (0..255) for k < n, zero beyond
      if (kc * 16 < n) {
        const uint4 qa = __ldg(reinterpret_cast<const uint4*>(q + kc * 16));
        const uint4 qb = __ldg(reinterpret_cast<const uint4*>(q + kc * 16 + 8));
        out = make_uint4(__byte_perm(qa.x, qa.y, 0x6420), __byte_perm(qa.z, qa.w, 0x6420),
                         __byte_perm(qb.x, qb.y, 0x6420), __byte_perm(qb.z, qb.w, 0x6420));
      }
    } else if (kc * 16 < kbase) {
      // 16 q values at once (int16 pairs): -q, or its two s8 planes
      // b = clamp(-q, -127, 127) and -q - b; the low byte of each int16 is the s8
      const bool first = kc * 16 < n;
      const int kk0 = first ? kc * 16 : kc * 16 - n;  // the second plane repeats the pixels
      const uint4 qa = __ldg(reinterpret_cast<const uint4*>(q + kk0));
      const uint4 qb = __ldg(reinterpret_cast<const uint4*>(q + kk0 + 8));
      const uint32_t qw[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      uint32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t neg = __vneg2(qw[i]);
        if (planes == 1) {
          v[i] = neg;
        } else {
          const uint32_t lo = __vmins2(__vmaxs2(neg, 0xff81ff81u), 0x007f007fu);  // clamp to +-127
          v[i] = first ? lo : __vsub2(neg, lo);
        }
      }
      out = make_uint4(__byte_perm(v[0], v[1], 0x6420), __byte_perm(v[2], v[3], 0x6420),
                       __byte_perm(v[4], v[5], 0x6420), __byte_perm(v[6], v[7], 0x6420));
    } else if (kc * 16 < kbase + m_digits + 4) {
      const int k0 = kc * 16;
      out = make_uint4(extra_word(k0, kbase, m_digits, Q, r1, R, q1a, st.x),
                       extra_word(k0 + 4, kbase, m_digits, Q, r1, R, q1a, st.x),
                       extra_word(k0 + 8, kbase, m_digits, Q, r1, R, q1a, st.x),
                       extra_word(k0 + 12, kbase, m_digits, Q, r1, R, q1a, st.x));
    }
    // a warp's 32 consecutive columns of one parity group: 512 contiguous bytes per chunk
    *reinterpret_cast<uint4*>(dst + (int64_t)kc * (kTileN * 16)) = out;
  }
}

// A operand: row (range, iso) of each 128-row tile = 16 ranges x 8 isometries:
// r_iso bytes (again for a second plane), then 255 x m, 1, 1, o, o, zeros.
__global__ void build_a_kernel(const uint8_t* __restrict__ rtiles, const double* __restrict__ rmean,
                               const int32_t* __restrict__ rsq, const TcPlan* __restrict__ plan,
                               int n, int kpad, int planes, int m_digits, int baseline,
                               const uint16_t* __restrict__ inv, uint8_t* __restrict__ a_tiles,
                               int4* __restrict__ row_meta) {
  const int chunks = kpad / 16;
  const int64_t M = plan->M;
  const int64_t rows_pad = plan->rows_pad;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_pad * chunks) return;
  const int64_t row = i / chunks;
  const int kc = (int)(i - row * chunks);
  const int64_t m = row >> 3;
  const int iso = (int)(row & 7);
  const int64_t tile = row / kTileM;
  const int rrow = (int)(row - tile * kTileM);
  const int kbase = planes * n;
  uint32_t w[4] = {0, 0, 0, 0};
  int o = 0;
  if (m < M) o = (int)rint(rmean[m]);
  if (m < M) {
    const uint8_t* r = rtiles + m * n;
#pragma unroll
    for (int b4 = 0; b4 < 4; ++b4) {
      uint32_t word = 0;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) {
        const int k = kc * 16 + b4 * 4 + bb;
        uint32_t v = 0;
        if (k < kbase) {
          const int kk = k < n ? k : k - n;
          v = r[inv[iso * n + kk]];
        } else if (!baseline) {
          const int sl = k - kbase;
          if (sl < m_digits) v = 255;
          else if (sl < m_digits + 2) v = 1;
          else if (sl < m_digits + 4) v = (uint32_t)o;
        }
        word |= v << (8 * bb);
      }
      w[b4] = word;
    }
  }
  uint8_t* dst = a_tiles + tile * ((int64_t)kTileM * kpad) + (int64_t)kc * (kTileM * 16) +
                 (rrow >> 3) * 128 + (rrow & 7) * 16;
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  if (kc == 0) {
    if (m < M) {
      const int s1 = (int)rint(rmean[m] * n);  // exact: rmean = s1 / n, n a power of two
      const int R = rsq[m] - 2 * o * s1 + n * o * o;
      row_meta[row] = baseline ? make_int4(s1, rsq[m], (int)m, 2 * s1) : make_int4(o, R, (int)m, 0);
    } else {
      row_meta[row] = make_int4(0, 0, -1, 0);
    }
  }
}

// Clamp-reach lists by counting sort: columns bucketed by qmin (ascending) and
// by qmax (descending); the order inside a bucket does not matter.  A block
// takes 256 * per columns: shared-memory counts per bucket, ONE global cursor
// update per non-empty bucket and list, then shared-memory slot claims (the
// per-warp global atomics on a few hot buckets serialised in L2 before).
constexpr int kReachPerMax = 8;
__global__ void __launch_bounds__(256) reach_scatter_kernel(
    const int4* __restrict__ stats, int64_t ncols, int per, int32_t* __restrict__ cur_low,
    int32_t* __restrict__ cur_high, int32_t* __restrict__ reach_low, int32_t* __restrict__ reach_high) {
  __shared__ int cnt[2048];  // [0, 1024): qmin + 512, [1024, 2048): qmax + 512
  for (int i = threadIdx.x; i < 2048; i += 256) cnt[i] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)blockIdx.x * (256 * per) + threadIdx.x;
  int lo[kReachPerMax], hi[kReachPerMax];
#pragma unroll
  for (int k = 0; k < kReachPerMax; ++k) {
    const int64_t col = c0 + k * 256;
    lo[k] = -1;
    hi[k] = -1;
    if (k < per && col < ncols) {
      const int4 st = __ldg(stats + col);
      lo[k] = st.z + 512;
      hi[k] = st.w + 512 + 1024;
      atomicAdd(&cnt[lo[k]], 1);
      atomicAdd(&cnt[hi[k]], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += 256) {
    const int v = cnt[i];
    if (v) cnt[i] = atomicAdd(i < 1024 ? &cur_low[i] : &cur_high[i - 1024], v);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kReachPerMax; ++k) {
    if (lo[k] < 0) continue;
    const int32_t col = (int32_t)(c0 + k * 256);
    reach_low[atomicAdd(&cnt[lo[k]], 1)] = col;
    reach_high[atomicAdd(&cnt[hi[k]], 1)] = col;
  }
}

// All per-level launch planning in ONE single-block kernel (the host never
// waits for it):
//  * work decomposition of the contraction: RG row tiles per group and the
//    (group, tile) pair count the CTAs split evenly (see TcPlan);
//  * clamp-correction jobs from the offset histogram: ranges with offset o
//    against the columns whose qmin < -o (list 0) or qmax > 255 - o (list 1),
//    units of fix_rpu ranges x fix_cols columns (fix_pairs_kernel);
//  * the ranges bucketed by offset (counting sort, bucket order free).
constexpr int kPlanThreads = 1024;
__global__ void __launch_bounds__(kPlanThreads)
level_plan_kernel(const int32_t* __restrict__ d_M, int RG, const TcDims* __restrict__ dims,
                  long long b_tile_bytes, long long rr_bytes, int grid,
                  const int32_t* __restrict__ hist, const long long* __restrict__ reach_counts,
                  int fcols, int max_rpu, long long target_units,
                  const int32_t* __restrict__ roff, TcPlan* __restrict__ plan,
                  int4* __restrict__ jobs, long long* __restrict__ prefix,
                  FixPlan* __restrict__ fplan, int32_t* __restrict__ order,
                  long long* __restrict__ fix_pairs_out) {
  __shared__ int cursor[256];
  __shared__ unsigned long long best[kPlanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = *d_M;
  // ---- unit decomposition ----
  const int n_rtiles = (M * 8 + kTileM - 1) / kTileM;
  const int n_rg = (n_rtiles + RG - 1) / RG;
  const int ntiles = (int)dims->ntiles;
  // mode 1 when B does not fit comfortably in L2: span length minimising the
  // per-CTA makespan ceil(units / grid) * (ct + 2) (smallest span count wins)
  const bool rr = (long long)ntiles * b_tile_bytes > rr_bytes && n_rg > 0;
  if (rr) {
    unsigned long long mine = ~0ull;
    const int smax = min(ntiles, 8192);
    for (int sc = tid + 1; sc <= smax; sc += kPlanThreads) {
      const unsigned ctv = ((unsigned)ntiles + sc - 1) / (unsigned)sc;
      const unsigned nsp = ((unsigned)ntiles + ctv - 1) / ctv;
      const unsigned long long units = (unsigned long long)nsp * (unsigned)n_rg;
      const unsigned long long cost = ((units + grid - 1) / (unsigned)grid) * (ctv + 2);
      const unsigned long long key = (cost << 24) | (unsigned long long)sc;
      mine = key < mine ? key : mine;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long w = __shfl_xor_sync(0xffffffffu, mine, o);
      mine = w < mine ? w : mine;
    }
    if (lane == 0) best[warp] = mine;
  }
  // ---- correction jobs: thread o < 256 owns offset bucket o ----
  int cnt = 0, njob = 0;
  long long lists[2] = {0, 0}, blocks = 0, pairs = 0, u1 = 0;
  if (tid < 256) {
    cnt = hist[tid];
    lists[0] = reach_counts[tid];
    lists[1] = reach_counts[256 + tid];
    for (int k = 0; k < 2; ++k)
      if (cnt && lists[k]) u1 += (long long)cnt * ((lists[k] + fcols - 1) / fcols);
  }
  // ranges per unit: up to max_rpu while about target_units remain
  __shared__ long long u1_w[8];
  __shared__ int s_rpu;
  if (tid < 256) {
    long long v = u1;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) u1_w[warp] = v;
  }
  __syncthreads();
  if (tid == 0) {
    long long t = 0;
    for (int w2 = 0; w2 < 8; ++w2) t += u1_w[w2];
    s_rpu = (int)max(1ll, min((long long)max_rpu, t / max(1ll, target_units)));
  }
  __syncthreads();
  const int frpu = s_rpu;
  if (tid < 256) {
    for (int k = 0; k < 2; ++k)
      if (cnt && lists[k]) {
        ++njob;
        blocks += (long long)((cnt + frpu - 1) / frpu) * ((lists[k] + fcols - 1) / fcols);  // frpu ranges x fcols columns
        pairs += (long long)cnt * lists[k];
      }
  }
  // exclusive scans over the 256 buckets: warp scans + warp totals
  __shared__ int wt_c[8], wt_j[8];
  __shared__ long long wt_b[8], wt_p[8];
  int ic = cnt, ij = njob;
  long long ib = blocks, ip = pairs;
  if (tid < 256) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int c2 = __shfl_up_sync(0xffffffffu, ic, o), j2 = __shfl_up_sync(0xffffffffu, ij, o);
      const long long b2 = __shfl_up_sync(0xffffffffu, ib, o), p2 = __shfl_up_sync(0xffffffffu, ip, o);
      if (lane >= o) {
        ic += c2;
        ij += j2;
        ib += b2;
        ip += p2;
      }
    }
    if (lane == 31) {
      wt_c[warp] = ic;
      wt_j[warp] = ij;
      wt_b[warp] = ib;
      wt_p[warp] = ip;
    }
  }
  __syncthreads();
  if (tid < 256) {
    int pc = 0, pj = 0;
    long long pb = 0;
    for (int w2 = 0; w2 < warp; ++w2) {
      pc += wt_c[w2];
      pj += wt_j[w2];
      pb += wt_b[w2];
    }
    cursor[tid] = pc + ic - cnt;  // exclusive
    int j = pj + ij - njob;
    long long b = pb + ib - blocks;
    for (int k = 0; k < 2; ++k)
      if (cnt && lists[k]) {
        jobs[j] = make_int4(k, cursor[tid], cnt, (int)lists[k]);
        prefix[j] = b;
        b += (long long)((cnt + frpu - 1) / frpu) * ((lists[k] + fcols - 1) / fcols);
        ++j;
      }
    if (tid == 255) {
      long long tp = 0;
      for (int w2 = 0; w2 < 8; ++w2) tp += wt_p[w2];
      FixPlan fp{};
      fp.n_jobs = j;
      fp.rpu = frpu;
      fp.total_units = b;
      fp.fix_pairs = tp;
      *fplan = fp;
      if (fix_pairs_out) *fix_pairs_out = tp;
      prefix[j] = b;
    }
  }
  if (tid == 0) {
    TcPlan pl{};
    pl.M = M;
    pl.n_rgroups = M > 0 ? n_rg : 0;
    pl.ntiles = ntiles;
    pl.n_pairs = M > 0 ? n_rg * ntiles : 0;
    pl.mode = rr ? 1 : 0;
    if (rr) {
      unsigned long long bk = best[0];
      for (int w = 1; w < kPlanThreads / 32; ++w) bk = best[w] < bk ? best[w] : bk;
      const int sc = (int)(bk & 0xffffff);
      pl.ct = (ntiles + sc - 1) / sc;
      pl.n_units = M > 0 ? ((ntiles + pl.ct - 1) / pl.ct) * n_rg : 0;
    }
    pl.rows_pad = n_rg * RG * kTileM;
    *plan = pl;
  }
  __syncthreads();
  // ---- ranges bucketed by offset ----
  for (int i = tid; i < M; i += kPlanThreads) order[atomicAdd(&cursor[roff[i]], 1)] = i;
}

// Proposed-mode unit: R ranges of one job (one offset o) x 32 * CPL columns
// (R from the plan: up to fix_rpu while about 16 units per SM remain; the
// per-unit column set-up dominates below that).
// Each lane packs clip(q + o) of its CPL columns to bytes once (N / 4 words
// per column, in registers), then streams the R ranges' isometry rows
// (warp-uniform broadcast loads) past them: per range and isometry one
// |x - r|^2 dp4a chain per column, the minimum over (err, isometry) kept per
// column, then the warp minimum and one atomicMin per range.
constexpr int kFixStage = 256;  // uint4 per warp: staged isometry rows of up to 32 ranges (B = 4)

template <int N, int CPL>
__device__ __forceinline__ void fix_unit_batched(const FixArgs& F, const long long* __restrict__ pre,
                                                 int n_jobs, long long u, int lane, int R,
                                                 uint4* __restrict__ a_s) {
  constexpr int kCols = 32 * CPL;
  constexpr int kW = N / 4;  // packed words per column
  int lo = 0, hi = n_jobs - 1;  // last job with prefix <= u (warp-uniform)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= u) lo = mid; else hi = mid - 1;
  }
  const int4 job = F.jobs[lo];  // {list, r_off, r_cnt, col_cnt}
  const long long local = u - pre[lo];
  const unsigned ncc = (unsigned)(job.w + kCols - 1) / kCols;
  const unsigned rg = local < 0x7fffffffll ? (unsigned)local / ncc : (unsigned)(local / ncc);
  const int c0 = (int)((unsigned)(local - (long long)rg * ncc) * (unsigned)kCols);
  const int r0 = (int)rg * R, r1 = min(job.z, r0 + R);
  const int32_t* list = job.x ? F.list_high : F.list_low;
  int col[CPL];
  bool valid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int ci = c0 + c * 32 + lane;
    valid[c] = ci < job.w;
    col[c] = valid[c] ? list[ci] : list[c0];  // padding lanes repeat a real column
  }
  // the job's ranges share one offset: the first one's
  const unsigned o = (unsigned)F.roff[F.sorted_ranges[job.y + r0]];
  const unsigned o2 = o | (o << 16);
  unsigned x[CPL][kW];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
#pragma unroll
    for (int kc = 0; kc < N / 16; ++kc) {
      const int16_t* qc = F.qbase + (int64_t)col[c] * N + kc * 16;
      const uint4 qa = __ldg(reinterpret_cast<const uint4*>(qc));
      const uint4 qb = __ldg(reinterpret_cast<const uint4*>(qc + 8));
      const unsigned qw[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        // clip(q + o, 0, 255) on int16 pairs, then packed to 4 bytes
        const unsigned lo2 = __vmins2(__vmaxs2(__vadd2(qw[2 * w], o2), 0u), 0x00ff00ffu);
        const unsigned hi2 = __vmins2(__vmaxs2(__vadd2(qw[2 * w + 1], o2), 0u), 0x00ff00ffu);
        x[c][kc * 4 + w] = __byte_perm(lo2, hi2, 0x6420);
      }
    }
  }
  const int S = F.S;
  unsigned cbase[CPL];  // candidate index of (column, isometry 0): (e * 8) * S + si
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int si = S == 1 ? 0 : (S == 2 ? (col[c] & 1) : col[c] % S);
    cbase[c] = (unsigned)(8 * (col[c] - si) + si);
  }
  // the ranges' isometry rows are staged in shared memory in batches (all
  // loads of a batch in flight at once), then read back as broadcasts
  constexpr int kChunks = 8 * (N / 16);  // uint4 per range
  constexpr int kBatch = kFixStage / kChunks;
#pragma unroll 1
  for (int rb = r0; rb < r1; rb += kBatch) {
    const int nb = min(kBatch, r1 - rb);
    __syncwarp();  // the previous batch is consumed
    for (int i = lane; i < nb * kChunks; i += 32) {
      const int rr = i / kChunks, ch = i - rr * kChunks;  // ch = kc * 8 + iso
      const int64_t row0 = (int64_t)F.sorted_ranges[job.y + rb + rr] * 8;
      const uint8_t* abase = F.a_tiles + (row0 >> 7) * ((int64_t)kTileM * F.kpad) +
                             ((int)(row0 & 127) >> 3) * 128;
      a_s[i] = __ldg(reinterpret_cast<const uint4*>(abase + (ch >> 3) * (kTileM * 16) + (ch & 7) * 16));
    }
    __syncwarp();
#pragma unroll 1
    for (int ri = rb; ri < rb + nb; ++ri) {
      const int m = F.sorted_ranges[job.y + ri];
      const uint4* as = a_s + (ri - rb) * kChunks;
      unsigned k[CPL];  // err << 3 | isometry, minimum over the isometries
#pragma unroll
      for (int c = 0; c < CPL; ++c) k[c] = ~0u;
#pragma unroll
      for (int iso = 0; iso < 8; ++iso) {
        unsigned acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = 0u;
#pragma unroll
        for (int kc = 0; kc < N / 16; ++kc) {
          const uint4 r4 = as[kc * 8 + iso];
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            unsigned a = acc[c], d;
            d = __vabsdiffu4(x[c][kc * 4 + 0], r4.x); a = __dp4a(d, d, a);
            d = __vabsdiffu4(x[c][kc * 4 + 1], r4.y); a = __dp4a(d, d, a);
            d = __vabsdiffu4(x[c][kc * 4 + 2], r4.z); a = __dp4a(d, d, a);
            d = __vabsdiffu4(x[c][kc * 4 + 3], r4.w); a = __dp4a(d, d, a);
            acc[c] = a;
          }
        }
        // err <= 256 * 255^2 < 2^24: (err << 3 | iso) orders by err, then iso
#pragma unroll
        for (int c = 0; c < CPL; ++c) k[c] = min(k[c], (acc[c] << 3) | (unsigned)iso);
      }
      unsigned long long best = ~0ull;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const unsigned cidx = cbase[c] + (k[c] & 7) * (unsigned)S;
        const unsigned long long key = ((unsigned long long)(k[c] >> 3) << 32) | cidx;
        if (valid[c] && key < best) best = key;
      }
      const unsigned err = (unsigned)(best >> 32);  // 0xffffffff: no valid column
      const unsigned werr = __reduce_min_sync(0xffffffffu, err);
      const unsigned widx = __reduce_min_sync(0xffffffffu, err == werr ? (unsigned)best : 0xffffffffu);
      if (lane == 0 && werr != 0xffffffffu)
        atomicMin(&F.keys[m], ((unsigned long long)werr << 32) | widx);
    }
  }
}

constexpr int kFixThreads = 256;
template <int N>
__global__ void __launch_bounds__(kFixThreads)
fix_pairs_kernel(FixArgs F, unsigned long long* __restrict__ t_end) {
  static_assert(N % 16 == 0, "tensor levels have n >= 16");
  constexpr int kWarps = kFixThreads / 32;
  __shared__ long long s_prefix[513];  // at most 2 jobs per offset bucket, + the total
  __shared__ uint4 a_stage[kWarps][kFixStage];
  const int tid = threadIdx.x, lane = tid & 31;
  const int n_jobs = F.fplan->n_jobs;
  const long long total = F.fplan->total_units;
  if ((long long)blockIdx.x * kWarps >= total) return;
  for (int j = tid; j <= n_jobs; j += kFixThreads) s_prefix[j] = F.prefix[j];
  __syncthreads();
  const long long u0 = (long long)blockIdx.x * kWarps + (tid >> 5), du = (long long)gridDim.x * kWarps;
  if constexpr (N >= 256) {
    for (long long u = u0; u < total; u += du)
      fix_unit<N, fix_cpl(N, false)>(F, s_prefix, n_jobs, u, lane, a_stage[tid >> 5]);
  } else {
    if (F.baseline) {
      for (long long u = u0; u < total; u += du)
        fix_unit<N, fix_cpl(N, false)>(F, s_prefix, n_jobs, u, lane, a_stage[tid >> 5]);
    } else {
      const int R = F.fplan->rpu;
      for (long long u = u0; u < total; u += du)
        fix_unit_batched<N, fix_cpl(N, true)>(F, s_prefix, n_jobs, u, lane, R, a_stage[tid >> 5]);
    }
  }
  if (t_end && tid == 0) atomicMax(t_end, global_ns());
}

// fc_encode's fused level start (one warp per range slot):
//  * range m < M: gather its B x B tile from the image, exact moments, offset
//    histogram, candidate key reset (gather_kernel + level reset);
//  * tensor levels, m < rows_pad / 8: its 8 A rows (one per isometry, inverse
//    permutation of the staged tile, K extra block) and row meta; padding
//    rows are zero with m = -1 (build_a_kernel).
struct GatherBuild {
  const uint8_t* img;
  int width, B, n;
  const int32_t* origins;
  const int32_t* d_M;
  int64_t slots;          // warps launched (>= bound and >= the padded row groups)
  uint8_t* rtiles;
  double* rmean;
  int32_t* roff;
  int32_t* rsq;
  int32_t* hist;
  unsigned long long* keys;
  unsigned long long* tspan;
  // tensor operand (kpad == 0: exact level)
  int kpad, planes, m_digits, RG;
  int baseline, shift;  // baseline tensor levels: roff = floor(mean) (clamp bucket), no K extra block
  const uint16_t* inv;
  uint8_t* a_tiles;
  int4* row_meta;
};

__global__ void __launch_bounds__(256) gather_build_kernel(GatherBuild P) {
  // the staged tile and its transpose: every isometry row of A is a row of
  // one of them, possibly read backwards (see the table below)
  __shared__ __align__(16) uint8_t tile_s[8][256];
  __shared__ __align__(16) uint8_t tile_t[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.tspan[0] = ~0ull;
    P.tspan[1] = 0;
    P.tspan[2] = 0;
  }
  if (m >= P.slots) return;
  const int64_t M = *P.d_M;
  const int n = P.n, B = P.B;
  uint8_t* ts = tile_s[warp];
  int o = 0, s1 = 0, s2 = 0;
  if (m < M) {
    const int x = P.origins[2 * m], y = P.origins[2 * m + 1];
    for (int p = lane; p < n; p += 32) {
      const int r = p / B, col = p - r * B;
      const int v = P.img[(int64_t)(y + r) * P.width + x + col];
      P.rtiles[m * n + p] = (uint8_t)v;
      ts[p] = (uint8_t)v;
      tile_t[warp][col * B + r] = (uint8_t)v;
      s1 += v;
      s2 += v * v;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    const double mean = __ddiv_rn((double)s1, (double)n);
    o = P.baseline ? (s1 >> P.shift) : (int)rint(mean);
    if (lane == 0) {
      P.rmean[m] = mean;
      P.roff[m] = o;
      P.rsq[m] = s2;
      P.keys[m] = ~0ull;
      atomicAdd(&P.hist[o], 1);
    }
  }
  if (P.kpad == 0) return;
  const int n_rtiles = (int)((M * 8 + kTileM - 1) / kTileM);
  const int64_t mpad = (int64_t)((n_rtiles + P.RG - 1) / P.RG) * P.RG * kTileM / 8;
  if (m >= mpad) return;
  __syncwarp();
  const int chunks = P.kpad / 16;
  const int kbase = P.planes * n;
  const bool real = m < M;
  const uint8_t* tt = tile_t[warp];
  for (int it = lane; it < 8 * chunks; it += 32) {
    const int iso = it / chunks, kc = it - iso * chunks;
    const int64_t row = m * 8 + iso;
    const int64_t tile = row / kTileM;
    const int rrow = (int)(row - tile * kTileM);
    uint32_t w[4] = {0, 0, 0, 0};
    if (real && kc * 16 < kbase) {
      // A row (iso) position k = r*B + c holds t[i][j] with iso(i, j) = (r, c)
      // (image.py:140-155): output row r is row r or b-r of the tile or of its
      // transpose, forward or reversed:
      //   iso:       0  1  2  3  4  5  6  7
      //   transpose: 0  1  0  1  0  1  0  1
      //   flip row:  0  1  1  0  0  0  1  1
      //   reverse:   0  0  1  1  1  0  0  1
      const bool tr = iso & 1;
      const bool flip = (0xC6u >> iso) & 1u;
      const bool rev = (0x9Cu >> iso) & 1u;
      const uint8_t* src = tr ? tt : ts;
      const int kk0 = (kc * 16) % n;  // the second plane repeats the first
      const int per = B / 4;          // words per tile row (B >= 4)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = (kk0 + 4 * q) / B;      // output row of this word
        const int cw = ((kk0 + 4 * q) % B) / 4;  // word within the row
        const int sr = flip ? B - 1 - r : r;
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(src + sr * B);
        w[q] = rev ? __byte_perm(rw[per - 1 - cw], 0, 0x0123) : rw[cw];
      }
    } else if (real && !P.baseline) {
#pragma unroll
      for (int b4 = 0; b4 < 4; ++b4) {
        uint32_t word = 0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const int k = kc * 16 + b4 * 4 + bb;
          uint32_t v = 0;
          {
            const int sl = k - kbase;
            if (sl < P.m_digits) v = 255;
            else if (sl < P.m_digits + 2) v = 1;
            else if (sl < P.m_digits + 4) v = (uint32_t)o;
          }
          word |= v << (8 * bb);
        }
        w[b4] = word;
      }
    }
    uint8_t* dst = P.a_tiles + tile * ((int64_t)kTileM * P.kpad) + (int64_t)kc * (kTileM * 16) +
                   (rrow >> 3) * 128 + (rrow & 7) * 16;
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (lane < 8) {
    int4 meta = make_int4(0, 0, -1, 0);
    if (real && P.baseline) {
      meta = make_int4(s1, s2, (int)m, 2 * s1);  // {R1, R2, m, 2 R1}
    } else if (real) {
      meta = make_int4(o, s2 - 2 * o * s1 + n * o * o, (int)m, 0);  // {o, R, m, -}
    }
    P.row_meta[m * 8 + lane] = meta;
  }
}

}  // namespace

static int tc_config(Ctx* c, int kpad, int base, TcParams* prm, int real = 0, int64_t pairs = 0);
static int64_t tc_pairs_bound(const Level& L, int64_t M_bound) {
  return (M_bound * 8 + kTileM - 1) / kTileM * L.tc.ntiles;
}

int gather_build(Ctx* c, Level& L, const int32_t* d_origins, const int32_t* d_M, int64_t bound,
                 int32_t* d_hist, uint64_t* d_keys, unsigned long long* d_time) {
  GatherBuild P{};
  P.img = c->img_ptr;
  P.width = c->width;
  P.B = L.side;
  P.n = L.n;
  P.origins = d_origins;
  P.d_M = d_M;
  P.rtiles = c->rtiles.as<uint8_t>();
  P.rmean = c->rmean.as<double>();
  P.roff = c->roff.as<int32_t>();
  P.rsq = c->rsq.as<int32_t>();
  P.hist = d_hist;
  P.keys = reinterpret_cast<unsigned long long*>(d_keys);
  P.tspan = d_time;
  int64_t slots = bound;
  if (L.path == FC_PATH_TENSOR) {
    TcParams prm{};
    FC_TRY(tc_config(c, L.tc.kpad, L.baseline, &prm, 0, tc_pairs_bound(L, bound)));
    P.kpad = L.tc.kpad;
    P.planes = L.tc.planes;
    P.m_digits = L.tc.m_digits;
    P.baseline = L.baseline;
    P.shift = L.n == 256 ? 8 : L.n == 64 ? 6 : 4;
    P.RG = prm.rg;
    P.inv = c->iso_inv.as<uint16_t>() + iso_table_offset(L.side);
    P.a_tiles = c->a_tiles.as<uint8_t>();
    P.row_meta = c->row_meta.as<int4>();
    const int64_t rtiles_max = (bound * 8 + kTileM - 1) / kTileM;
    slots = std::max<int64_t>(slots, ((rtiles_max + prm.rg - 1) / prm.rg) * prm.rg * kTileM / 8);
  }
  P.slots = slots;
  FC_CUDA(c, launch_k(c, gather_build_kernel, dim3((unsigned)((slots * 32 + 255) / 256)), dim3(256),
                      0, P));
  c->total_launches += 1;
  return FC_OK;
}

// Phase 2a (host, no readback): the K layout from the proposed-mode bound on
// the candidates (|q| = |rint(s (d - mean))| <= rint(s 255 (n-1)/n), since
// one pixel can differ from the mean of n by at most 255 (n-1)/n), and every
// device buffer of the operand set reserved for the tile-count bound.  The
// exact parity-group sizes, tile table and clamp-reach cursors are computed
// on the device (tc_tables_kernel), so no host synchronisation is needed.
int level_prepare_tc_host(Ctx* c, Level& L) {
  TcOperands& T = L.tc;
  const int64_t ncols = T.ncols;
  if (ncols == 0) return set_error(c, FC_ERR_EMPTY_POOL, "no domain entries");
  if (L.baseline) {
    // baseline mode: B = q = rint(s d) in [0, 255] as one u8 plane, A = the
    // permuted range; no extra K block (the epilogue adds the per-pair terms)
    T.planes = 1;
    T.m_digits = 0;
    T.kpad = ((L.n + 31) / 32) * 32;
  } else {
    double smax = 0.0;
    for (int k = 0; k < L.s_count; ++k) smax = std::max(smax, std::fabs(L.svals[k]));
    const int qabs = (int)std::rint(smax * 255.0 * (double)(L.n - 1) / (double)L.n);
    if (qabs > 254) return set_error(c, FC_ERR_ARG, "operand outside two s8 planes");
    T.planes = qabs <= 127 ? 1 : 2;
    const long long hq_max = (long long)L.n * qabs * qabs / 2;  // >= floor(sum q^2 / 2)
    T.m_digits = std::max(1, (int)((hq_max / 255 + 126) / 127));
    T.kpad = ((T.planes * L.n + T.m_digits + 4 + 31) / 32) * 32;
  }
  if (c->trace)
    fprintf(stderr, "[fc_trace] tc operands B=%d cols=%lld planes=%d m_digits=%d kpad=%d\n", L.side,
            (long long)ncols, T.planes, T.m_digits, T.kpad);
  T.ntiles = (ncols + kTileN - 1) / kTileN + 1;
  const int64_t slots = T.ntiles * kTileN;
  FC_CUDA(c, T.reach_low.reserve(ncols * 4));
  FC_CUDA(c, T.reach_high.reserve(ncols * 4));
  FC_CUDA(c, T.b_tiles.reserve(slots * T.kpad));
  FC_CUDA(c, T.meta.reserve(slots * 4));
  FC_CUDA(c, T.tile_q1.reserve(kUpCursorBytes + kUpReachBytes + kUpDimsBytes + T.ntiles * 8 + 16));
  return FC_OK;
}

// Phase 2b (stream-ordered, capturable): the level's tables from the operand
// statistics (tc_tables_kernel), the clamp-reach lists and the grouped B
// operand (+ column map).  Launch sizes use the tile-count bound.
int level_prepare_tc_launch(Ctx* c, Level& L) {
  TcOperands& T = L.tc;
  const int64_t ncols = T.ncols;
  const int li = (int)(&L - c->lv);
  uint8_t* tab = T.tile_q1.as<uint8_t>();
  int32_t* d_cur = reinterpret_cast<int32_t*>(tab);
  auto* dims = reinterpret_cast<TcDims*>(tab + kUpCursorBytes + kUpReachBytes);
  tc_tables_kernel<<<1, 1024, 0, c->stream>>>(c->prep_dev.as<unsigned>() + li * kTcHistWords, ncols,
                                              T.ntiles, tab);
  // columns per thread: up to kReachPerMax, but at least two blocks per SM
  const int reach_per = (int)std::min<int64_t>(
      kReachPerMax, std::max<int64_t>(1, ncols / ((int64_t)256 * 2 * c->sm_count)));
  reach_scatter_kernel<<<(unsigned)std::max<int64_t>(1, (ncols + 256 * reach_per - 1) / (256 * reach_per)),
                         256, 0, c->stream>>>(
      T.col_stats.as<int4>(), ncols, reach_per, d_cur, d_cur + 1024, T.reach_low.as<int32_t>(),
      T.reach_high.as<int32_t>());
  const int64_t pad_max = T.ntiles * kTileN - ncols;
  build_b_kernel<<<(unsigned)std::max<int64_t>(1, (ncols + pad_max + 255) / 256), 256, 0, c->stream>>>(
      L.qbase.as<int16_t>(), L.n, T.kpad, T.planes, T.m_digits, L.baseline, ncols, T.col_stats.as<int4>(),
      T.odd.as<int32_t>() + ncols, dims, T.b_tiles.as<int8_t>(), T.meta.as<int32_t>());
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 3;
  T.ready = true;
  return FC_OK;
}

int level_prepare_tc_finish(Ctx* c, Level& L) {
  FC_TRY(level_prepare_tc_host(c, L));
  return level_prepare_tc_launch(c, L);
}

// Resident A row tiles and B ring depth within the shared-memory budget.
// pairs: bound on the (row tile, column tile) pairs of the launch.  Short K:
// many resident row tiles amortise the per-tile B load and bookkeeping on
// large levels (c5: RG 8), few give more row groups and a shorter segment
// start / resolution on small ones (c2 L2/L3: RG 2 is 4-12% faster).
static int tc_config(Ctx* c, int kpad, int base, TcParams* prm, int real, int64_t pairs) {
  prm->kpad = kpad;
  prm->base = base && !real;
  prm->real = real;
  const bool large = pairs >= 2048ll * c->sm_count;
  prm->rg = real ? (kpad <= 128 ? 2 : 1)
                 : kpad <= 128 ? (large ? 8 : 2) : kpad <= 320 ? 2 : 1;
  if (c->tc_rg > 0 && !real) prm->rg = c->tc_rg;  // FC_TC_RG (measurement)
  // ring stages: whole tiles up to K = 128; longer K in chunks of the largest
  // of 128 / 96 / 64 / 32 bytes dividing it (FC_TC_KC overrides, measurement)
  prm->kc = kpad;
  if (kpad > 128)
    for (int kc : {128, 96, 64, 32})
      if (kpad % kc == 0) {
        prm->kc = kc;
        break;
      }
  if (c->tc_kc > 0 && kpad % c->tc_kc == 0 && c->tc_kc % 32 == 0) prm->kc = c->tc_kc;
  // chunked ring: every chunk of a tile stays resident until the issuers'
  // last pairs of the tile consumed it, and the next tile's first chunk must
  // be in flight meanwhile, so STAGES >= chunks + 1 (else the producer would
  // wait for a stage it has yet to release: a deadlock)
  auto ring_ok = [&]() { return prm->kc == kpad || prm->stages >= kpad / prm->kc + 1; };
  for (;;) {
    prm->stages = 8;
    while (prm->stages > 2 && (int)smem_bytes(*prm) > kSmemBudget) --prm->stages;
    if (((int)smem_bytes(*prm) <= kSmemBudget && ring_ok()) || prm->rg == 1) break;
    prm->rg /= 2;
  }
  if (!ring_ok()) {  // whole-tile stages
    prm->kc = kpad;
    prm->stages = 8;
    while (prm->stages > 2 && (int)smem_bytes(*prm) > kSmemBudget) --prm->stages;
  }
  if ((int)smem_bytes(*prm) > 227 * 1024) return set_error(c, FC_ERR_ARG, "K too large for smem");
  return FC_OK;
}

static int tc_set_smem_attrs(Ctx* c) {
  void (*kernels[])(const TcParams) = {tc_scan_kernel<0, false>, tc_scan_kernel<0, true>,
                                       tc_scan_kernel<1, false>, tc_scan_kernel<1, true>,
                                       tc_scan_kernel<2, false>, tc_scan_kernel<2, true>};
  for (auto k : kernels)
    FC_CUDA(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  return FC_OK;
}

// Every buffer a level's scan may touch, reserved for `bound` ranges ahead of
// a CUDA-graph capture (nothing may allocate while the stream is captured).
int reserve_level_scan(Ctx* c, Level& L, int64_t bound) {
  FC_TRY(ensure_iso_tables(c));
  FC_TRY(reserve_ranges(c, L, bound));
  if (L.path != FC_PATH_TENSOR) return FC_OK;
  // reserved for the largest row-group size any launch may pick
  const int64_t rtiles_max = (bound * 8 + kTileM - 1) / kTileM;
  const int64_t rows_max = ((rtiles_max + 7) / 8) * 8 * kTileM;
  FC_CUDA(c, c->a_tiles.reserve(rows_max * L.tc.kpad));
  FC_CUDA(c, c->row_meta.reserve(rows_max * 16));
  FC_CUDA(c, c->tc_plan.reserve(sizeof(TcPlan) + sizeof(FixPlan) + 64));
  FC_CUDA(c, c->fix_rows.reserve(bound * 4 + 64));
  FC_CUDA(c, c->fix_jobs.reserve(512 * 16 + 64));
  FC_CUDA(c, c->fix_cols.reserve(513 * 8 + 64));
  if (!c->tc_attr_set) {
    FC_TRY(tc_set_smem_attrs(c));
    c->tc_attr_set = true;
  }
  return FC_OK;
}

// Device-driven launch: range count d_M (<= M_bound) and the offset
// histogram d_hist live on the device; nothing here waits for the GPU.
int scan_tc_launch(Ctx* c, Level& L, int64_t M_bound, const int32_t* d_M, const int32_t* d_hist,
                   uint64_t* d_keys, cudaEvent_t ev_main_end, int64_t* d_fix_pairs,
                   unsigned long long* d_time, bool a_built, cudaStream_t jobs_stream,
                   cudaEvent_t ev_plan, cudaEvent_t ev_jobs, unsigned long long* real_out) {
  TcOperands& T = L.tc;
  if (!T.ready) return set_error(c, FC_ERR_STATE, "tensor operands not prepared");
  if (M_bound == 0) return FC_OK;
  FC_TRY(ensure_iso_tables(c));
  TcParams prm{};
  FC_TRY(tc_config(c, T.kpad, L.baseline, &prm, real_out ? 1 : 0, tc_pairs_bound(L, M_bound)));
  const int RG = prm.rg;
  const int64_t rtiles_max = (M_bound * 8 + kTileM - 1) / kTileM;
  const int64_t rows_max = ((rtiles_max + RG - 1) / RG) * RG * kTileM;
  FC_CUDA(c, c->a_tiles.reserve(rows_max * T.kpad));
  FC_CUDA(c, c->row_meta.reserve(rows_max * 16));
  FC_CUDA(c, c->tc_plan.reserve(sizeof(TcPlan) + sizeof(FixPlan) + 64));
  TcPlan* d_plan = c->tc_plan.as<TcPlan>();
  FixPlan* d_fplan = reinterpret_cast<FixPlan*>(c->tc_plan.as<uint8_t>() + sizeof(TcPlan));
  FC_CUDA(c, c->fix_rows.reserve(M_bound * 4 + 64));
  FC_CUDA(c, c->fix_jobs.reserve(512 * 16 + 64));
  FC_CUDA(c, c->fix_cols.reserve(513 * 8 + 64));
  FC_CUDA(c, launch_k(c, level_plan_kernel, dim3(1), dim3(kPlanThreads), 0,
      d_M, RG,
      reinterpret_cast<const TcDims*>(T.tile_q1.as<uint8_t>() + kUpCursorBytes + kUpReachBytes),
      (long long)kTileN * T.kpad, c->tc_span_units ? 0ll : (48ll << 20), c->sm_count, d_hist,
      reinterpret_cast<const long long*>(T.tile_q1.as<uint8_t>() + kUpCursorBytes),
      fix_cols(L.n, !L.baseline), fix_rpu(L.n, !L.baseline),
      (long long)c->sm_count * 16,
      c->roff.as<int32_t>(), d_plan,
      c->fix_jobs.as<int4>(),
      c->fix_cols.as<long long>(), d_fplan, c->fix_rows.as<int32_t>(),
      reinterpret_cast<long long*>(d_fix_pairs)));
  c->stats.kernel_launches += 1;
  if (!a_built) {
    const uint16_t* inv = c->iso_inv.as<uint16_t>() + iso_table_offset(L.side);
    const int64_t work = rows_max * (T.kpad / 16);
    build_a_kernel<<<(unsigned)((work + 255) / 256), 256, 0, c->stream>>>(
        c->rtiles.as<uint8_t>(), c->rmean.as<double>(), c->rsq.as<int32_t>(), d_plan, L.n, T.kpad,
        T.planes, T.m_digits, L.baseline, inv, c->a_tiles.as<uint8_t>(), c->row_meta.as<int4>());
    FC_CUDA(c, cudaGetLastError());
    c->stats.kernel_launches += 1;
  }

  prm.a_tiles = c->a_tiles.as<uint8_t>();
  prm.row_meta = c->row_meta.as<int4>();
  prm.b_tiles = T.b_tiles.as<int8_t>();
  prm.colmap = T.meta.as<int32_t>();
  prm.tile_info = reinterpret_cast<const int2*>(T.tile_q1.as<uint8_t>() + kUpCursorBytes +
                                                kUpReachBytes + kUpDimsBytes);
  prm.keys = reinterpret_cast<unsigned long long*>(d_keys);
  prm.S = L.s_count;
  prm.shift = L.n == 256 ? 8 : L.n == 64 ? 6 : 4;
  prm.bconst = L.baseline || real_out ? T.bconst.as<int4>() : nullptr;
  prm.cnorm = L.cnorm.as<double>();
  prm.real_out = real_out;
  prm.plan = d_plan;
  prm.tspan = d_time;
  prm.fix.qbase = L.qbase.as<int16_t>();
  prm.fix.a_tiles = c->a_tiles.as<uint8_t>();
  prm.fix.roff = c->roff.as<int32_t>();
  prm.fix.jobs = c->fix_jobs.as<int4>();
  prm.fix.prefix = c->fix_cols.as<long long>();
  prm.fix.fplan = d_fplan;
  prm.fix.sorted_ranges = c->fix_rows.as<int32_t>();
  prm.fix.list_low = T.reach_low.as<int32_t>();
  prm.fix.list_high = T.reach_high.as<int32_t>();
  prm.fix.keys = reinterpret_cast<unsigned long long*>(d_keys);
  prm.fix.S = L.s_count;
  prm.fix.kpad = T.kpad;
  prm.fix.n = L.n;
  prm.fix.baseline = L.baseline;
  prm.fix.rmean = c->rmean.as<double>();
  prm.fix.dmean = L.mean.as<double>();
  prm.fix.svals = L.svals_d.as<double>();
  const uint32_t smem = smem_bytes(prm);
  if (!c->tc_attr_set) {
    FC_TRY(tc_set_smem_attrs(c));
    c->tc_attr_set = true;
  }
  const bool chunk = prm.kc != prm.kpad;
  auto kern = prm.real ? (chunk ? tc_scan_kernel<2, true> : tc_scan_kernel<2, false>)
              : prm.base ? (chunk ? tc_scan_kernel<1, true> : tc_scan_kernel<1, false>)
                         : (chunk ? tc_scan_kernel<0, true> : tc_scan_kernel<0, false>);
  FC_CUDA(c, launch_k(c, kern, dim3(c->sm_count), dim3(kThreads), smem, prm));
  if (ev_main_end) FC_CUDA(c, record_event(c, ev_main_end));
  c->stats.kernel_launches += 1;

  // ---- clamp corrections (exact kernel on clamp-active pairs), planned above ----
  // A separate kernel, on the jobs stream when given (both only atomicMin
  // into the same keys).  The real-valued search has no clamping.
  if (real_out) return FC_OK;
  cudaStream_t main = c->stream;
  if (jobs_stream) {
    FC_CUDA(c, cudaEventRecord(ev_plan, main));
    FC_CUDA(c, cudaStreamWaitEvent(jobs_stream, ev_plan, 0));
    c->stream = jobs_stream;
  }
  {
    const unsigned grid = (unsigned)(c->sm_count * (2048 / kFixThreads));
    unsigned long long* t_end = d_time ? d_time + 2 : nullptr;
    switch (L.n) {
      case 256: fix_pairs_kernel<256><<<grid, kFixThreads, 0, c->stream>>>(prm.fix, t_end); break;
      case 64: fix_pairs_kernel<64><<<grid, kFixThreads, 0, c->stream>>>(prm.fix, t_end); break;
      default: fix_pairs_kernel<16><<<grid, kFixThreads, 0, c->stream>>>(prm.fix, t_end); break;
    }
    const cudaError_t err = cudaGetLastError();
    c->stream = main;
    if (err != cudaSuccess) return set_error(c, FC_ERR_CUDA, cudaGetErrorString(err));
    c->stats.kernel_launches += 1;
  }
  if (jobs_stream) FC_CUDA(c, cudaEventRecord(ev_jobs, jobs_stream));
  return FC_OK;
}

// Baseline levels: the clamp-correction bucket of a range is floor(mean)
// (rmean = R1 / n exactly), stored where proposed mode keeps its offset.
__global__ void floor_bucket_kernel(const double* __restrict__ rmean, int64_t M,
                                    int32_t* __restrict__ roff) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) roff[i] = (int32_t)floor(rmean[i]);
}

// Real-valued slope search: per column (= pool entry, S = 1) the epilogue's
// {D1, flat, rcp(cnorm) / n^2} (rcp correctly rounded, as fc_real.cu screens).
// The real-valued search's operands in one launch: B = the decimated domains
// themselves (column e at slot e, u8, zero beyond n and on padding slots),
// the epilogue's column constants {D1 as fp32, sqrt(cnorm) as fp32 rounded
// down} and the level tables (one group, no parity split, no clamp reach).
__global__ void real_prep_kernel(const uint8_t* __restrict__ dtiles, const int32_t* __restrict__ dsum,
                                 const double* __restrict__ cnorm, int n, int kpad, int64_t ncols,
                                 int64_t ntiles, int8_t* __restrict__ b_tiles,
                                 int4* __restrict__ bconst, uint8_t* __restrict__ tab,
                                 unsigned long long* __restrict__ rec, int64_t M,
                                 int32_t* __restrict__ d_M, int32_t* __restrict__ hist) {
  const int chunks = kpad / 16;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // the launch's range count, the empty winner records, no clamp work
  if (i < 2 * M) rec[i] = ~0ull;
  if (i < 256) hist[i] = 0;
  if (i == 0) *d_M = (int32_t)M;
  if (i < 512) reinterpret_cast<long long*>(tab + kUpCursorBytes)[i] = 0;
  if (i < ntiles) {
    const int64_t left = ncols - i * kTileN;
    reinterpret_cast<int2*>(tab + kUpCursorBytes + kUpReachBytes + kUpDimsBytes)[i] =
        make_int2(0, left <= 0 ? 0 : left < kTileN ? (int)left : kTileN);
  }
  if (i == 0) {
    const long long te = (ncols + kTileN - 1) / kTileN;
    TcDims d{};
    d.n_even = ncols;
    d.ntiles = te;
    d.odd_base = te * kTileN;
    d.n_pad = te * kTileN - ncols;
    *reinterpret_cast<TcDims*>(tab + kUpCursorBytes + kUpReachBytes) = d;
  }
  // (tile, k chunk, slot): consecutive threads write consecutive 16-byte rows
  if (i >= ntiles * chunks * kTileN) return;
  const int cc = (int)(i % kTileN);
  const int64_t tk = i / kTileN;
  const int kc = (int)(tk % chunks);
  const int64_t tile = tk / chunks;
  const int64_t col = tile * kTileN + cc;
  uint4 w = make_uint4(0, 0, 0, 0);
  if (col < ncols && kc * 16 < n) w = __ldg(reinterpret_cast<const uint4*>(dtiles + col * n + kc * 16));
  *reinterpret_cast<uint4*>(b_tiles + tile * ((int64_t)kTileN * kpad) + (int64_t)kc * (kTileN * 16) + cc * 16) = w;
  if (kc == 0) {
    int2 k = make_int2(0, 0);
    if (col < ncols) {
      const double norm = cnorm[col];
      // the screen's column factor: sqrt(cnorm) rounded down (+inf for flat columns)
      const float sqn = norm == 0.0 ? __int_as_float(0x7f800000) : __double2float_rd(__dsqrt_rd(norm));
      k = make_int2(__float_as_int((float)dsum[col]), __float_as_int(sqn));
    }
    reinterpret_cast<int2*>(bconst)[col] = k;
  }
}

// Winner records {err bits, e * 8 + iso} -> (err, s = cross / cnorm, index),
// s recomputed for the winner exactly as fc_real.cu (one thread per range).
__global__ void real_finalize_kernel(const unsigned long long* __restrict__ rec, int64_t M, int n,
                                     const uint8_t* __restrict__ rtiles,
                                     const uint16_t* __restrict__ inv,
                                     const uint8_t* __restrict__ dtiles,
                                     const int32_t* __restrict__ dsum,
                                     const double* __restrict__ cnorm, double* __restrict__ out_err,
                                     double* __restrict__ out_s, int64_t* __restrict__ out_idx) {
  // one warp per range: the lanes split the n products, then a shuffle sum
  const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (m >= M) return;
  const double err = __longlong_as_double((long long)rec[2 * m]);
  const long long idx = (long long)rec[2 * m + 1];
  const long long e = idx >> 3;
  const int iso = (int)(idx & 7);
  const uint8_t* r = rtiles + m * n;
  const uint8_t* d = dtiles + e * n;
  long long X = 0, R1 = 0;
  for (int j = lane; j < n; j += 32) {
    X += (long long)d[j] * r[inv[iso * n + j]];
    R1 += r[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    X += __shfl_xor_sync(0xffffffffu, X, o);
    R1 += __shfl_xor_sync(0xffffffffu, R1, o);
  }
  if (lane != 0) return;
  const double norm = cnorm[e];
  const double cross = __dmul_rn((double)((long long)n * X - (long long)dsum[e] * R1), 1.0 / n);
  out_err[m] = err;
  out_s[m] = norm == 0.0 ? 0.0 : __ddiv_rn(cross, norm);
  out_idx[m] = idx;
}

// Per-call API variant (fc_match_level / fc_match_tiles): M is known here.
int scan_tc(Ctx* c, Level& L, int64_t M, uint64_t* d_keys) {
  FC_CUDA(c, c->enc_hist.reserve(256 * 4 + 64));
  FC_CUDA(c, c->enc_count.reserve(64 * 4));
  int32_t* d_M = c->enc_count.as<int32_t>() + 16;
  auto* d_fix = reinterpret_cast<int64_t*>(c->enc_count.as<int32_t>() + 20);
  const int32_t m32 = (int32_t)M;
  FC_TRY(stage_h2d(c, d_M, &m32, 4));
  if (L.baseline && M > 0) {
    floor_bucket_kernel<<<(unsigned)((M + 255) / 256), 256, 0, c->stream>>>(
        c->rmean.as<double>(), M, c->roff.as<int32_t>());
    FC_CUDA(c, cudaGetLastError());
    c->stats.kernel_launches += 1;
  }
  FC_TRY(roff_hist(c, M, c->enc_hist.as<int32_t>()));
  FC_CUDA(c, cudaEventRecord(c->tc_ev[0], c->stream));
  FC_TRY(scan_tc_launch(c, L, M, d_M, c->enc_hist.as<int32_t>(), d_keys, c->tc_ev[1], d_fix));
  FC_CUDA(c, cudaEventRecord(c->tc_ev[2], c->stream));
  FC_CUDA(c, c->readback.reserve(64));
  FC_CUDA(c, cudaMemcpyAsync(c->readback.ptr, d_fix, 8, cudaMemcpyDeviceToHost, c->stream));
  FC_TRY(sync_stream(c));
  float main_ms = 0.f, fix_ms = 0.f;
  cudaEventElapsedTime(&main_ms, c->tc_ev[0], c->tc_ev[1]);
  cudaEventElapsedTime(&fix_ms, c->tc_ev[1], c->tc_ev[2]);
  c->stats.main_ms = main_ms;
  c->stats.fix_ms = fix_ms;
  c->stats.fix_pairs = *c->readback.as<int64_t>();
  c->stats.rescans = 0;
  return FC_OK;
}

int real_tc_match(Ctx* c, Level& L, int level, int64_t M, double* d_err, double* d_s,
                  int64_t* d_idx) {
  // operands: B = the decimated domains themselves, A = the permuted ranges
  // (build_a's baseline layout: u8 rows, no extra K block).  The level's
  // encoder operands are replaced: it is prepared afresh on its next use.
  (void)level;
  L.baseline = 1;
  L.s_count = 1;
  L.svals[0] = 1.0;
  L.prepared = false;
  TcOperands& T = L.tc;
  T.planes = 1;
  T.m_digits = 0;
  T.kpad = ((L.n + 31) / 32) * 32;
  T.ncols = L.count;
  T.ntiles = (L.count + kTileN - 1) / kTileN + 1;
  FC_CUDA(c, T.b_tiles.reserve(T.ntiles * kTileN * T.kpad));
  FC_CUDA(c, T.bconst.reserve(T.ntiles * kTileN * 8));
  FC_CUDA(c, T.tile_q1.reserve(kUpCursorBytes + kUpReachBytes + kUpDimsBytes + T.ntiles * 8 + 16));
  FC_CUDA(c, c->real_part.reserve(M * 16 + 64));
  auto* rec = c->real_part.as<unsigned long long>();
  FC_CUDA(c, c->enc_hist.reserve(256 * 4 + 64));
  FC_CUDA(c, c->enc_count.reserve(64 * 4));
  int32_t* d_M = c->enc_count.as<int32_t>() + 16;
  auto* d_fix = reinterpret_cast<int64_t*>(c->enc_count.as<int32_t>() + 20);
  {
    const int64_t work = std::max<int64_t>(std::max<int64_t>(T.ntiles * kTileN * (T.kpad / 16), 512), 2 * M);
    real_prep_kernel<<<(unsigned)((work + 255) / 256), 256, 0, c->stream>>>(
        L.tiles.as<uint8_t>(), L.sum.as<int32_t>(), L.cnorm.as<double>(), L.n, T.kpad, L.count,
        T.ntiles, T.b_tiles.as<int8_t>(), T.bconst.as<int4>(), T.tile_q1.as<uint8_t>(), rec, M, d_M,
        c->enc_hist.as<int32_t>());
    FC_CUDA(c, cudaGetLastError());
  }
  T.ready = true;
  FC_TRY(scan_tc_launch(c, L, M, d_M, c->enc_hist.as<int32_t>(), nullptr, nullptr, d_fix, nullptr,
                        false, nullptr, nullptr, nullptr, rec));
  real_finalize_kernel<<<(unsigned)((M * 32 + 255) / 256), 256, 0, c->stream>>>(
      rec, M, L.n, c->rtiles.as<uint8_t>(), c->iso_inv.as<uint16_t>() + iso_table_offset(L.side),
      L.tiles.as<uint8_t>(), L.sum.as<int32_t>(), L.cnorm.as<double>(), d_err, d_s, d_idx);
  FC_CUDA(c, cudaGetLastError());
  c->stats.kernel_launches += 3;
  return FC_OK;
}

}  // namespace fcb
