// Device-driven quadtree encode (codec.py:114-161 level loop, codec.py:185-193
// match_level, codec.py:196-224 record assembly).
//
// The host keeps only launch decisions and never waits inside the level loop:
// every kernel reads the level's range count from device memory and is
// launched for the level's upper bound (n_top * 4^(level-1) ranges); the
// tensor path plans its unit decomposition and clamp-correction jobs on the
// device.  The split test, child origins, depth-first codes and leaf records
// are all produced on the device:
//
//   classify_kernel : err = key >> 32; split = err > t^2 * B^2 (levels 1-3);
//                     split ranges append their four children (origins and
//                     codes) to the next level with warp-aggregated atomics;
//                     leaves write their record into a slot indexed by the
//                     depth-first code top*64 + d1*16 + d2*4 + d3;
//   gather (next)   : range tiles, moments and the offset histogram.
//
// After level 4 the code-indexed records are compacted in code order, which
// is the reference's depth-first record order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "fc_internal.cuh"

namespace fcb {

namespace {

constexpr int kTop = 16;  // codec.py:114 top-level range side

// Encode start in one launch: the counter block zeroed (level-1 range count
// = n_top), the leaf flags cleared, and the top-level ranges.  The encoded
// top-level slots are the raster slab [first, first + n_top) (all of them
// unless the context restricts it, fc_set_option "top_begin" / "top_end");
// depth-first codes are local to the slab.
__global__ void encode_init_kernel(int nxt, int32_t first, int32_t n_top, int64_t n_codes,
                                   int32_t* __restrict__ origins, int32_t* __restrict__ codes,
                                   int32_t* __restrict__ d_count, int count_words,
                                   int32_t* __restrict__ leaf_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count_words) d_count[i] = i == 0 ? n_top : 0;
  if (i < n_codes) leaf_flag[i] = 0;
  if (i >= n_top) return;
  const int32_t gi = first + (int32_t)i;
  const int32_t ty = gi / nxt, tx = gi - ty * nxt;
  origins[2 * i] = tx * kTop;
  origins[2 * i + 1] = ty * kTop;
  codes[i] = i * 64;
}


// Split test, leaf records and children in one pass.  A leaf writes its
// record {step, offset, iso, addr, sidx, err} into the slot of its depth-first
// code; a split range appends its four children (TL, TR, BL, BR,
// codec.py:146-150) to the next level with a warp-aggregated atomic: the
// order of ranges inside a level never affects results (keys are reduced by
// value, records are ordered by code), so no prefix scan is needed.
__global__ void classify_kernel(const unsigned long long* __restrict__ keys,
                                const int32_t* __restrict__ d_M, int64_t bound, int level,
                                int can_split, double thr2, int S, int baseline,
                                const double* __restrict__ svals, const double* __restrict__ dmean,
                                const double* __restrict__ rmean, const int32_t* __restrict__ roff,
                                const int32_t* __restrict__ origins,
                                const int32_t* __restrict__ codes, int half, int weight,
                                int32_t* __restrict__ leaf_flag, int32_t* __restrict__ leaf_rec,
                                int32_t* __restrict__ next_origins,
                                int32_t* __restrict__ next_codes, int32_t* __restrict__ d_next_M) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < bound && i < *d_M;
  int sp = 0;
  unsigned long long key = 0;
  if (in) {
    key = keys[i];
    const int32_t err = (int32_t)(key >> 32);
    // codec.py:140: errs > thresholds[level-1]**2 * side*side (int64 vs float64)
    sp = can_split && (double)err > thr2;
  }
  const int lane = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(0xffffffffu, sp);
  if (bal) {
    int base = 0;
    const int leader = __ffs(bal) - 1;
    if (lane == leader) base = atomicAdd(d_next_M, 4 * __popc(bal));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (sp) {
      const int64_t j0 = base + 4 * __popc(bal & ((1u << lane) - 1));
      const int32_t x = origins[2 * i], y = origins[2 * i + 1], code = codes[i];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        next_origins[2 * (j0 + k)] = x + (k & 1) * half;
        next_origins[2 * (j0 + k) + 1] = y + (k >> 1) * half;
        next_codes[j0 + k] = code + k * weight;
      }
    }
  }
  if (!in || sp) return;
  const int32_t err = (int32_t)(key >> 32);
  const int64_t cidx = (int64_t)(key & 0xffffffffull);
  const int64_t e = cidx / (8 * S);
  const int rem = (int)(cidx - e * 8 * S);
  const int iso = rem / S, si = rem - iso * S;
  const int o = baseline ? baseline_offset(rmean[i], svals[si], dmean[e]) : roff[i];
  const int32_t code = codes[i];
  int32_t* r = leaf_rec + (int64_t)code * 6;
  r[0] = level;
  r[1] = o;
  r[2] = iso;
  r[3] = (int32_t)e;
  r[4] = si;
  r[5] = err;
  leaf_flag[code] = 1;
}

// Records in code (= depth-first) order, written straight into pinned host
// memory: a block's records are contiguous in the output, so they are staged
// in shared memory and written as one coalesced run (no copy node).
// Leaf records in depth-first code order: a block-level exclusive scan of the
// leaf flags plus the block's offset (record_block_offsets_kernel), records
// staged per block and written contiguously straight into pinned memory.
__global__ void __launch_bounds__(256) record_block_sums_kernel(int64_t n_codes,
                                                                const int32_t* __restrict__ flag,
                                                                int32_t* __restrict__ bsum) {
  using Red = cub::BlockReduce<int, 256>;
  __shared__ typename Red::TempStorage tmp;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int s = Red(tmp).Sum(i < n_codes ? flag[i] : 0);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

// Exclusive scan of the per-block counts in place (one block; nb <= 1024 * 64).
__global__ void __launch_bounds__(1024) record_block_offsets_kernel(int32_t* __restrict__ bsum,
                                                                    int nb) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int part = 0;
  for (int k = 0; k < per && b0 + k < nb; ++k) part += bsum[b0 + k];
  int excl;
  Scan(tmp).ExclusiveSum(part, excl);
  for (int k = 0; k < per && b0 + k < nb; ++k) {
    const int v = bsum[b0 + k];
    bsum[b0 + k] = excl;
    excl += v;
  }
}

__global__ void __launch_bounds__(256) compact_records_kernel(int64_t n_codes,
                                                              const int32_t* __restrict__ flag,
                                                              const int32_t* __restrict__ boff,
                                                              const int32_t* __restrict__ rec,
                                                              int32_t* __restrict__ out,
                                                              int32_t* __restrict__ d_count) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t rs[256 * 6];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = i < n_codes ? flag[i] : 0;
  int local, cnt;
  Scan(tmp).ExclusiveSum(f, local, cnt);
  const int32_t base = boff[blockIdx.x];
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *d_count = base + cnt;
  if (f) {
    const int32_t* src = rec + i * 6;
    int32_t* dst = rs + local * 6;
#pragma unroll
    for (int k = 0; k < 6; ++k) dst[k] = src[k];
  }
  __syncthreads();
  int32_t* o = out + (int64_t)base * 6;
  for (int w = threadIdx.x; w < cnt * 6; w += blockDim.x) o[w] = rs[w];
}

inline unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int encode_device(Ctx* c, const double thresholds[3], int baseline, const double* svals,
                  const int32_t s_counts[4], int path, int32_t* out_records, int64_t capacity,
                  int64_t* out_count) {
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  if (c->width % kTop || c->height % kTop) {
    char buf[96];
    snprintf(buf, sizeof buf, "dimensions not multiple of 16: %dx%d", c->width, c->height);
    return set_error(c, FC_ERR_DIMS, buf);
  }
  for (int l = 0; l < kLevels; ++l)
    if (c->lv[l].n == 0) return set_error(c, FC_ERR_STATE, "pool not built");
  if (path < FC_PATH_AUTO || path > FC_PATH_TENSOR) return set_error(c, FC_ERR_ARG, "bad path");
  if (!c->enc_ev_ready) {
    for (auto& pr : c->enc_ev)
      for (auto& e : pr) FC_CUDA(c, cudaEventCreate(&e));
    FC_CUDA(c, cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    for (int l = 0; l < kLevels; ++l) {
      FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_prep[l], cudaEventDisableTiming));
      FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_plan[l], cudaEventDisableTiming));
      FC_CUDA(c, cudaEventCreateWithFlags(&c->ev_jobs[l], cudaEventDisableTiming));
    }
    c->enc_ev_ready = true;
  }
  for (auto& st : c->enc_stats) st = fc_stats{};
  c->enc_records = 0;
  const int64_t launches0 = c->total_launches;
  c->stats = fc_stats{};

  trace_mark(c, "encode_begin");
  // ---- operands for every level, sharing one synchronisation ----
  int pending[kLevels] = {0, 0, 0, 0};
  int lpath[kLevels];
  Level* prep_lv[kLevels];
  int prep_stats[kLevels];
  int n_prep = 0;
  const double* sv = svals;
  for (int l = 0; l < kLevels; ++l) {
    Level& L = c->lv[l];
    lpath[l] = path;
    if (path == FC_PATH_TENSOR && L.n < 16) lpath[l] = FC_PATH_EXACT;
    int needs = 0;
    if (L.count > 0)
      FC_TRY(prepare_begin(c, L, l + 1, baseline, sv, s_counts[l], lpath[l], &pending[l], &needs));
    if (needs) {
      prep_lv[n_prep] = &L;
      prep_stats[n_prep++] = pending[l];
    }
    sv += s_counts[l];
  }
  if (n_prep) FC_TRY(prep_launch(c, prep_lv, prep_stats, n_prep));

  // ---- top-level ranges ----
  const int nxt = c->width / kTop, nyt = c->height / kTop;
  const int64_t n_top_all = (int64_t)nxt * nyt;
  // range-sharded encoding: this context's slab of top-level slots
  const int64_t top_first = std::min<int64_t>(std::max<int64_t>(c->top_begin, 0), n_top_all);
  const int64_t top_last =
      c->top_end < 0 ? n_top_all : std::min<int64_t>(std::max(c->top_end, top_first), n_top_all);
  const int64_t n_top = top_last - top_first;
  if (n_top == 0) return set_error(c, FC_ERR_ARG, "empty top-level slab");
  const int64_t n_codes = n_top * 64;
  const int64_t max_ranges = n_top * 64;  // level 4 bound
  for (int b = 0; b < 2; ++b) {
    FC_CUDA(c, c->enc_orig[b].reserve(max_ranges * 8 + 64));
    FC_CUDA(c, c->enc_code[b].reserve(max_ranges * 4 + 64));
  }
  FC_CUDA(c, c->enc_count.reserve(kEncBytes + 64));
  FC_CUDA(c, c->leaf_flag.reserve(n_codes * 4 + 64));
  FC_CUDA(c, c->leaf_pos.reserve(n_codes * 4 + 64));
  FC_CUDA(c, c->leaf_rec.reserve(n_codes * 24 + 64));
  FC_CUDA(c, c->readback.reserve(kEncBytes + 64));
  FC_CUDA(c, c->keys.reserve(max_ranges * 8 + 64));
  int32_t* d_count = c->enc_count.as<int32_t>();
  int32_t* d_hist = reinterpret_cast<int32_t*>(c->enc_count.as<uint8_t>() + kEncHistOff);
  int32_t* h_rb = c->readback.as<int32_t>();
  auto launch_init = [&]() -> int {  // first operation of the encode body
    const int64_t work = std::max<int64_t>(n_codes, kEncBytes / 4);
    encode_init_kernel<<<blocks_for(work), 256, 0, c->stream>>>(
        nxt, (int32_t)top_first, (int32_t)n_top, n_codes, c->enc_orig[0].as<int32_t>(),
        c->enc_code[0].as<int32_t>(), d_count, kEncBytes / 4, c->leaf_flag.as<int32_t>());
    FC_CUDA(c, cudaGetLastError());
    c->total_launches += 1;
    return FC_OK;
  };

  int64_t* d_fix = reinterpret_cast<int64_t*>(c->enc_count.as<uint8_t>() + kEncFixOff);
  auto* d_time = reinterpret_cast<unsigned long long*>(c->enc_count.as<uint8_t>() + kEncTimeOff);
  // every range buffer is sized for the level-4 bound up front: a later
  // reserve must never reallocate (and so drop) gathered ranges
  FC_TRY(reserve_ranges(c, c->lv[kLevels - 1], max_ranges));
  FC_TRY(reserve_ranges(c, c->lv[0], n_top));
  auto gather = [&](int l, int cur, int64_t bound) -> int {
    return gather_build(c, c->lv[l], c->enc_orig[cur].as<int32_t>(), d_count + l, bound,
                        d_hist + 256 * l, c->keys.as<uint64_t>(), d_time + 4 * l);
  };
  trace_mark(c, "prep_launched");
  // no synchronisation: the K layout is fixed by the s values and the tables
  // that depend on the operand statistics are built on the device
  bool tc_launch[kLevels] = {false, false, false, false};
  for (int l = 0; l < kLevels; ++l) {
    if (!pending[l]) continue;
    FC_TRY(prepare_finish(c, c->lv[l], lpath[l], pending[l], /*launch=*/false));
    tc_launch[l] = c->lv[l].path == FC_PATH_TENSOR;
  }
  trace_mark(c, "prep_finished");
  // ---- operand builds, the level loop and the record compaction run as ONE
  // CUDA graph (~50 stream operations per encode; a graph launch cuts the
  // per-operation cost from ~3.7 us to ~0.5-1 us, tools/microbench/launch_gap.cu).
  // Every buffer is reserved for its upper bound first, so nothing allocates
  // while the stream is being captured.
  bool use_graph = c->use_graph;
  {
    // range buffers were sized for the largest level before the first gather
    int64_t b = n_top;
    for (int l = 0; l < kLevels; ++l, b *= 4) {
      Level& L = c->lv[l];
      if (L.count == 0) {  // the empty-pool check needs a host sync: run eagerly
        use_graph = false;
        break;
      }
      FC_TRY(reserve_level_scan(c, L, b));
    }
    FC_CUDA(c, c->rec_pinned.reserve(n_codes * 24 + 64));
  }
  trace_mark(c, "reserved");
  // A graph whose every launch parameter (sizes, scalars, buffer addresses)
  // is unchanged is relaunched as it is: same image geometry, same pools.
  std::vector<uint64_t> sig;
  if (use_graph) {
    auto put = [&](uint64_t v) { sig.push_back(v); };
    auto putd = [&](double v) {
      uint64_t u;
      memcpy(&u, &v, 8);
      put(u);
    };
    auto putp = [&](const void* p) { put((uint64_t)(uintptr_t)p); };
    put(c->width);
    put(c->height);
    putp(c->img_ptr);
    put(baseline);
    put(path);
    put(c->sm_count);
    put(c->overlap);
    put(top_first);
    put(top_last);
    for (int l = 0; l < 3; ++l) putd(thresholds[l]);
    for (int l = 0; l < kLevels; ++l) {
      const Level& L = c->lv[l];
      const TcOperands& T = L.tc;
      put(L.count);
      put(L.n);
      put(L.s_count);
      for (int k = 0; k < L.s_count; ++k) putd(L.svals[k]);
      put(L.path);
      put(L.baseline);
      put(tc_launch[l]);
      put(T.kpad);
      put(T.planes);
      put(T.m_digits);
      put(T.ntiles);
      put(T.ncols);
      const DevBuf* lb[] = {&L.xy, &L.tiles, &L.mean, &L.qbase, &L.svals_d, &T.b_tiles, &T.meta,
                            &T.tile_q1, &T.col_stats, &T.reach_low, &T.reach_high, &T.odd};
      for (const DevBuf* b : lb) putp(b->ptr);
    }
    const DevBuf* cb[] = {&c->keys, &c->rtiles, &c->rmean, &c->roff, &c->rsq, &c->a_tiles,
                          &c->row_meta, &c->tc_plan, &c->fix_rows, &c->fix_jobs, &c->fix_cols,
                          &c->enc_orig[0], &c->enc_orig[1], &c->enc_code[0], &c->enc_code[1],
                          &c->enc_count, &c->leaf_flag, &c->leaf_pos,
                          &c->leaf_rec, &c->cub_tmp, &c->iso_inv, &c->prep_dev};
    for (const DevBuf* b : cb) {
      putp(b->ptr);
      put(b->bytes);
    }
    putp(c->coords_pinned.ptr);
    putp(c->rec_pinned.ptr);
    putp(c->readback.ptr);
    put(c->tc_span_units);
  }
  const bool reuse = use_graph && c->trace != 1 && c->enc_exec && sig == c->enc_sig;
  int levels_run = 0;
  const int64_t launches_body0 = c->total_launches;
  if (reuse) {
    levels_run = c->enc_levels_run;
    c->total_launches += c->enc_body_launches;
    for (int l = 0; l < kLevels; ++l) {
      c->enc_stats[l].kernel_launches = c->enc_level_launches[l];
      c->enc_stats[l].path = c->lv[l].path;
      if (tc_launch[l]) c->lv[l].tc.ready = true;
    }
    FC_CUDA(c, cudaGraphLaunch(c->enc_exec, c->stream));
    trace_mark(c, "graph_launched");
  }
  if (!reuse && use_graph) {
    FC_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
  }
  const int body_rc = reuse ? FC_OK : [&]() -> int {
  FC_TRY(launch_init());
  // fork the second stream: later levels' operand builds run there while the
  // first level is gathered and contracted
  const bool overlap = c->overlap;
  if (overlap) {
    FC_CUDA(c, cudaEventRecord(c->ev_fork, c->stream));
    FC_CUDA(c, cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
  }
  for (int l = 0; l < kLevels; ++l) {
    if (!tc_launch[l]) continue;
    if (overlap && l > 0) {
      cudaStream_t main = c->stream;
      c->stream = c->aux;
      const int r = level_prepare_tc_launch(c, c->lv[l]);
      c->stream = main;
      FC_TRY(r);
      FC_CUDA(c, cudaEventRecord(c->ev_prep[l], c->aux));
    } else {
      FC_TRY(level_prepare_tc_launch(c, c->lv[l]));
    }
  }
  if (c->lv[0].count > 0) FC_TRY(gather(0, 0, n_top));

  // ---- level loop: no host synchronisation ----
  int cur = 0;
  int64_t bound = n_top;
  for (int l = 0; l < kLevels; ++l) {
    Level& L = c->lv[l];
    if (L.count == 0) {
      // rare: an empty pool errors only if ranges reach it (matcher.py:34)
      FC_CUDA(c, cudaMemcpyAsync(h_rb, d_count + l, 4, cudaMemcpyDeviceToHost, c->stream));
      FC_TRY(sync_stream(c));
      if (h_rb[0] > 0) {
        char buf[64];
        snprintf(buf, sizeof buf, "no domain entries at level %d", l + 1);
        return set_error(c, FC_ERR_EMPTY_POOL, buf);
      }
      break;
    }
    levels_run = l + 1;
    const int32_t* d_M = d_count + l;
    const int64_t launches_before = c->total_launches + c->stats.kernel_launches;
    uint64_t* keys = c->keys.as<uint64_t>();
    unsigned long long* tspan = d_time + 4 * l;
    if (L.path == FC_PATH_TENSOR) {
      if (overlap && l > 0 && tc_launch[l]) FC_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_prep[l], 0));
      FC_TRY(scan_tc_launch(c, L, bound, d_M, d_hist + 256 * l, keys, nullptr, d_fix + l, tspan,
                            /*a_built=*/true, overlap ? c->aux : nullptr, c->ev_plan[l],
                            c->ev_jobs[l]));
      if (overlap) FC_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_jobs[l], 0));
    } else {
      FC_TRY(scan_exact(c, L, bound, nullptr, 0, nullptr, 0, keys, d_M, tspan));
    }
    const int side = L.side;
    const int can_split = l < kLevels - 1;
    double thr2 = 0.0;
    if (can_split) {
      thr2 = thresholds[l] * thresholds[l];
      thr2 = thr2 * side;
      thr2 = thr2 * side;
    }
    int32_t* codes = c->enc_code[cur].as<int32_t>();
    const int nxt_buf = cur ^ 1;
    FC_CUDA(c, launch_k(c, classify_kernel, dim3(blocks_for(bound)), dim3(256), 0,
        reinterpret_cast<const unsigned long long*>(keys), d_M, bound, l + 1, can_split, thr2,
        L.s_count, L.baseline, L.svals_d.as<double>(), L.mean.as<double>(), c->rmean.as<double>(),
        c->roff.as<int32_t>(), c->enc_orig[cur].as<int32_t>(), codes, side / 2,
        can_split ? 1 << (2 * (2 - l)) : 0, c->leaf_flag.as<int32_t>(), c->leaf_rec.as<int32_t>(),
        c->enc_orig[nxt_buf].as<int32_t>(), c->enc_code[nxt_buf].as<int32_t>(), d_count + l + 1));
    c->total_launches += 1;
    // a split needs err > T^2 B^2, and no error exceeds B^2 * 255^2: with a
    // threshold at or above that bound no range reaches the next level, whose
    // launches (sized for the 4x range bound) are skipped altogether
    const bool next_reachable = can_split && thr2 < (double)side * side * 65025.0;
    if (next_reachable) {
      cur = nxt_buf;
      bound *= 4;
      FC_TRY(gather(l + 1, cur, bound));
    }
    c->enc_stats[l].kernel_launches =
        (int32_t)(c->total_launches + c->stats.kernel_launches - launches_before);
    c->enc_stats[l].path = L.path;
    static const char* kLevelMark[4] = {"level1_launched", "level2_launched", "level3_launched",
                                        "level4_launched"};
    trace_mark(c, kLevelMark[l]);
    if (can_split && !next_reachable) break;
  }
  c->total_launches += c->stats.kernel_launches;
  c->stats.kernel_launches = 0;

  // ---- records in depth-first order ----
  {
    int32_t* flag = c->leaf_flag.as<int32_t>();
    int32_t* pos = c->leaf_pos.as<int32_t>();
    const unsigned nb = blocks_for(n_codes);  // n_codes <= 2^16 top slots * 64
    FC_CUDA(c, launch_k(c, record_block_sums_kernel, dim3(nb), dim3(256), 0, n_codes,
                        (const int32_t*)flag, pos));
    FC_CUDA(c, launch_k(c, record_block_offsets_kernel, dim3(1), dim3(1024), 0, pos, (int)nb));
    FC_CUDA(c, launch_k(c, compact_records_kernel, dim3(nb), dim3(256), 0, n_codes,
                        (const int32_t*)flag, (const int32_t*)pos,
                        (const int32_t*)c->leaf_rec.as<int32_t>(), c->rec_pinned.as<int32_t>(),
                        d_count + 8));
    c->total_launches += 3;
    FC_CUDA(c, cudaMemcpyAsync(h_rb, d_count, kEncReadBytes, cudaMemcpyDeviceToHost, c->stream));
  }
  return FC_OK;
  }();
  if (!reuse) {
    c->enc_levels_run = levels_run;
    c->enc_body_launches = c->total_launches - launches_body0;
    for (int l = 0; l < kLevels; ++l) c->enc_level_launches[l] = c->enc_stats[l].kernel_launches;
  }
  if (use_graph && !reuse) {
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    if (body_rc != FC_OK) {
      if (g) cudaGraphDestroy(g);
      return body_rc;
    }
    c->enc_sig.clear();
    FC_CUDA(c, ce);
    trace_mark(c, "captured");
    bool ok = false;
    if (c->enc_exec) {
      cudaGraphExecUpdateResultInfo info;
      ok = cudaGraphExecUpdate(c->enc_exec, g, &info) == cudaSuccess;
      if (!ok) {
        cudaGetLastError();  // clear the update failure
        cudaGraphExecDestroy(c->enc_exec);
        c->enc_exec = nullptr;
      }
    }
    if (!ok) {
      const cudaError_t ie = cudaGraphInstantiate(&c->enc_exec, g, 0);
      if (ie != cudaSuccess) {
        cudaGraphDestroy(g);
        c->enc_exec = nullptr;
        return cuda_check(c, ie, "cudaGraphInstantiate");
      }
    }
    cudaGraphDestroy(g);
    c->enc_sig = sig;
    trace_mark(c, "exec_ready");
    FC_CUDA(c, cudaGraphLaunch(c->enc_exec, c->stream));
  } else if (body_rc != FC_OK) {
    return body_rc;
  }
  trace_mark(c, "records_launched");
  FC_TRY(sync_stream(c));
  trace_mark(c, "records_sync");
  const int64_t n = h_rb[8];
  const int64_t* h_fix = reinterpret_cast<const int64_t*>(c->readback.as<uint8_t>() + kEncFixOff);
  const auto* h_time =
      reinterpret_cast<const unsigned long long*>(c->readback.as<uint8_t>() + kEncTimeOff);
  for (int l = 0; l < levels_run; ++l) {
    Level& L = c->lv[l];
    fc_stats& st = c->enc_stats[l];
    const int64_t M = h_rb[l];
    st.ranges = M;
    st.columns = L.count * L.s_count;
    st.comparisons = M * L.count * 8 * L.s_count;
    st.fix_pairs = h_fix[l];
  }
  c->enc_records = n;
  if (out_count) *out_count = n;
  for (int l = 0; l < kLevels; ++l) {
    fc_stats& st = c->enc_stats[l];
    if (st.ranges == 0) continue;
    // spans stamped by the kernels themselves (global ns): contraction or exact
    // scan, then the clamp corrections
    const unsigned long long* t = h_time + 4 * l;
    const double t0 = (double)t[0], t1 = (double)t[1], t2 = (double)std::max(t[2], t[1]);
    st.main_ms = t[1] > t[0] ? (float)((t1 - t0) * 1e-6) : 0.f;
    st.fix_ms = t[1] > t[0] ? (float)((t2 - t1) * 1e-6) : 0.f;
    st.scan_ms = st.main_ms + st.fix_ms;
  }
  (void)launches0;
  {
    // summary of the records (step counts, collage SSD) for the report
    const int32_t* r = c->rec_pinned.as<int32_t>();
    int64_t sm[5] = {0, 0, 0, 0, 0};
    for (int64_t i = 0; i < n; ++i, r += 6) {
      const int step = r[0];
      if (step >= 1 && step <= 4) ++sm[step - 1];
      sm[4] += r[5];
    }
    for (int k = 0; k < 5; ++k) c->enc_summary[k] = sm[k];
  }
  trace_dump(c);
  if (!out_records) return FC_OK;
  if (n > capacity) return set_error(c, FC_ERR_ARG, "record buffer too small");
  // the compaction kernel wrote the records straight into pinned host memory
  if (n > 0) memcpy(out_records, c->rec_pinned.ptr, n * 24);
  return FC_OK;
}

}  // namespace fcb
