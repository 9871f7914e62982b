// Internal definitions shared by the fracodec_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "fracodec_b200.h"

namespace fcb {

constexpr int kLevels = 4;
constexpr int kRangeSide[kLevels] = {16, 8, 4, 2};   // pool.py:20 LEVEL_RANGE_SIDES
constexpr int kDomainSide[kLevels] = {32, 16, 8, 4}; // pool.py:21 LEVEL_DOMAIN_SIDES
constexpr int kMaxS = 16;
// exact CUDA-core kernel: ranges per 128-column block (fewer for long ranges
// so small correction sets still spread over the SMs)
__host__ __device__ constexpr int ranges_per_block(int n) { return n >= 256 ? 2 : n >= 64 ? 4 : 8; }
constexpr int kTcHistWords = 1024 + 1024 + 4;  // qmin | qmax histograms, q2max, pad
constexpr int kUpCursorBytes = 2048 * 4;        // tensor-operand table image layout
constexpr int kUpReachBytes = 512 * 8;
constexpr int kUpDimsBytes = 64;                // TcDims (device-computed group sizes)

struct Status {
  int code = FC_OK;
  std::string msg;
};

// A growable device buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t cap = want + want / 4 + 256;
    cudaError_t e = cudaMalloc(&ptr, cap);
    if (e == cudaSuccess) bytes = cap;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};

// A growable pinned host buffer (async D2H/H2D staging).
struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t cap = want + want / 4 + 256;
    cudaError_t e = cudaMallocHost(&ptr, cap);
    if (e == cudaSuccess) bytes = cap;
    return e;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(ptr); }
};

// Tensor-core operand set for one level (see fc_scan_tc.cu).
struct TcOperands {
  bool ready = false;
  int planes = 1;        // int8 planes of q (1 or 2)
  int m_digits = 1;      // base-255 digit slots carrying hq = floor(Q2/2) in the K extra block
                         // (proposed mode; 0 in baseline mode: no extra block)
  int kpad = 0;          // K bytes per row: planes*B*B + m_digits + 4 (baseline: B*B), padded to 32
  int64_t ncols = 0;     // real columns E*S
  int64_t ntiles = 0;    // bound on the 256-column tiles: ceil(ncols / 256) + 1 (the
                         // two parity groups are each padded; the exact count and
                         // group sizes are computed on the device, TcDims)
  DevBuf b_tiles;        // int8 [ntiles][kpad/16][32 groups][8][16]   (UMMA K-major, no swizzle)
  DevBuf bconst;         // baseline mode: int4 [ncols] per column {W', 2 Q1, Q2, tie mask} (slot order)
  DevBuf meta;           // uint32 [ntiles*256]: (Q2 & 1) << 31 | column, 0xffffffff = padding
  DevBuf tile_q1;        // device tables: cursors [2048 i32] | reach counts [512 i64] | TcDims | tile info
  DevBuf col_stats;      // int4 [ncols]: {Q1, Q2, qmin, qmax} (unsorted order)
  DevBuf reach_low;      // int32 [ncols]: columns sorted by qmin ascending
  DevBuf reach_high;     // int32 [ncols]: columns sorted by qmax descending
  DevBuf odd;            // int32 [2*ncols]: parity flags, then their exclusive prefix
};

struct Level {
  int side = 0;           // range side B
  int n = 0;              // B*B
  int stride = 0;
  int64_t count = 0;      // pool length E
  bool synthetic = false; // set via fc_pool_set_level
  DevBuf xy;              // uint32 (x | y << 16), rank order
  DevBuf ent;             // double
  DevBuf tiles;           // uint8 [E][n] decimated
  DevBuf sum;             // int32 [E]
  DevBuf sumsq;           // int64 [E]
  DevBuf mean;            // double [E]
  DevBuf cnorm;           // double [E]
  // prepared operands
  bool prepared = false;
  int baseline = 0;
  int s_count = 0;
  double svals[kMaxS] = {0};
  double svals_up[kMaxS] = {0};   // the values last uploaded to svals_d
  int svals_up_count = -1;
  void* svals_up_ptr = nullptr;
  int path = FC_PATH_EXACT;
  DevBuf qbase;           // int16 [E*S][n] base operand (column = e*S + si)
  DevBuf svals_d;         // double [S] on the device
  // pool-build scratch over all lattice windows of this level
  DevBuf win_ent, win_key, win_key2, win_val, win_val2;
  TcOperands tc;
};

struct Ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  cudaEvent_t tc_ev[3] = {nullptr, nullptr, nullptr};
  // FC_TRACE=1: host / device timestamps of the encode phases (stderr)
  int trace = 0;
  std::vector<std::string> trace_name;
  std::vector<double> trace_host_us;
  std::vector<cudaEvent_t> trace_ev;
  bool tc_attr_set = false;
  int tc_forward = 0;    // FC_TC_FORWARD: tile scan order of the tensor kernel  // FC_TC_WAIT: spin-wait roles of the tensor kernel
  bool ent_attr_set = false;
  bool ent_attr_batch = false;  // the batched entropy launch (fc_pool_entropy_batch)
  // pool phase timing (fc_pool_times): before the entropy kernels, after them, after the survivors
  cudaEvent_t pool_ev[3] = {nullptr, nullptr, nullptr};
  bool pool_timed = false;
  Status st;
  int device_io = 0;
  // image
  int width = 0, height = 0;
  DevBuf img;
  const uint8_t* img_ptr = nullptr;  // img or adopted device pointer
  // entropy LUTs for n = 16, 64, 256, 1024
  DevBuf lut[4];
  bool lut_set[4] = {false, false, false, false};
  Level lv[kLevels];
  // scratch
  DevBuf ent_scratch, key_in, key_out, val_in, val_out, cub_tmp, count_buf;
  DevBuf origins, rtiles, rmean, roff, rsq, keys, out_err, out_idx;
  DevBuf real_part, real_out;  // fc_real_match_level: per-chunk winners, device outputs
  DevBuf fix_rows, fix_cols, fix_jobs, svals_dev;
  DevBuf a_tiles, row_meta, fix_prefix, tc_scratch, tc_plan, pool_rank;
  std::vector<int32_t> h_roff;
  // pinned staging: uploads go through an arena that is recycled at every
  // full stream synchronisation (stage_h2d / sync_stream)
  PinnedBuf up_arena;
  size_t up_off = 0;
  PinnedBuf readback;     // small D2H results (counts, histograms)
  PinnedBuf pool_rb;      // threshold-survivor counts per level
  DevBuf prep_dev;  // per-level qmin/qmax histograms + q2max + odd total, then chunk parity counts
  PinnedBuf coords_pinned;  // pool origins of all levels, fetched with fc_encode's last sync
  int64_t coords_off[kLevels] = {0, 0, 0, 0};
  bool coords_valid = false;
  // device-driven encode (fc_encode.cu)
  DevBuf enc_orig[2], enc_code[2], enc_flag, enc_pfx, enc_count, enc_hist, enc_fix;
  DevBuf leaf_flag, leaf_pos, leaf_rec;
  PinnedBuf rec_pinned;   // depth-first records, written by the compaction kernel
  int64_t enc_records = 0;
  fc_stats enc_stats[kLevels]{};
  cudaEvent_t enc_ev[kLevels][3] = {};
  bool enc_ev_ready = false;
  bool use_graph = true;               // FC_GRAPH=0 launches the level loop eagerly
  bool capturing = false;              // the stream is being captured into a graph
  // second stream for work that overlaps the contraction inside fc_encode
  // (operand builds of later levels, clamp corrections); joined per level
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_prep[kLevels] = {}, ev_plan[kLevels] = {},
              ev_jobs[kLevels] = {};
  bool overlap = true;                 // FC_OVERLAP=0 / option "overlap": single stream
  int64_t enc_summary[5] = {0, 0, 0, 0, 0};  // leaf counts per step, collage SSD
  int64_t top_begin = 0, top_end = -1;       // fc_encode's top-level slab (-1: to the end)
  bool nsel_clean = false;                   // pool survivor counters already zero
  // geometry and parameters of the pool build in progress (pool_entropy -> pool_rank)
  int pool_nx[4] = {0, 0, 0, 0}, pool_ny[4] = {0, 0, 0, 0};
  int64_t pool_caps[4] = {1, 1, 1, 1};
  int32_t pool_use_tau[4] = {0, 0, 0, 0};
  DevBuf dec_img, dec_leaves, dec_state, dec_svals;  // device decoder (fc_decode.cu)
  int pool_chunk = 0;                  // FC_POOL_CHUNK=1024 / 2048: force the rank-sort chunk
  int tc_span_units = 0;               // 1: the contraction's round-robin span schedule at any B size (tests)
  int real_cuda_cores = 0;             // 1: real-valued slope search on the dp4a kernel (tests, timing)
  int tc_rg = 0;                       // FC_TC_RG: resident row tiles of the contraction (0 = by K)
  int tc_kc = 0;                       // FC_TC_KC: ring-stage K bytes (measurement)
  cudaGraphExec_t enc_exec = nullptr;  // instantiated level-loop graph, updated per encode
  std::vector<uint64_t> enc_sig;       // launch signature of enc_exec (reuse when equal)
  int enc_levels_run = 0;              // host-side results of the captured body
  int64_t enc_body_launches = 0;
  int32_t enc_level_launches[kLevels] = {0, 0, 0, 0};
  DevBuf iso_inv;  // uint16 [4 sides][8][256] inverse isometry maps
  bool iso_ready = false;
  fc_stats stats{};
  int64_t total_launches = 0;  // kernels launched outside the per-match stats
};

int set_error(Ctx* c, int code, const std::string& msg);
int cuda_check(Ctx* c, cudaError_t e, const char* what);
int lut_slot(int n);

// Device timestamps (ns) for per-kernel spans inside CUDA graphs: kernels
// atomicMin their start / atomicMax their end into u64 slots.
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
#ifdef __CUDACC__
// baseline-mode offset of a (range, domain, s) candidate
__device__ __forceinline__ int baseline_offset(double rmean, double s, double dmean) {
  // codec.py:214-218 (== _scan.py:39-43): clip(rint(rmean - s*dmean), 0, 255)
  const int o = (int)rint(__dsub_rn(rmean, __dmul_rn(s, dmean)));
  return o < 0 ? 0 : (o > 255 ? 255 : o);
}

// Kernel launch on the context stream.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(const Ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block,
                            size_t smem, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#endif

// enc_count buffer layout: int32 counters [16] | int64 clamp pairs [4] | u64 spans [4][4]
// | int32 range-offset histograms [4][256]; the first kEncReadBytes are read back
constexpr int kEncFixOff = 64;
constexpr int kEncTimeOff = 96;
constexpr int kEncReadBytes = 96 + 4 * 4 * 8;
constexpr int kEncHistOff = kEncReadBytes;
constexpr int kEncBytes = kEncHistOff + 4 * 256 * 4;

// Timing event on the context stream.  Inside a stream capture a plain
// cudaEventRecord only marks a dependency; the External flag turns it into a
// real event-record node of the graph, so elapsed times still work.
inline cudaError_t record_event(Ctx* c, cudaEvent_t ev) {
  return c->capturing ? cudaEventRecordWithFlags(ev, c->stream, cudaEventRecordExternal)
                      : cudaEventRecord(ev, c->stream);
}

// phase tracing (fc_api.cu); no-ops unless FC_TRACE is set
void trace_reset(Ctx* c);
void trace_mark(Ctx* c, const char* name);
void trace_dump(Ctx* c);

// pinned staging helpers (fc_api.cu)
int stage_h2d(Ctx* c, void* dst, const void* src, size_t bytes);
int sync_stream(Ctx* c);

// fc_api.cu: operand preparation around a shared synchronisation
// host half: validation and level state; *needs_prep = q operands must be
// (re)built, *pending = 1 when the tensor path waits for prep_launch's readback
int prepare_begin(Ctx* c, Level& L, int level, int baseline, const double* svals, int s_count,
                  int path, int* pending, int* needs_prep);
// launch = false: host half only (fc_encode issues level_prepare_tc_launch itself)
int prepare_finish(Ctx* c, Level& L, int path, int pending, bool launch = true);

// fc_pool.cu
int pool_build(Ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
               const int32_t use_tau[4], int64_t out_sizes[4]);
int pool_entropy(Ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
                 const int32_t use_tau[4], const int32_t* row_lo, const int32_t* row_hi);
int pool_rank(Ctx* c, const int64_t* sel, int64_t out_sizes[4]);
int pool_entropy_batch(Ctx** cs, int n, const int32_t strides[4], const int64_t caps[4],
                       const double taus[4], const int32_t use_tau[4]);
int pool_window_buffers(Ctx* c, int li, void** key, void** val, void** ent, int64_t* nx,
                        int64_t* ny, int64_t* local_sel);
int pool_set_level(Ctx* c, int level, int64_t count, const uint8_t* tiles);

// fc_scan_exact.cu
int ensure_iso_tables(Ctx* c);
// device half of the operand preparation for several levels (one qprep launch,
// one parity-slot launch, one readback of the tensor-path statistics)
int prep_launch(Ctx* c, Level* const* levels, const int* stats, int count);
int gather_ranges(Ctx* c, Level& L, const int32_t* d_origins, int64_t M);
// gather with the range count read on the device (<= M_bound) and the
// histogram of range offsets o = rint(rmean) accumulated into d_hist[256]
int gather_ranges_dev(Ctx* c, Level& L, const int32_t* d_origins, const int32_t* d_M,
                      int64_t M_bound, int32_t* d_hist);
int roff_hist(Ctx* c, int64_t M, int32_t* d_hist);
int reserve_ranges(Ctx* c, Level& L, int64_t M);
int load_ranges(Ctx* c, Level& L, const uint8_t* h_tiles, int64_t M);
// d_M (optional): device range count <= M (M is then the launch bound)
int scan_exact(Ctx* c, Level& L, int64_t M, const int32_t* d_range_list, int64_t n_range_list,
               const int32_t* d_col_list, int64_t n_col_list, uint64_t* d_keys,
               const int32_t* d_M = nullptr, unsigned long long* d_time = nullptr);
int decode_keys(Ctx* c, const uint64_t* d_keys, int64_t M, int64_t* d_err, int64_t* d_idx);
int iso_table_offset(int side);
// fc_real.cu: real-valued slope search over the gathered ranges (device outputs)
int real_s_match(Ctx* c, Level& L, int64_t M, double* d_err, double* d_s, int64_t* d_idx);
int scan_rows_dropin(Ctx* c, const int16_t* ranges, const double* rmeans, int64_t M, int32_t n,
                     const int16_t* q, const double* dmeans, int64_t E, const double* svals,
                     int32_t S, int32_t baseline, int64_t* out_err, int64_t* out_idx);

// fc_scan_tc.cu
int level_prepare_tc_finish(Ctx* c, Level& L);  // after a stream sync: layout + operand build
int level_prepare_tc_host(Ctx* c, Level& L);    // the host half of it (no launches)
int level_prepare_tc_launch(Ctx* c, Level& L);  // the stream half (capturable)
// Launch the contraction and its clamp corrections for *d_M (<= M_bound)
// gathered ranges; d_hist[o] = #ranges with offset o.  No synchronisation:
// the unit decomposition and the correction jobs are planned on the device.
// d_time (optional): u64 [3] span slots {contraction start, contraction end, fix end}
// jobs_stream (optional): the clamp corrections run there, after ev_plan, and
// signal ev_jobs (they only atomicMin into the same keys as the contraction)
int scan_tc_launch(Ctx* c, Level& L, int64_t M_bound, const int32_t* d_M, const int32_t* d_hist,
                   uint64_t* d_keys, cudaEvent_t ev_main_end, int64_t* d_fix_pairs,
                   unsigned long long* d_time = nullptr, bool a_built = false,
                   cudaStream_t jobs_stream = nullptr, cudaEvent_t ev_plan = nullptr,
                   cudaEvent_t ev_jobs = nullptr, unsigned long long* real_out = nullptr);
// real-valued slope search on the contraction (fc_real.cu caller): winners per
// range as {err bits, e * 8 + iso} 128-bit records (see tc_scan_kernel<2>)
int real_tc_match(Ctx* c, Level& L, int level, int64_t M, double* d_err, double* d_s,
                  int64_t* d_idx);
// fc_encode's fused level start: gather the level's ranges (tiles, moments,
// offset histogram), reset their candidate keys and the level's span slots,
// and for tensor levels write the A operand tiles + row meta (build_a_kernel)
int gather_build(Ctx* c, Level& L, const int32_t* d_origins, const int32_t* d_M, int64_t bound,
                 int32_t* d_hist, uint64_t* d_keys, unsigned long long* d_time);
int scan_tc(Ctx* c, Level& L, int64_t M, uint64_t* d_keys);
// reserve every buffer the level's scan may touch for `bound` ranges (graph capture)
int reserve_level_scan(Ctx* c, Level& L, int64_t bound);

// fc_encode.cu
int decode_device(Ctx* c, const int32_t* leaves, int64_t n_leaves, int width, int height,
                  const double* svals, const int32_t* s_counts, int proposed, int iterations,
                  int tolerance, uint8_t* out_image, int32_t* out_deltas, int32_t* out_passes);
int encode_device(Ctx* c, const double thresholds[3], int baseline, const double* svals,
                  const int32_t s_counts[4], int path, int32_t* out_records, int64_t capacity,
                  int64_t* out_count);

}  // namespace fcb

#define FC_CUDA(c, expr)                                  \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return fcb::cuda_check(c, _e, #expr); \
  } while (0)

#define FC_TRY(expr)          \
  do {                        \
    int _r = (expr);          \
    if (_r != FC_OK) return _r; \
  } while (0)
