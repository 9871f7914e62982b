/* fracodec_b200 -- C ABI of the B200-native fractal encoder search.
 *
 * Plain C types only (no torch / CUDA types in signatures).  Every entry
 * point returns an FC_* status; on failure fc_last_error(ctx) holds a one-line
 * message.  All calls are stream-ordered on the context's CUDA stream and
 * synchronous at return unless noted.  Host pointers are plain pageable or
 * pinned memory; device-resident variants say so.
 *
 * The reference (`fracodec`, Python + numba) has no FFI of its own; these
 * entry points replace the interfaces a ctypes binding of the reference hot
 * path would bind (paths relative to /root/reference/pkg/src/fracodec):
 *
 *   fc_scan_candidates  <- _scan.py:14       scan_candidates(...) kernel seam
 *   fc_pool_build       <- pool.py:155       build_pool(image, params)
 *   fc_pool_coords      <- pool.py:84        DomainPool.coords(level)
 *   fc_pool_entries     <- pool.py:138-152   DomainEntry fields per survivor
 *   fc_pool_set_level   <- tests/oracles.py:29 make_test_pool (synthetic pools)
 *   fc_level_prepare    <- matcher.py:132    build_candidate_set(pool, level, policy)
 *   fc_match_tiles      <- matcher.py:162    scan_tiles(tiles, candidate_set)
 *   fc_match_level      <- codec.py:185-193  match_level(level, origins) incl.
 *                          codec.py:164 _gather_tiles + matcher.py:162 scan_tiles
 *   fc_set_entropy_lut  <- pool.py:88-92     the p*log(p) terms numpy produces
 *   fc_encode           <- codec.py:114-224  the quadtree level loop (split test,
 *                          children, depth-first records) around match_level
 */
#ifndef FRACODEC_B200_H_
#define FRACODEC_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FC_OK = 0,
  FC_ERR_CUDA = 1,         /* CUDA runtime / launch failure */
  FC_ERR_ARG = 2,          /* invalid argument (ValueError in the reference) */
  FC_ERR_POOL_CONFIG = 3,  /* pool.py:28 PoolConfigError: domain side exceeds image */
  FC_ERR_EMPTY_POOL = 4,   /* matcher.py:34 EmptyPoolError: no entries at level */
  FC_ERR_TILE_SIZE = 5,    /* matcher.py:168-169 tile size does not match level */
  FC_ERR_DIMS = 6,         /* codec.py:173-176 dimensions not multiple of 16 */
  FC_ERR_NO_DEVICE = 7,    /* no sm_100 device visible */
  FC_ERR_STATE = 8         /* call order violated (no image / pool / LUT) */
};

enum { FC_PATH_AUTO = 0, FC_PATH_EXACT = 1, FC_PATH_TENSOR = 2 };

typedef struct fc_ctx fc_ctx;

typedef struct fc_stats {
  int64_t comparisons;      /* ranges * E * 8 * S of the last fc_match_level */
  int64_t ranges;
  int64_t columns;          /* E * S */
  int32_t path;             /* FC_PATH_EXACT or FC_PATH_TENSOR actually used */
  int32_t kernel_launches;  /* launches issued by the last call */
  float scan_ms;            /* device time of the scan kernels (CUDA events) */
  float main_ms;            /* tensor path: main contraction kernel only */
  float fix_ms;             /* tensor path: exact clamp-correction kernel */
  int64_t fix_pairs;        /* (range, column) pairs re-evaluated exactly */
  int64_t rescans;          /* tensor path: epilogue warp rescans (tie / improvement checks) */
} fc_stats;

int fc_version(void);
int fc_ctx_create(int device, fc_ctx** out);
void fc_ctx_destroy(fc_ctx* ctx);
const char* fc_last_error(fc_ctx* ctx);
int fc_synchronize(fc_ctx* ctx);
/* Device-resident mode for benchmarking: when set, fc_set_image's pixels and
 * fc_match_level's origins/outputs are DEVICE pointers (no host copies). */
int fc_set_device_io(fc_ctx* ctx, int device_io);
/* Options.  Execution (results never depend on them): "graph" (1 = run
 * fc_encode's level loop as one CUDA graph, the default; 0 = eager
 * launches), "overlap" (second stream for operand builds / clamp
 * corrections, default 1).  Range sharding: "top_begin" / "top_end" restrict
 * fc_encode to the raster slab [top_begin, top_end) of 16x16 top-level slots
 * (default 0 / -1 = all); the records are then exactly that slab's run of the
 * full depth-first record list, so per-rank slabs concatenate in rank order.
 * Variants with identical results, kept for tests and timing:
 * "tc_span_units" (1: the contraction's round-robin span schedule, otherwise
 * only used when the B operand exceeds L2), "real_cuda_cores" (1: the
 * real-valued slope search on the dp4a kernel instead of the tensor cores). */
int fc_set_option(fc_ctx* ctx, const char* name, int64_t value);

/* terms[k-1] = (k/n) * log(k/n), k = 1..n, produced by the host's numpy so the
 * entropy bits equal pool.py:88-92 on the same host.  n in {16,64,256,1024}. */
int fc_set_entropy_lut(fc_ctx* ctx, int n, const double* terms);

/* Upload (or, in device-io mode, adopt) a row-major uint8 height x width image. */
int fc_set_image(fc_ctx* ctx, const uint8_t* pixels, int width, int height);

/* Build all four levels' pools (pool.py:155-178).  Per level: keep the top
 * caps[l] windows by entropy (stable raster tie order), or, when use_tau[l]
 * is nonzero, every window with entropy > taus[l] (threshold compaction;
 * equals the reference with level_caps[l] = #{ent > tau}).  out_sizes gets
 * the pool length per level. */
int fc_pool_build(fc_ctx* ctx, const int32_t strides[4], const int64_t caps[4],
                  const double taus[4], const int32_t use_tau[4], int64_t out_sizes[4]);
/* fc_pool_build in two phases, for a pool built by several ranks
 * (the entropy pass sharded, then a replicated ranking).
 * fc_pool_entropy: the windows' entropies of window rows [row_lo[l],
 * row_hi[l]) per level (row_lo / row_hi NULL: all rows).  Without a
 * threshold a level's entropy, key (~bits(|H|)) and window index are written
 * at the window's raster index; with one, the entropy at the window index and
 * the survivors' (key, index) appended (count: fc_pool_window_buffers).
 * fc_pool_window_buffers: device pointers of a level's window buffers
 * (u64 key, u32 index, f64 entropy; capacity nx * ny each), its window grid
 * and, when local_sel is non-NULL, the survivors appended so far (one
 * synchronisation).  The caller completes the buffers (all-gather) on the
 * context's stream or before the next call.
 * fc_pool_rank: ranking, truncation and the survivors' tiles and moments;
 * sel_counts (NULL: the device counters) are the threshold levels' survivor
 * counts in the completed buffers. */
int fc_pool_entropy(fc_ctx* ctx, const int32_t strides[4], const int64_t caps[4],
                    const double taus[4], const int32_t use_tau[4], const int32_t row_lo[4],
                    const int32_t row_hi[4]);
int fc_pool_window_buffers(fc_ctx* ctx, int level, void** key, void** val, void** ent,
                           int64_t* nx, int64_t* ny, int64_t* local_sel);
int fc_pool_rank(fc_ctx* ctx, const int64_t sel_counts[4], int64_t out_sizes[4]);
/* fc_pool_entropy (all rows) for n contexts holding images of one size, in
 * one pair of launches on ctxs[0]'s stream (a batch of small images: one
 * launch fills the GPU where each image alone would not).  Each context then
 * continues with its own fc_pool_rank (sel_counts NULL). Errors are reported
 * on ctxs[0]. */
int fc_pool_entropy_batch(fc_ctx** ctxs, int n, const int32_t strides[4], const int64_t caps[4],
                          const double taus[4], const int32_t use_tau[4]);
/* Replace one level's pool by explicit decimated tiles (E x B x B uint8). */
int fc_pool_set_level(fc_ctx* ctx, int level, int64_t count, const uint8_t* tiles);
int fc_pool_size(fc_ctx* ctx, int level, int64_t* out_count);
/* Origins in rank order, interleaved (x, y) as uint16 -- the stream header. */
int fc_pool_coords(fc_ctx* ctx, int level, uint16_t* xy);
/* All four levels' origins in one call, level 1 first (sum of the pool
 * sizes x 2 uint16); the per-level runs are in fc_pool_coords order. */
int fc_pool_coords_all(fc_ctx* ctx, uint16_t* xy);
/* Zero-copy variant: *out points at the same runs in the context's pinned
 * host memory (after a stream synchronisation).  Valid until the next
 * fc_pool_build or fc_ctx_destroy; NULL when the pool was not built by
 * fc_pool_build (e.g. fc_pool_set_level). */
int fc_pool_coords_view(fc_ctx* ctx, const uint16_t** out);
/* Inspection of the survivors (any pointer may be NULL). */
int fc_pool_entries(fc_ctx* ctx, int level, double* entropy, uint8_t* tiles, double* means,
                    double* cnorm);

/* Quantised candidate operands for a level (matcher.py:132-159).
 * baseline = 0: proposed mode rint(s*(d - mean)); 1: rint(s*d).
 * path: FC_PATH_AUTO / FC_PATH_EXACT / FC_PATH_TENSOR; the tensor path
 * (tcgen05 int8 contraction) covers both modes for B >= 4. */
int fc_level_prepare(fc_ctx* ctx, int level, int baseline, const double* svals, int32_t s_count,
                     int32_t path);

/* Match ranges at `level` whose origins are (x, y) int32 pairs: best error,
 * flat candidate index (e*8 + iso)*S + si, and exact range mean per origin
 * (codec.py:185-193).  Requires fc_level_prepare for the level. */
int fc_match_level(fc_ctx* ctx, int level, const int32_t* origins_xy, int64_t count,
                   int64_t* out_err, int64_t* out_idx, double* out_rmean);

/* Match explicit range tiles (uint8 [count][B*B], row-major per tile) --
 * matcher.py:162 scan_tiles(tiles, candidate_set). */
int fc_match_tiles(fc_ctx* ctx, int level, const uint8_t* tiles, int64_t count, int64_t* out_err,
                   int64_t* out_idx, double* out_rmean);

/* Real-valued slope search of the s-histogram analysis -- bench.py:117-139
 * _real_s_matches(tiles, basis, norms) over codec.py:164 _gather_tiles(origins),
 * the basis being bench.py:104-114 _level_basis(pool.entries(level)).  Per
 * origin: the minimal projection error max(rnorm - cross^2/cnorm, 0), the
 * slope cross/cnorm of that candidate (0 for a flat domain) and its flat
 * index e*8 + iso (first minimum), all fp64 bit-identical to the reference.
 * B >= 4 runs on the tcgen05 contraction (X = <d, r_iso> u8 x u8, fp64
 * epilogue); B = 2 on CUDA cores.  Needs the pool only (no fc_level_prepare;
 * it re-prepares the level's operands); host buffers (out_idx may be NULL). */
int fc_real_match_level(fc_ctx* ctx, int level, const int32_t* origins_xy, int64_t count,
                        double* out_err, double* out_s, int64_t* out_idx);

/* Kernel-level drop-in for _scan.py:14 with the reference's host layout:
 * ranges int16 [M, n], rmeans f64 [M], q int16 [E*8*S, n] (isometry copies),
 * dmeans f64 [E], svals f64 [S].  Exact CUDA-core path; for parity tests. */
int fc_scan_candidates(fc_ctx* ctx, const int16_t* ranges, const double* rmeans, int64_t M,
                       int32_t n, const int16_t* q, const double* dmeans, int64_t E,
                       const double* svals, int32_t s_count, int32_t baseline, int64_t* out_err,
                       int64_t* out_idx);

/* Whole quadtree encode on the device (codec.py:114-224) after fc_set_image
 * and fc_pool_build: for levels 1..3 a range splits into its four quadrants
 * when its best error exceeds thresholds[l]^2 * B^2; level-4 ranges never
 * split.  svals holds the four levels' s sets back to back (s_counts[l]
 * values each); baseline 0 = proposed mode; path FC_PATH_*, where
 * FC_PATH_TENSOR uses the exact kernel on the level the contraction does
 * not cover (2x2 ranges).  Leaf records come out in the
 * reference's depth-first order as int32 [count][6] =
 * {step, offset, iso, addr, sidx, err}; records may be NULL (fetch them
 * later with fc_encode_records).  Raises FC_ERR_EMPTY_POOL when ranges reach
 * a level whose pool is empty, FC_ERR_DIMS for sides not multiple of 16. */
int fc_encode(fc_ctx* ctx, const double thresholds[3], int32_t baseline, const double* svals,
              const int32_t s_counts[4], int32_t path, int32_t* records, int64_t capacity,
              int64_t* out_count);
int fc_encode_records(fc_ctx* ctx, int32_t* records, int64_t capacity);
/* Per-level statistics of the last fc_encode (ranges, comparisons, path,
 * scan / main / fix device times, clamp pairs). */
int fc_encode_level_stats(fc_ctx* ctx, int level, fc_stats* out);
/* Summary of the last fc_encode's records: out[0..3] = leaf count per step
 * 1..4 (codec.py step_blocks), out[4] = collage SSD (sum of the leaf errors). */
int fc_encode_summary(fc_ctx* ctx, int64_t out[5]);

/* Device decoder (codec.py:257-363 decode_trace): `iterations` collage
 * passes from a mid-gray (128) image, stopping after the first pass whose
 * max |new - cur| <= tolerance.  leaves: int32 [n][8] rows (rx, ry, level,
 * dx, dy, iso, s_index, offset) in any order, one per range block (they must
 * tile the image); svals / s_counts as in fc_encode; proposed = 1 for the
 * proposed mode (q = rint(s (t - mean))), 0 for baseline (rint(s t)).
 * out_image: width*height uint8; out_deltas (optional): one per pass run;
 * out_passes: passes run. */
int fc_decode(fc_ctx* ctx, const int32_t* leaves, int64_t n, int32_t width, int32_t height,
              const double* svals, const int32_t s_counts[4], int32_t proposed,
              int32_t iterations, int32_t tolerance, uint8_t* out_image, int32_t* out_deltas,
              int32_t* out_passes);

int fc_last_stats(fc_ctx* ctx, fc_stats* out);
/* The context's CUDA stream (cudaStream_t) so callers can time on it. */
int fc_get_stream(fc_ctx* ctx, void** out_stream);
/* Kernels this library launched on the context since creation (excludes CUB
 * sort internals and memcpy/memset). */
int fc_launch_count(fc_ctx* ctx, int64_t* out_count);
/* Device time of the last fc_pool_build (CUDA events on the context stream):
 * out_ms[0] = the window-entropy kernels, out_ms[1] = ranking + survivor
 * tiles/moments (including any survivor-count readback), out_ms[2] = total. */
int fc_pool_times(fc_ctx* ctx, float out_ms[3]);
/* Roofline denominator measured in-run: dense tcgen05.mma kind::i8 rate
 * (M=128, N=256, operands in smem, no epilogue) over all SMs, in TOP/s. */
int fc_probe_int8_peak(fc_ctx* ctx, double* out_tops);

/* Host-only (no context, no device): the FRAK record payload (stream.py:175-207
 * serialisation).  Each record (step, offset, iso, addr, s_index) becomes one
 * MSB-first field of 13 + abits[step-1] + sbits[step-1] bits: step-1 (2),
 * offset (8), iso (3), addr, s_index; fields are concatenated and the last
 * byte zero-padded.  rec: int32 rows of `stride` ints (the first five used).
 * Validates every field (addr < plen[step-1], s_index < slen[step-1]); on a
 * bad record returns FC_ERR_ARG and *bad_index = its row.  out must hold
 * (sum of widths + 7) / 8 bytes (+ 8 bytes of slack). */
int fc_pack_records(const int32_t* rec, int64_t stride, int64_t n, const int32_t abits[4],
                    const int32_t sbits[4], const int64_t plen[4], const int64_t slen[4],
                    uint8_t* out, int64_t out_bytes, int64_t* out_bits, int64_t* bad_index);

#ifdef __cplusplus
}
#endif

#endif /* FRACODEC_B200_H_ */
