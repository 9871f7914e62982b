// C ABI of fracodec_b200 (declared in include/fracodec_b200.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <new>

#include "fc_internal.cuh"

namespace fcb {

int set_error(Ctx* c, int code, const std::string& msg) {
  if (c) {
    c->st.code = code;
    c->st.msg = msg;
  }
  return code;
}

int cuda_check(Ctx* c, cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e),
           what);
  return set_error(c, FC_ERR_CUDA, buf);
}

static double host_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void trace_reset(Ctx* c) {
  if (!c->trace) return;
  c->trace_name.clear();
  c->trace_host_us.clear();
}

void trace_mark(Ctx* c, const char* name) {
  // FC_TRACE=2: marks outside graph capture only, graph reuse kept
  if (!c->trace || (c->trace == 2 && c->capturing)) return;
  const size_t k = c->trace_name.size();
  if (k >= c->trace_ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->trace_ev.push_back(e);
  }
  record_event(c, c->trace_ev[k]);
  c->trace_name.push_back(name);
  c->trace_host_us.push_back(host_us());
}

void trace_dump(Ctx* c) {
  if (!c->trace || c->trace_name.empty()) return;
  cudaStreamSynchronize(c->stream);
  fprintf(stderr, "[fc_trace] %-22s %10s %10s\n", "mark", "host_us", "dev_us");
  for (size_t k = 0; k < c->trace_name.size(); ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->trace_ev[0], c->trace_ev[k]);
    fprintf(stderr, "[fc_trace] %-22s %10.1f %10.1f\n", c->trace_name[k].c_str(),
            c->trace_host_us[k] - c->trace_host_us[0], 1e3 * ms);
  }
}

int sync_stream(Ctx* c) {
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  c->up_off = 0;
  return FC_OK;
}

// Copy host bytes into the pinned arena and enqueue the H2D copy from there,
// so the call never blocks on the stream (a pageable source would).
int stage_h2d(Ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return FC_OK;
  const size_t padded = (bytes + 255) & ~(size_t)255;
  if (c->up_off + padded > c->up_arena.bytes) {
    if (c->up_off > 0) FC_TRY(sync_stream(c));  // recycle the arena
    FC_CUDA(c, c->up_arena.reserve(std::max<size_t>(padded, 1 << 20)));
  }
  char* slot = c->up_arena.as<char>() + c->up_off;
  memcpy(slot, src, bytes);
  FC_CUDA(c, cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, c->stream));
  c->up_off += padded;
  return FC_OK;
}

int lut_slot(int n) { return n == 16 ? 0 : n == 64 ? 1 : n == 256 ? 2 : n == 1024 ? 3 : -1; }

namespace {

int check_level(Ctx* c, int level) {
  if (level < 1 || level > kLevels) return set_error(c, FC_ERR_ARG, "level must be 1..4");
  return FC_OK;
}

int level_ready(Ctx* c, int level) {
  FC_TRY(check_level(c, level));
  Level& L = c->lv[level - 1];
  if (L.n == 0) return set_error(c, FC_ERR_STATE, "pool not built");
  return FC_OK;
}

}  // namespace

// Operand preparation split around one stream synchronisation so several
// levels share it (fc_encode).  *pending = 1 when a tensor-path readback is
// in flight and prepare_finish must run after the next sync.
int prepare_begin(Ctx* c, Level& L, int level, int baseline, const double* svals, int s_count,
                  int path, int* pending, int* needs_prep) {
  *pending = 0;
  *needs_prep = 0;
  if (s_count < 1 || s_count > kMaxS || !svals)
    return set_error(c, FC_ERR_ARG, "s set must have 1..16 values");
  for (int i = 0; i < s_count; ++i)
    if (!(svals[i] >= 0.0 && svals[i] <= 1.0))
      return set_error(c, FC_ERR_ARG, "s values must lie in [0, 1]");
  if (path < FC_PATH_AUTO || path > FC_PATH_TENSOR) return set_error(c, FC_ERR_ARG, "bad path");
  bool same = L.prepared && L.baseline == (baseline ? 1 : 0) && L.s_count == s_count;
  for (int i = 0; same && i < s_count; ++i) same = L.svals[i] == svals[i];
  if (same && (path == FC_PATH_AUTO || path == L.path)) return FC_OK;
  if (L.count == 0) {
    char buf[64];
    snprintf(buf, sizeof buf, "no domain entries at level %d", level);
    return set_error(c, FC_ERR_EMPTY_POOL, buf);
  }
  L.baseline = baseline ? 1 : 0;
  L.s_count = s_count;
  for (int i = 0; i < s_count; ++i) L.svals[i] = svals[i];
  L.prepared = false;
  L.tc.ready = false;
  *needs_prep = 1;
  const bool tc_ok = L.n >= 16;  // both modes (baseline: u8 x u8, epilogue forms o per pair)
  if (path == FC_PATH_TENSOR && !tc_ok)
    return set_error(c, FC_ERR_ARG, "tensor path needs B >= 4");
  bool want_tc = path == FC_PATH_TENSOR || (path == FC_PATH_AUTO && tc_ok);
  if (want_tc && L.count * L.s_count >= (1ll << 31) - 1024) {
    if (path == FC_PATH_TENSOR) return set_error(c, FC_ERR_ARG, "too many columns");
    want_tc = false;  // auto: keep the exact path
  }
  if (want_tc) {
    *pending = 1;
    return FC_OK;
  }
  L.path = FC_PATH_EXACT;
  L.prepared = true;
  return FC_OK;
}

int prepare_finish(Ctx* c, Level& L, int path, int pending, bool launch) {
  if (!pending) return FC_OK;
  const int r = launch ? level_prepare_tc_finish(c, L) : level_prepare_tc_host(c, L);
  if (r == FC_OK) {
    L.path = FC_PATH_TENSOR;
  } else if (path == FC_PATH_TENSOR) {
    return r;
  } else {
    c->st = Status{};  // auto: operands out of the two-plane range -> exact path
    L.path = FC_PATH_EXACT;
  }
  L.prepared = true;
  return FC_OK;
}

namespace {

}  // namespace
}  // namespace fcb

using namespace fcb;

struct fc_ctx : public Ctx {};

extern "C" {

int fc_version(void) { return 1; }

int fc_pack_records(const int32_t* rec, int64_t stride, int64_t n, const int32_t abits[4],
                    const int32_t sbits[4], const int64_t plen[4], const int64_t slen[4],
                    uint8_t* out, int64_t out_bytes, int64_t* out_bits, int64_t* bad_index) {
  if (bad_index) *bad_index = -1;
  if (!out_bits || (n > 0 && (!rec || !out))) return FC_ERR_ARG;
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t* r = rec + i * stride;
    const int step = r[0];
    if (step < 1 || step > 4 || r[1] < 0 || r[1] > 255 || r[2] < 0 || r[2] > 7 || r[3] < 0 ||
        r[3] >= plen[step - 1] || r[4] < 0 || r[4] >= slen[step - 1]) {
      if (bad_index) *bad_index = i;
      return FC_ERR_ARG;
    }
    total += 13 + abits[step - 1] + sbits[step - 1];
  }
  *out_bits = total;
  if ((total + 7) / 8 + 8 > out_bytes) return FC_ERR_ARG;
  // MSB-first bit writer: `acc` holds `nacc` pending bits (right-aligned)
  unsigned __int128 acc = 0;
  int nacc = 0;
  uint8_t* o = out;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t* r = rec + i * stride;
    const int l = r[0] - 1;
    const int ab = abits[l], sb = sbits[l];
    uint64_t v = (uint64_t)l;
    v = (v << 8) | (uint64_t)r[1];
    v = (v << 3) | (uint64_t)r[2];
    v = (ab ? (v << ab) : v) | (uint64_t)r[3];
    v = (sb ? (v << sb) : v) | (uint64_t)r[4];
    acc = (acc << (13 + ab + sb)) | v;
    nacc += 13 + ab + sb;
    while (nacc >= 8) {
      nacc -= 8;
      *o++ = (uint8_t)(acc >> nacc);
    }
    acc &= ((unsigned __int128)1 << nacc) - 1;
  }
  if (nacc > 0) *o++ = (uint8_t)(acc << (8 - nacc));
  return FC_OK;
}

int fc_ctx_create(int device, fc_ctx** out) {
  if (!out) return FC_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return FC_ERR_NO_DEVICE;
  if (device < 0 || device >= ndev) return FC_ERR_ARG;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return FC_ERR_CUDA;
  if (prop.major != 10) return FC_ERR_NO_DEVICE;  // sm_100a build only
  if (cudaSetDevice(device) != cudaSuccess) return FC_ERR_CUDA;
  fc_ctx* c = new (std::nothrow) fc_ctx();
  if (!c) return FC_ERR_ARG;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (const char* t = getenv("FC_TRACE")) c->trace = atoi(t);
  if (const char* g = getenv("FC_GRAPH")) c->use_graph = atoi(g) != 0;
  if (const char* o = getenv("FC_OVERLAP")) c->overlap = atoi(o) != 0;
  if (const char* d = getenv("FC_POOL_CHUNK")) c->pool_chunk = atoi(d);
  if (const char* d = getenv("FC_TC_RG")) c->tc_rg = atoi(d);
  if (const char* d = getenv("FC_TC_KC")) c->tc_kc = atoi(d);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
      cudaEventCreate(&c->ev2) != cudaSuccess || cudaEventCreate(&c->tc_ev[0]) != cudaSuccess ||
      cudaEventCreate(&c->tc_ev[1]) != cudaSuccess || cudaEventCreate(&c->tc_ev[2]) != cudaSuccess) {
    delete c;
    return FC_ERR_CUDA;
  }
  for (int i = 0; i < kLevels; ++i) {
    c->lv[i].side = kRangeSide[i];
    c->lv[i].n = 0;
  }
  *out = c;
  return FC_OK;
}

void fc_ctx_destroy(fc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  DevBuf* bufs[] = {&c->img, &c->ent_scratch, &c->key_in, &c->key_out, &c->val_in, &c->val_out,
                    &c->cub_tmp, &c->count_buf, &c->origins, &c->rtiles, &c->rmean, &c->roff,
                    &c->rsq, &c->keys, &c->out_err, &c->out_idx, &c->fix_rows, &c->fix_cols,
                    &c->fix_jobs, &c->svals_dev, &c->iso_inv, &c->a_tiles, &c->row_meta,
                    &c->fix_prefix, &c->tc_scratch, &c->enc_orig[0], &c->enc_orig[1],
                    &c->enc_code[0], &c->enc_code[1], &c->enc_flag, &c->enc_pfx,
                    &c->enc_count, &c->enc_hist, &c->leaf_flag, &c->leaf_pos, &c->leaf_rec, &c->tc_plan, &c->enc_fix, &c->pool_rank};
  for (DevBuf* b : bufs) b->release();
  c->up_arena.release();
  c->readback.release();
  c->pool_rb.release();
  c->prep_dev.release();
  c->coords_pinned.release();
  c->rec_pinned.release();
  if (c->enc_ev_ready)
    for (auto& pr : c->enc_ev)
      for (auto& e : pr) cudaEventDestroy(e);
  for (auto& b : c->lut) b.release();
  for (auto& L : c->lv) {
    DevBuf* lb[] = {&L.xy, &L.ent, &L.tiles, &L.sum, &L.sumsq, &L.mean, &L.cnorm, &L.qbase,
                    &L.tc.b_tiles, &L.tc.bconst, &L.tc.meta, &L.tc.tile_q1, &L.tc.col_stats,
                    &L.tc.reach_low, &L.tc.reach_high, &L.tc.odd, &L.svals_d, 
                    &L.win_ent, &L.win_key, &L.win_key2, &L.win_val, &L.win_val2};
    for (DevBuf* b : lb) b->release();
  }
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  cudaEventDestroy(c->ev2);
  for (auto& e : c->tc_ev) cudaEventDestroy(e);
  for (auto& e : c->pool_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->trace_ev) cudaEventDestroy(e);
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
    cudaEventDestroy(c->ev_fork);
    for (int l = 0; l < kLevels; ++l) {
      cudaEventDestroy(c->ev_prep[l]);
      cudaEventDestroy(c->ev_plan[l]);
      cudaEventDestroy(c->ev_jobs[l]);
    }
  }
  if (c->enc_exec) cudaGraphExecDestroy(c->enc_exec);
  cudaStreamDestroy(c->stream);
  delete c;
}

const char* fc_last_error(fc_ctx* c) { return c ? c->st.msg.c_str() : "null context"; }

int fc_synchronize(fc_ctx* c) {
  cudaSetDevice(c->device);
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_set_device_io(fc_ctx* c, int device_io) {
  c->device_io = device_io ? 1 : 0;
  return FC_OK;
}

int fc_set_option(fc_ctx* c, const char* name, int64_t value) {
  if (!name) return set_error(c, FC_ERR_ARG, "null option name");
  if (strcmp(name, "graph") == 0) {
    c->use_graph = value != 0;
    return FC_OK;
  }
  if (strcmp(name, "overlap") == 0) {
    c->overlap = value != 0;
    return FC_OK;
  }
  if (strcmp(name, "top_begin") == 0) {  // range sharding: first top-level slot
    c->top_begin = value;
    return FC_OK;
  }
  if (strcmp(name, "top_end") == 0) {  // range sharding: end of the slab (-1: all)
    c->top_end = value;
    return FC_OK;
  }
  // schedule / launch variants (results identical by construction; tests run both)
  if (strcmp(name, "tc_span_units") == 0) {  // force the B > L2 round-robin span schedule
    c->tc_span_units = (int)value;
    return FC_OK;
  }
  if (strcmp(name, "real_cuda_cores") == 0) {  // s-histogram search on the dp4a kernel
    c->real_cuda_cores = (int)value;
    return FC_OK;
  }
  return set_error(c, FC_ERR_ARG, std::string("unknown option ") + name);
}

int fc_set_entropy_lut(fc_ctx* c, int n, const double* terms) {
  cudaSetDevice(c->device);
  const int slot = lut_slot(n);
  if (slot < 0 || !terms) return set_error(c, FC_ERR_ARG, "LUT size must be 16/64/256/1024");
  FC_CUDA(c, c->lut[slot].reserve(n * 8));
  FC_TRY(stage_h2d(c, c->lut[slot].ptr, terms, n * 8));
  c->lut_set[slot] = true;
  return FC_OK;
}

int fc_set_image(fc_ctx* c, const uint8_t* pixels, int width, int height) {
  cudaSetDevice(c->device);
  if (width < 1 || height < 1 || !pixels) return set_error(c, FC_ERR_ARG, "bad image");
  if (width > 65535 || height > 65535)
    return set_error(c, FC_ERR_ARG, "image sides must fit the u16 stream coordinates");
  trace_reset(c);
  trace_mark(c, "set_image");
  c->coords_valid = false;
  c->width = width;
  c->height = height;
  if (c->device_io) {
    c->img_ptr = pixels;
  } else {
    FC_CUDA(c, c->img.reserve((size_t)width * height));
    FC_TRY(stage_h2d(c, c->img.ptr, pixels, (size_t)width * height));
    c->img_ptr = c->img.as<uint8_t>();
  }
  for (auto& L : c->lv) {
    L.n = 0;
    L.count = 0;
    L.prepared = false;
    L.tc.ready = false;
  }
  return FC_OK;
}

int fc_pool_build(fc_ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
                  const int32_t use_tau[4], int64_t out_sizes[4]) {
  cudaSetDevice(c->device);
  c->coords_valid = false;
  const double zero_taus[4] = {0, 0, 0, 0};
  const int32_t no_tau[4] = {0, 0, 0, 0};
  return pool_build(c, strides, caps, taus ? taus : zero_taus, use_tau ? use_tau : no_tau,
                    out_sizes);
}

int fc_pool_entropy(fc_ctx* c, const int32_t strides[4], const int64_t caps[4], const double taus[4],
                    const int32_t use_tau[4], const int32_t row_lo[4], const int32_t row_hi[4]) {
  cudaSetDevice(c->device);
  c->coords_valid = false;
  const double zero_taus[4] = {0, 0, 0, 0};
  const int32_t no_tau[4] = {0, 0, 0, 0};
  return pool_entropy(c, strides, caps, taus ? taus : zero_taus, use_tau ? use_tau : no_tau, row_lo,
                      row_hi);
}

int fc_pool_entropy_batch(fc_ctx** ctxs, int n, const int32_t strides[4], const int64_t caps[4],
                          const double taus[4], const int32_t use_tau[4]) {
  if (n < 1 || !ctxs) return FC_ERR_ARG;
  fc_ctx* c = ctxs[0];
  cudaSetDevice(c->device);
  for (int i = 0; i < n; ++i) ctxs[i]->coords_valid = false;
  const double zero_taus[4] = {0, 0, 0, 0};
  const int32_t no_tau[4] = {0, 0, 0, 0};
  std::vector<Ctx*> cs(ctxs, ctxs + n);
  return pool_entropy_batch(cs.data(), n, strides, caps, taus ? taus : zero_taus,
                            use_tau ? use_tau : no_tau);
}

int fc_pool_rank(fc_ctx* c, const int64_t sel_counts[4], int64_t out_sizes[4]) {
  cudaSetDevice(c->device);
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  if (sel_counts)
    for (int li = 0; li < 4; ++li)
      if (c->pool_use_tau[li] &&
          (sel_counts[li] < 0 || sel_counts[li] > (int64_t)c->pool_nx[li] * c->pool_ny[li]))
        return set_error(c, FC_ERR_ARG, "survivor count out of range");
  return pool_rank(c, sel_counts, out_sizes);
}

int fc_pool_window_buffers(fc_ctx* c, int level, void** key, void** val, void** ent, int64_t* nx,
                           int64_t* ny, int64_t* local_sel) {
  cudaSetDevice(c->device);
  FC_TRY(check_level(c, level));
  return pool_window_buffers(c, level - 1, key, val, ent, nx, ny, local_sel);
}

int fc_pool_set_level(fc_ctx* c, int level, int64_t count, const uint8_t* tiles) {
  cudaSetDevice(c->device);
  FC_TRY(check_level(c, level));
  if (count < 0 || (count > 0 && !tiles)) return set_error(c, FC_ERR_ARG, "bad tiles");
  c->coords_valid = false;
  return pool_set_level(c, level, count, tiles);
}

int fc_pool_size(fc_ctx* c, int level, int64_t* out_count) {
  FC_TRY(level_ready(c, level));
  *out_count = c->lv[level - 1].count;
  return FC_OK;
}

int fc_pool_coords(fc_ctx* c, int level, uint16_t* xy) {
  cudaSetDevice(c->device);
  FC_TRY(level_ready(c, level));
  Level& L = c->lv[level - 1];
  if (L.count == 0) return FC_OK;
  // xy words are x | y << 16: in little-endian memory exactly the (x, y) u16 pair
  if (c->coords_valid) {  // written to pinned memory by the pool build's survivors kernel
    FC_TRY(sync_stream(c));
    memcpy(xy, c->coords_pinned.as<uint32_t>() + c->coords_off[level - 1], L.count * 4);
    return FC_OK;
  }
  FC_CUDA(c, cudaMemcpyAsync(xy, L.xy.ptr, L.count * 4, cudaMemcpyDeviceToHost, c->stream));
  return sync_stream(c);
}

int fc_pool_coords_all(fc_ctx* c, uint16_t* xy) {
  cudaSetDevice(c->device);
  if (!xy) return set_error(c, FC_ERR_ARG, "null output");
  if (c->coords_valid) {  // one run per level, level 1 first, in pinned memory
    int64_t total = 0;
    for (int l = 0; l < kLevels; ++l) total += c->lv[l].count;
    FC_TRY(sync_stream(c));
    if (total) memcpy(xy, c->coords_pinned.ptr, total * 4);
    return FC_OK;
  }
  int64_t off = 0;
  for (int l = 0; l < kLevels; ++l) {
    FC_TRY(fc_pool_coords(c, l + 1, xy + 2 * off));
    off += c->lv[l].count;
  }
  return FC_OK;
}

int fc_pool_coords_view(fc_ctx* c, const uint16_t** out) {
  cudaSetDevice(c->device);
  if (!out) return set_error(c, FC_ERR_ARG, "null output");
  *out = nullptr;
  if (!c->coords_valid) return FC_OK;
  FC_TRY(sync_stream(c));
  *out = c->coords_pinned.as<uint16_t>();
  return FC_OK;
}

int fc_pool_entries(fc_ctx* c, int level, double* entropy, uint8_t* tiles, double* means,
                    double* cnorm) {
  cudaSetDevice(c->device);
  FC_TRY(level_ready(c, level));
  Level& L = c->lv[level - 1];
  if (L.count == 0) return FC_OK;
  if (entropy)
    FC_CUDA(c, cudaMemcpyAsync(entropy, L.ent.ptr, L.count * 8, cudaMemcpyDeviceToHost, c->stream));
  if (tiles)
    FC_CUDA(c, cudaMemcpyAsync(tiles, L.tiles.ptr, L.count * L.n, cudaMemcpyDeviceToHost, c->stream));
  if (means)
    FC_CUDA(c, cudaMemcpyAsync(means, L.mean.ptr, L.count * 8, cudaMemcpyDeviceToHost, c->stream));
  if (cnorm)
    FC_CUDA(c, cudaMemcpyAsync(cnorm, L.cnorm.ptr, L.count * 8, cudaMemcpyDeviceToHost, c->stream));
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_level_prepare(fc_ctx* c, int level, int baseline, const double* svals, int32_t s_count,
                     int32_t path) {
  cudaSetDevice(c->device);
  FC_TRY(level_ready(c, level));
  Level& L = c->lv[level - 1];
  int pending = 0, needs = 0;
  FC_TRY(prepare_begin(c, L, level, baseline, svals, s_count, path, &pending, &needs));
  if (needs) {
    Level* lv[1] = {&L};
    const int st[1] = {pending};
    FC_TRY(prep_launch(c, lv, st, 1));
  }
  return prepare_finish(c, L, path, pending);
}

static int run_match(fc_ctx* c, Level& L, int64_t count, int64_t* out_err, int64_t* out_idx,
                     double* out_rmean, bool device_out) {
  FC_CUDA(c, c->keys.reserve(count * 8));
  FC_CUDA(c, cudaMemsetAsync(c->keys.ptr, 0xff, count * 8, c->stream));
  FC_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  if (L.path == FC_PATH_TENSOR) {
    FC_TRY(scan_tc(c, L, count, c->keys.as<uint64_t>()));
  } else {
    FC_TRY(scan_exact(c, L, count, nullptr, 0, nullptr, 0, c->keys.as<uint64_t>()));
  }
  FC_CUDA(c, cudaEventRecord(c->ev2, c->stream));
  int64_t* d_err;
  int64_t* d_idx;
  if (device_out) {
    d_err = out_err;
    d_idx = out_idx;
  } else {
    FC_CUDA(c, c->out_err.reserve(count * 8));
    FC_CUDA(c, c->out_idx.reserve(count * 8));
    d_err = c->out_err.as<int64_t>();
    d_idx = c->out_idx.as<int64_t>();
  }
  FC_TRY(decode_keys(c, c->keys.as<uint64_t>(), count, d_err, d_idx));
  const cudaMemcpyKind kind = device_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (!device_out) {
    FC_CUDA(c, cudaMemcpyAsync(out_err, d_err, count * 8, kind, c->stream));
    FC_CUDA(c, cudaMemcpyAsync(out_idx, d_idx, count * 8, kind, c->stream));
  }
  if (out_rmean) FC_CUDA(c, cudaMemcpyAsync(out_rmean, c->rmean.ptr, count * 8, kind, c->stream));
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev2);
  c->stats.scan_ms = ms;
  if (L.path != FC_PATH_TENSOR) c->stats.main_ms = ms;
  return FC_OK;
}

static int begin_match(fc_ctx* c, int level, int64_t count) {
  FC_TRY(level_ready(c, level));
  Level& L = c->lv[level - 1];
  if (L.count == 0) {
    char buf[64];
    snprintf(buf, sizeof buf, "no domain entries at level %d", level);
    return set_error(c, FC_ERR_EMPTY_POOL, buf);
  }
  if (!L.prepared) return set_error(c, FC_ERR_STATE, "level not prepared");
  if (count < 0) return set_error(c, FC_ERR_ARG, "negative range count");
  c->total_launches += c->stats.kernel_launches;
  c->stats = fc_stats{};
  c->stats.ranges = count;
  c->stats.columns = L.count * L.s_count;
  c->stats.comparisons = count * L.count * 8 * L.s_count;
  c->stats.path = L.path;
  return FC_OK;
}

int fc_match_level(fc_ctx* c, int level, const int32_t* origins_xy, int64_t count, int64_t* out_err,
                   int64_t* out_idx, double* out_rmean) {
  cudaSetDevice(c->device);
  FC_TRY(begin_match(c, level, count));
  if (count == 0) return FC_OK;
  Level& L = c->lv[level - 1];
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  const int32_t* d_orig = origins_xy;
  if (!c->device_io) {
    for (int64_t i = 0; i < count; ++i) {
      const int x = origins_xy[2 * i], y = origins_xy[2 * i + 1];
      if (x < 0 || y < 0 || x + L.side > c->width || y + L.side > c->height)
        return set_error(c, FC_ERR_ARG, "range origin outside the image");
    }
    FC_CUDA(c, c->origins.reserve(count * 8));
    FC_CUDA(c, cudaMemcpyAsync(c->origins.ptr, origins_xy, count * 8, cudaMemcpyHostToDevice,
                               c->stream));
    d_orig = c->origins.as<int32_t>();
  }
  FC_TRY(gather_ranges(c, L, d_orig, count));
  return run_match(c, L, count, out_err, out_idx, out_rmean, c->device_io != 0);
}

// Real-valued slope search (bench.py:117-139 _real_s_matches over the ranges
// codec.py:164 _gather_tiles cuts at `origins_xy`): per range the exact fp64
// projection error, slope and flat index e*8 + iso of the first minimum.
// Needs the pool only (no fc_level_prepare); host buffers.
int fc_real_match_level(fc_ctx* c, int level, const int32_t* origins_xy, int64_t count,
                        double* out_err, double* out_s, int64_t* out_idx) {
  cudaSetDevice(c->device);
  FC_TRY(level_ready(c, level));
  Level& L = c->lv[level - 1];
  if (count < 0) return set_error(c, FC_ERR_ARG, "negative range count");
  if (c->device_io) return set_error(c, FC_ERR_STATE, "fc_real_match_level takes host buffers");
  if (!c->img_ptr) return set_error(c, FC_ERR_STATE, "no image set");
  if (L.count == 0) {
    char buf[64];
    snprintf(buf, sizeof buf, "no domain entries at level %d", level);
    return set_error(c, FC_ERR_EMPTY_POOL, buf);
  }
  c->total_launches += c->stats.kernel_launches;
  c->stats = fc_stats{};
  c->stats.ranges = count;
  c->stats.columns = L.count;
  c->stats.comparisons = count * L.count * 8;
  if (count == 0) return FC_OK;
  for (int64_t i = 0; i < count; ++i) {
    const int x = origins_xy[2 * i], y = origins_xy[2 * i + 1];
    if (x < 0 || y < 0 || x + L.side > c->width || y + L.side > c->height)
      return set_error(c, FC_ERR_ARG, "range origin outside the image");
  }
  FC_CUDA(c, c->origins.reserve(count * 8));
  FC_CUDA(c, cudaMemcpyAsync(c->origins.ptr, origins_xy, count * 8, cudaMemcpyHostToDevice,
                             c->stream));
  FC_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  FC_TRY(gather_ranges(c, L, c->origins.as<int32_t>(), count));
  FC_CUDA(c, c->real_out.reserve(count * 24));
  double* d_err = c->real_out.as<double>();
  double* d_s = d_err + count;
  auto* d_idx = reinterpret_cast<int64_t*>(d_s + count);
  FC_TRY(real_s_match(c, L, count, d_err, d_s, d_idx));
  FC_CUDA(c, cudaEventRecord(c->ev2, c->stream));
  FC_CUDA(c, cudaMemcpyAsync(out_err, d_err, count * 8, cudaMemcpyDeviceToHost, c->stream));
  FC_CUDA(c, cudaMemcpyAsync(out_s, d_s, count * 8, cudaMemcpyDeviceToHost, c->stream));
  if (out_idx)
    FC_CUDA(c, cudaMemcpyAsync(out_idx, d_idx, count * 8, cudaMemcpyDeviceToHost, c->stream));
  FC_CUDA(c, cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev0, c->ev2);
  c->stats.scan_ms = ms;
  c->stats.main_ms = ms;
  return FC_OK;
}

int fc_match_tiles(fc_ctx* c, int level, const uint8_t* tiles, int64_t count, int64_t* out_err,
                   int64_t* out_idx, double* out_rmean) {
  cudaSetDevice(c->device);
  FC_TRY(begin_match(c, level, count));
  if (count == 0) return FC_OK;
  Level& L = c->lv[level - 1];
  FC_TRY(load_ranges(c, L, tiles, count));
  return run_match(c, L, count, out_err, out_idx, out_rmean, false);
}

int fc_scan_candidates(fc_ctx* c, const int16_t* ranges, const double* rmeans, int64_t M, int32_t n,
                       const int16_t* q, const double* dmeans, int64_t E, const double* svals,
                       int32_t s_count, int32_t baseline, int64_t* out_err, int64_t* out_idx) {
  cudaSetDevice(c->device);
  if (M < 0 || n < 1 || E < 0 || s_count < 1) return set_error(c, FC_ERR_ARG, "bad scan shape");
  return scan_rows_dropin(c, ranges, rmeans, M, n, q, dmeans, E, svals, s_count, baseline, out_err,
                          out_idx);
}

int fc_encode(fc_ctx* c, const double thresholds[3], int32_t baseline, const double* svals,
              const int32_t s_counts[4], int32_t path, int32_t* records, int64_t capacity,
              int64_t* out_count) {
  cudaSetDevice(c->device);
  if (!thresholds || !svals || !s_counts) return set_error(c, FC_ERR_ARG, "null argument");
  return encode_device(c, thresholds, baseline, svals, s_counts, path, records, capacity,
                       out_count);
}

int fc_encode_records(fc_ctx* c, int32_t* records, int64_t capacity) {
  cudaSetDevice(c->device);
  if (c->enc_records > capacity) return set_error(c, FC_ERR_ARG, "record buffer too small");
  if (c->enc_records == 0) return FC_OK;
  memcpy(records, c->rec_pinned.ptr, c->enc_records * 24);
  return FC_OK;
}

int fc_encode_level_stats(fc_ctx* c, int level, fc_stats* out) {
  FC_TRY(check_level(c, level));
  if (!out) return set_error(c, FC_ERR_ARG, "null stats");
  *out = c->enc_stats[level - 1];
  return FC_OK;
}

int fc_decode(fc_ctx* c, const int32_t* leaves, int64_t n, int32_t width, int32_t height,
              const double* svals, const int32_t s_counts[4], int32_t proposed,
              int32_t iterations, int32_t tolerance, uint8_t* out_image, int32_t* out_deltas,
              int32_t* out_passes) {
  cudaSetDevice(c->device);
  return decode_device(c, leaves, n, width, height, svals, s_counts, proposed, iterations,
                       tolerance, out_image, out_deltas, out_passes);
}

int fc_encode_summary(fc_ctx* c, int64_t out[5]) {
  if (!out) return set_error(c, FC_ERR_ARG, "null output");
  for (int k = 0; k < 5; ++k) out[k] = c->enc_summary[k];
  return FC_OK;
}

int fc_last_stats(fc_ctx* c, fc_stats* out) {
  *out = c->stats;
  return FC_OK;
}

}  // extern "C"

extern "C" {

int fc_get_stream(fc_ctx* c, void** out_stream) {
  if (!out_stream) return set_error(c, FC_ERR_ARG, "null output");
  *out_stream = reinterpret_cast<void*>(c->stream);
  return FC_OK;
}

int fc_pool_times(fc_ctx* c, float out_ms[3]) {
  cudaSetDevice(c->device);
  if (!c->pool_timed) return set_error(c, FC_ERR_STATE, "no pool build timed yet");
  FC_CUDA(c, cudaEventSynchronize(c->pool_ev[2]));
  float a = 0.f, b = 0.f;
  FC_CUDA(c, cudaEventElapsedTime(&a, c->pool_ev[0], c->pool_ev[1]));
  FC_CUDA(c, cudaEventElapsedTime(&b, c->pool_ev[1], c->pool_ev[2]));
  out_ms[0] = a;
  out_ms[1] = b;
  out_ms[2] = a + b;
  return FC_OK;
}

int fc_launch_count(fc_ctx* c, int64_t* out_count) {
  if (!out_count) return set_error(c, FC_ERR_ARG, "null output");
  *out_count = c->total_launches + c->stats.kernel_launches;
  return FC_OK;
}

}  // extern "C"
