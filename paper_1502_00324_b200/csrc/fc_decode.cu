// Device decoder: the iterated collage pass of the reference decoder
// (codec.py:257-363 decode_trace; our host restatement codec._collage_pass).
//
// Every leaf (range block) of one pass reads the current image and writes its
// own B x B block of the next one, so a pass is one launch over the leaves:
//  * the 2B x 2B domain at (dx, dy) of the current image, decimated
//    floor((a + b + c + d) / 4) (image.py:116-130),
//  * the leaf's isometry (image.py:140-155: out[i][j] = t[r][c]),
//  * proposed mode q = rint(s * (t - mean)), mean = sum / n (exact, n a power
//    of two); baseline q = rint(s * t) -- float64, separately rounded ops
//    (no FMA) like numpy -- then clip(q + offset, 0, 255),
//  * the pass's max |new - cur| (the reference's convergence delta).
// The passes run back to back on the device; a pass that reaches delta <=
// tolerance raises a flag and later passes return at once, so the host
// synchronises once for the whole decode.
#include "fc_internal.cuh"

namespace fcb {

namespace {

struct DecodeLeaf {  // one range block of the stream, host-built (iter_leaves order)
  int32_t rx, ry;    // range origin
  int32_t level;     // 1..4 (B = 16 >> (level - 1))
  int32_t dx, dy;    // domain origin (pool coordinates of the record's address)
  int32_t iso, sidx, offset;
};
static_assert(sizeof(DecodeLeaf) == 32, "C ABI row layout (8 x int32)");

struct DecodeParams {
  const DecodeLeaf* leaves;
  int64_t n_leaves;
  const double* svals;  // [4][kMaxS] per-level s values
  int width, height, proposed, tolerance;
  int32_t* state;       // [0] = converged flag, [1 + it] = delta of pass it
};

// One warp per leaf; lane p < n handles output pixel p of the B x B block
// (B <= 16: up to 8 pixels per lane).
__global__ void __launch_bounds__(256) collage_pass_kernel(DecodeParams P, int it,
                                                           const uint8_t* __restrict__ cur,
                                                           uint8_t* __restrict__ out) {
  if (P.state[0]) return;  // an earlier pass converged: keep its image
  const int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int delta = 0;
  if (leaf < P.n_leaves) {
    const DecodeLeaf L = P.leaves[leaf];
    const int B = 16 >> (L.level - 1), n = B * B, b = B - 1;
    const double s = P.svals[(L.level - 1) * kMaxS + L.sidx];
    constexpr int kPer = 8;  // pixels per lane (n <= 256)
    int tv[kPer];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int p = lane + 32 * k;
      tv[k] = 0;
      if (p < n) {
        const int i = p / B, j = p - i * B;  // output pixel (i, j) = decimated t[r][c]
        int r = i, c = j;
        switch (L.iso) {
          case 0: r = i; c = j; break;
          case 1: r = b - j; c = i; break;
          case 2: r = b - i; c = b - j; break;
          case 3: r = j; c = b - i; break;
          case 4: r = i; c = b - j; break;
          case 5: r = j; c = i; break;
          case 6: r = b - i; c = j; break;
          default: r = b - j; c = b - i; break;
        }
        const uint8_t* d = cur + (int64_t)(L.dy + 2 * r) * P.width + L.dx + 2 * c;
        const int v = ((int)d[0] + d[1] + d[P.width] + d[P.width + 1]) >> 2;
        tv[k] = v;
        sum += v;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const double mean = __ddiv_rn((double)sum, (double)n);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int p = lane + 32 * k;
      if (p < n) {
        const int i = p / B, j = p - i * B;
        const double x = P.proposed ? __dsub_rn((double)tv[k], mean) : (double)tv[k];
        int v = (int)rint(__dmul_rn(s, x)) + L.offset;
        v = v < 0 ? 0 : (v > 255 ? 255 : v);
        const int64_t a = (int64_t)(L.ry + i) * P.width + L.rx + j;
        const int old = cur[a];
        out[a] = (uint8_t)v;
        delta = max(delta, abs(v - old));
      }
    }
  }
  delta = __reduce_max_sync(0xffffffffu, delta);
  if (lane == 0 && delta > 0) atomicMax(&P.state[1 + it], delta);
}

// The pass's delta is final once every block of the pass has run: the flag
// for the following passes is raised by a one-thread kernel in between.
__global__ void converge_kernel(int32_t* state, int it, int tolerance) {
  if (!state[0] && state[1 + it] <= tolerance) state[0] = it + 1;  // passes run
}

}  // namespace

int decode_device(Ctx* c, const int32_t* leaves, int64_t n_leaves, int width, int height,
                  const double* svals, const int32_t* s_counts, int proposed, int iterations,
                  int tolerance, uint8_t* out_image, int32_t* out_deltas, int32_t* out_passes) {
  if (width < 1 || height < 1 || iterations < 1 || tolerance < 0 || n_leaves < 0 ||
      (n_leaves > 0 && !leaves) || !svals || !s_counts || !out_image)
    return set_error(c, FC_ERR_ARG, "bad decode arguments");
  const int64_t npx = (int64_t)width * height;
  FC_CUDA(c, c->dec_img.reserve(2 * npx + 64));
  FC_CUDA(c, c->dec_leaves.reserve(n_leaves * sizeof(DecodeLeaf) + 64));
  FC_CUDA(c, c->dec_state.reserve((2 + (size_t)iterations) * 4 + 64));
  double sv[kLevels * kMaxS] = {0};
  for (int l = 0, o = 0; l < kLevels; o += s_counts[l], ++l) {
    if (s_counts[l] < 0 || s_counts[l] > kMaxS) return set_error(c, FC_ERR_ARG, "bad s set size");
    for (int k = 0; k < s_counts[l]; ++k) sv[l * kMaxS + k] = svals[o + k];
  }
  FC_CUDA(c, c->dec_svals.reserve(sizeof sv));
  FC_TRY(stage_h2d(c, c->dec_svals.ptr, sv, sizeof sv));
  if (n_leaves) FC_TRY(stage_h2d(c, c->dec_leaves.ptr, leaves, n_leaves * sizeof(DecodeLeaf)));
  uint8_t* img[2] = {c->dec_img.as<uint8_t>(), c->dec_img.as<uint8_t>() + npx};
  FC_CUDA(c, cudaMemsetAsync(img[0], 128, npx, c->stream));  // codec.py: start from mid-gray
  FC_CUDA(c, cudaMemsetAsync(c->dec_state.ptr, 0, (2 + (size_t)iterations) * 4, c->stream));
  DecodeParams P{};
  P.leaves = c->dec_leaves.as<DecodeLeaf>();
  P.n_leaves = n_leaves;
  P.svals = c->dec_svals.as<double>();
  P.width = width;
  P.height = height;
  P.proposed = proposed;
  P.tolerance = tolerance;
  P.state = c->dec_state.as<int32_t>();
  const unsigned grid = (unsigned)std::max<int64_t>(1, (n_leaves * 32 + 255) / 256);
  for (int it = 0; it < iterations; ++it) {
    // a converged pass leaves its output in img[(it + 1) & 1]; later passes
    // return without touching either buffer
    collage_pass_kernel<<<grid, 256, 0, c->stream>>>(P, it, img[it & 1], img[(it + 1) & 1]);
    converge_kernel<<<1, 1, 0, c->stream>>>(P.state, it, tolerance);
  }
  FC_CUDA(c, cudaGetLastError());
  c->total_launches += 2 * iterations;
  FC_CUDA(c, c->readback.reserve((2 + (size_t)iterations) * 4 + 64));
  int32_t* h_state = c->readback.as<int32_t>();
  FC_CUDA(c, cudaMemcpyAsync(h_state, c->dec_state.ptr, (2 + (size_t)iterations) * 4,
                             cudaMemcpyDeviceToHost, c->stream));
  FC_TRY(sync_stream(c));
  const int passes = h_state[0] ? h_state[0] : iterations;
  FC_CUDA(c, cudaMemcpy(out_image, img[passes & 1], npx, cudaMemcpyDeviceToHost));
  if (out_deltas)
    for (int it = 0; it < passes; ++it) out_deltas[it] = h_state[1 + it];
  if (out_passes) *out_passes = passes;
  return FC_OK;
}

}  // namespace fcb
