// Attention head layout moves with the projection bias fused in.
//
// Reference: the encoder splits the q/k/v projections into heads and merges
// the context back (model.py:202-238 via reshape/transpose), after
// `x @ W + b` (tensor.py:337-379).  Here the projections run as plain GEMMs
// and one pass adds the bias while moving (B, T, h, dh) -> (B, h, T, dh),
// optionally emitting the Q4.4 codes the matmul cache stores (the codes of
// exactly the values written, as `quantize` would produce them).  The merge
// is the inverse move.  Both are pure HBM streams: 8 B/elt (+1 with codes).
#include "common.cuh"

namespace sf {

constexpr int kHT = 256;

// one thread per output float4; planes (b, j) on blockIdx.y, (t, d4) inside
template <bool BIAS, bool CODES>
__global__ void __launch_bounds__(kHT) k_split_heads(const float4* __restrict__ y,
                                                     const float4* __restrict__ bias,
                                                     float4* __restrict__ out,
                                                     uint32_t* __restrict__ codes, int T, int h,
                                                     int dh4, float scale, float lo, float hi) {
  const int plane = blockIdx.y;                     // b * h + j
  const int b = plane / h, j = plane - (plane / h) * h;
  const int per_plane = T * dh4;
  const int p = blockIdx.x * kHT + threadIdx.x;
  if (p >= per_plane) return;
  const int t = p / dh4, d = p - (p / dh4) * dh4;
  const int64_t src = (static_cast<int64_t>(b) * T + t) * h * dh4 + static_cast<int64_t>(j) * dh4 + d;
  float4 v = __ldg(y + src);
  if (BIAS) {
    const float4 c = __ldg(bias + j * dh4 + d);
    v = make_float4(v.x + c.x, v.y + c.y, v.z + c.z, v.w + c.w);
  }
  const int64_t dst = static_cast<int64_t>(plane) * per_plane + p;
  out[dst] = v;
  if (CODES) {
    const uint32_t c0 = static_cast<uint8_t>(fixed_code(v.x, scale, lo, hi));
    const uint32_t c1 = static_cast<uint8_t>(fixed_code(v.y, scale, lo, hi));
    const uint32_t c2 = static_cast<uint8_t>(fixed_code(v.z, scale, lo, hi));
    const uint32_t c3 = static_cast<uint8_t>(fixed_code(v.w, scale, lo, hi));
    codes[dst] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
  }
}

__global__ void __launch_bounds__(kHT) k_merge_heads(const float4* __restrict__ x,
                                                     float4* __restrict__ out, int T, int h,
                                                     int dh4, int64_t ld4) {
  const int plane = blockIdx.y;
  const int b = plane / h, j = plane - (plane / h) * h;
  const int per_plane = T * dh4;
  const int p = blockIdx.x * kHT + threadIdx.x;
  if (p >= per_plane) return;
  const int t = p / dh4, d = p - (p / dh4) * dh4;
  const int64_t dst = (static_cast<int64_t>(b) * T + t) * ld4 + static_cast<int64_t>(j) * dh4 + d;
  out[dst] = __ldg(x + static_cast<int64_t>(plane) * per_plane + p);
}

inline bool heads_ok(int64_t B, int64_t T, int64_t h, int64_t dh) {
  return B > 0 && T > 0 && h > 0 && dh > 0 && dh % 4 == 0 && B * h <= 65535 &&
         T * (dh / 4) <= 0x7FFFFFFF;
}

}  // namespace sf

using namespace sf;

extern "C" {

int sf_split_heads(const float* y, const float* bias, float* out, void* codes, int64_t B, int64_t T,
                   int64_t heads, int64_t dh, int fb, int is_signed, void* stream) {
  if (!y || !out || !heads_ok(B, T, heads, dh) || !aligned16(y) || !aligned16(out) ||
      (bias && !aligned16(bias)) || (codes && ((reinterpret_cast<uintptr_t>(codes) & 3u) || fb < 0 || fb > 8)))
    return SF_EINVAL;
  const int dh4 = static_cast<int>(dh / 4);
  const int per_plane = static_cast<int>(T) * dh4;
  const dim3 grid((per_plane + kHT - 1) / kHT, static_cast<unsigned>(B * heads));
  const float scale = static_cast<float>(1 << fb);
  const float lo = is_signed ? -128.f : 0.f, hi = is_signed ? 127.f : 255.f;
  cudaStream_t s = as_stream(stream);
  const float4* y4 = reinterpret_cast<const float4*>(y);
  const float4* b4 = reinterpret_cast<const float4*>(bias);
  float4* o4 = reinterpret_cast<float4*>(out);
  uint32_t* c4 = static_cast<uint32_t*>(codes);
  const int T32 = static_cast<int>(T), h32 = static_cast<int>(heads);
  if (bias && codes)
    k_split_heads<true, true><<<grid, kHT, 0, s>>>(y4, b4, o4, c4, T32, h32, dh4, scale, lo, hi);
  else if (bias)
    k_split_heads<true, false><<<grid, kHT, 0, s>>>(y4, b4, o4, c4, T32, h32, dh4, scale, lo, hi);
  else if (codes)
    k_split_heads<false, true><<<grid, kHT, 0, s>>>(y4, b4, o4, c4, T32, h32, dh4, scale, lo, hi);
  else
    k_split_heads<false, false><<<grid, kHT, 0, s>>>(y4, b4, o4, c4, T32, h32, dh4, scale, lo, hi);
  return check_launch();
}

int sf_merge_heads(const float* x, float* out, int64_t B, int64_t T, int64_t heads, int64_t dh,
                   void* stream) {
  return sf_merge_heads_ld(x, out, B, T, heads, dh, heads * dh, stream);
}

int sf_merge_heads_ld(const float* x, float* out, int64_t B, int64_t T, int64_t heads, int64_t dh,
                      int64_t out_ld, void* stream) {
  if (!x || !out || !heads_ok(B, T, heads, dh) || !aligned16(x) || !aligned16(out) ||
      out_ld < heads * dh || out_ld % 4)
    return SF_EINVAL;
  const int dh4 = static_cast<int>(dh / 4);
  const int per_plane = static_cast<int>(T) * dh4;
  const dim3 grid((per_plane + kHT - 1) / kHT, static_cast<unsigned>(B * heads));
  k_merge_heads<<<grid, kHT, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(x),
                                                      reinterpret_cast<float4*>(out),
                                                      static_cast<int>(T), static_cast<int>(heads), dh4,
                                                      out_ld / 4);
  return check_launch();
}

}  // extern "C"
