// K1 quant8 / K2 dequant8: saturating 8-bit fixed point.
//
// Reference: compression.quantize / dequantize (compression.py:61-79), called
// through CompressedActivation.quantized / decompress (:193-197, :213-215).
// HBM-bound: 4 B read + 1 B write per element.  Each thread moves 16
// elements per iteration with four 128-bit streaming loads and one 128-bit
// store; the grid is a multiple of the SM count (grid-stride loop).
#include "common.cuh"

namespace sf {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t pack_bytes(int a, int b, int c, int d) {
  return (static_cast<uint32_t>(a) & 0xFFu) | ((static_cast<uint32_t>(b) & 0xFFu) << 8) |
         ((static_cast<uint32_t>(c) & 0xFFu) << 16) | ((static_cast<uint32_t>(d) & 0xFFu) << 24);
}

__device__ __forceinline__ uint32_t quant_f4(float4 v, float s, float lo, float hi) {
  return pack_bytes(fixed_code(v.x, s, lo, hi), fixed_code(v.y, s, lo, hi),
                    fixed_code(v.z, s, lo, hi), fixed_code(v.w, s, lo, hi));
}

__global__ void __launch_bounds__(kThreads) k_quant8_vec(const float* __restrict__ x,
                                                         uint8_t* __restrict__ out, int64_t n16,
                                                         float scale, float lo, float hi) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += stride) {
    const float4* p = reinterpret_cast<const float4*>(x) + i * 4;
    float4 a = ld_stream(p), b = ld_stream(p + 1), c = ld_stream(p + 2), d = ld_stream(p + 3);
    uint4 w;
    w.x = quant_f4(a, scale, lo, hi);
    w.y = quant_f4(b, scale, lo, hi);
    w.z = quant_f4(c, scale, lo, hi);
    w.w = quant_f4(d, scale, lo, hi);
    reinterpret_cast<uint4*>(out)[i] = w;
  }
}

__global__ void k_quant8_scalar(const float* __restrict__ x, uint8_t* __restrict__ out,
                                int64_t begin, int64_t n, float scale, float lo, float hi) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = static_cast<uint8_t>(fixed_code(x[i], scale, lo, hi) & 0xFF);
}

template <bool SIGNED>
__device__ __forceinline__ float decode_byte(uint32_t byte, float inv) {
  int c = SIGNED ? static_cast<int>(static_cast<int8_t>(byte)) : static_cast<int>(byte);
  return static_cast<float>(c) * inv;   // exact: |c| < 2^8, inv a power of two
}

template <bool SIGNED>
__device__ __forceinline__ float4 decode_word(uint32_t w, float inv) {
  return make_float4(decode_byte<SIGNED>(w & 0xFF, inv), decode_byte<SIGNED>((w >> 8) & 0xFF, inv),
                     decode_byte<SIGNED>((w >> 16) & 0xFF, inv), decode_byte<SIGNED>(w >> 24, inv));
}

template <bool SIGNED>
__global__ void __launch_bounds__(kThreads) k_dequant8_vec(const uint8_t* __restrict__ codes,
                                                           float* __restrict__ y, int64_t n16,
                                                           float inv) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += stride) {
    uint4 w = ld_stream_u4(reinterpret_cast<const uint4*>(codes) + i);
    float4* o = reinterpret_cast<float4*>(y) + i * 4;
    o[0] = decode_word<SIGNED>(w.x, inv);
    o[1] = decode_word<SIGNED>(w.y, inv);
    o[2] = decode_word<SIGNED>(w.z, inv);
    o[3] = decode_word<SIGNED>(w.w, inv);
  }
}

template <bool SIGNED>
__global__ void k_dequant8_scalar(const uint8_t* __restrict__ codes, float* __restrict__ y,
                                  int64_t begin, int64_t n, float inv) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    y[i] = decode_byte<SIGNED>(codes[i], inv);
}

}  // namespace sf

using namespace sf;

extern "C" {

int sf_quantize(const float* x, void* codes, int64_t n, int bits, int fb, int is_signed,
                void* stream) {
  if (n < 0 || (bits != 4 && bits != 8) || fb < 0 || fb > bits || (n > 0 && (!x || !codes)))
    return SF_EINVAL;
  if (n == 0) return SF_OK;
  const float scale = static_cast<float>(1 << fb);
  const float lo = is_signed ? -static_cast<float>(1 << (bits - 1)) : 0.f;
  const float hi = is_signed ? static_cast<float>((1 << (bits - 1)) - 1)
                             : static_cast<float>((1 << bits) - 1);
  cudaStream_t s = as_stream(stream);
  uint8_t* out = static_cast<uint8_t*>(codes);
  int64_t n16 = (aligned16(x) && aligned16(out)) ? n / 16 : 0;
  if (n16 > 0)
    k_quant8_vec<<<grid_for(n16, kThreads), kThreads, 0, s>>>(x, out, n16, scale, lo, hi);
  if (n16 * 16 < n)
    k_quant8_scalar<<<grid_for(n - n16 * 16, kThreads), kThreads, 0, s>>>(x, out, n16 * 16, n,
                                                                         scale, lo, hi);
  return check_launch();
}

int sf_quant8(const float* x, void* codes, int64_t n, int fb, int is_signed, void* stream) {
  return sf_quantize(x, codes, n, 8, fb, is_signed, stream);
}

int sf_dequant8(const void* codes, float* y, int64_t n, int fb, int is_signed, void* stream) {
  if (n < 0 || fb < 0 || fb > 8 || (n > 0 && (!codes || !y))) return SF_EINVAL;
  if (n == 0) return SF_OK;
  const float inv = 1.0f / static_cast<float>(1 << fb);
  cudaStream_t s = as_stream(stream);
  const uint8_t* c = static_cast<const uint8_t*>(codes);
  int64_t n16 = (aligned16(c) && aligned16(y)) ? n / 16 : 0;
  if (is_signed) {
    if (n16 > 0) k_dequant8_vec<true><<<grid_for(n16, kThreads), kThreads, 0, s>>>(c, y, n16, inv);
    if (n16 * 16 < n)
      k_dequant8_scalar<true><<<grid_for(n - n16 * 16, kThreads), kThreads, 0, s>>>(c, y, n16 * 16,
                                                                                    n, inv);
  } else {
    if (n16 > 0)
      k_dequant8_vec<false><<<grid_for(n16, kThreads), kThreads, 0, s>>>(c, y, n16, inv);
    if (n16 * 16 < n)
      k_dequant8_scalar<false><<<grid_for(n - n16 * 16, kThreads), kThreads, 0, s>>>(
          c, y, n16 * 16, n, inv);
  }
  return check_launch();
}

}  // extern "C"
