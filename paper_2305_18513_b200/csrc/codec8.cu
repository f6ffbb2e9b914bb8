// K1 quant8 / K2 dequant8: saturating 8-bit fixed point.
//
// Reference: compression.quantize / dequantize (compression.py:61-79), called
// through CompressedActivation.quantized / decompress (:193-197, :213-215).
// HBM-bound: 4 B read + 1 B written per element.  Lane i of a warp handles
// float4 i (each load instruction covers one contiguous 512 B span, each
// store one contiguous 128 B span); every thread keeps 4 independent
// float4 loads in flight (grid-stride, 4-way unrolled); grid = a multiple
// of the SM count.
#include "common.cuh"

namespace sf {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint32_t pack_bytes(int a, int b, int c, int d) {
  return (static_cast<uint32_t>(a) & 0xFFu) | ((static_cast<uint32_t>(b) & 0xFFu) << 8) |
         ((static_cast<uint32_t>(c) & 0xFFu) << 16) | ((static_cast<uint32_t>(d) & 0xFFu) << 24);
}

__device__ __forceinline__ uint32_t quant_f4(float4 v, float s, float lo, float hi) {
  return pack_bytes(fixed_code(v.x, s, lo, hi), fixed_code(v.y, s, lo, hi),
                    fixed_code(v.z, s, lo, hi), fixed_code(v.w, s, lo, hi));
}

__global__ void __launch_bounds__(kThreads) k_quant8_vec(const float4* __restrict__ x,
                                                         uint32_t* __restrict__ out, int64_t n4,
                                                         float scale, float lo, float hi) {
  const int64_t S = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * S < n4; i += kUnroll * S) {
    float4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(x + i + u * S);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) out[i + u * S] = quant_f4(v[u], scale, lo, hi);
  }
  for (; i < n4; i += S) out[i] = quant_f4(ld_stream(x + i), scale, lo, hi);
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
__global__ void __launch_bounds__(kThreads) k_dequant8_vec(const uint32_t* __restrict__ codes,
                                                           float4* __restrict__ y, int64_t n4,
                                                           float inv) {
  const int64_t S = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * S < n4; i += kUnroll * S) {
    uint32_t w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) w[u] = __ldg(codes + i + u * S);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) y[i + u * S] = decode_word<SIGNED>(w[u], inv);
  }
  for (; i < n4; i += S) y[i] = decode_word<SIGNED>(__ldg(codes + i), inv);
}

template <bool SIGNED>
__global__ void k_dequant8_scalar(const uint8_t* __restrict__ codes, float* __restrict__ y,
                                  int64_t begin, int64_t n, float inv) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    y[i] = decode_byte<SIGNED>(codes[i], inv);
}

// float64 input (compression.quantize on a float64 array): the reference
// rounds in float64 as copysign(floor(|v| + 0.5), v) -- an f64 add whose
// rounding this reproduces literally (for v just below a half, |v| + 0.5
// can round up to the next integer, as it does in numpy).  NaN -> 0 and
// +-inf saturate, the reference's observed behaviour.  API-only path.
__global__ void k_quant_f64(const double* __restrict__ x, uint8_t* __restrict__ out, int64_t n,
                            double scale, double lo, double hi) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = __dmul_rn(x[i], scale);       // exact: scale is a power of two
    int c = 0;
    if (!isnan(v)) {
      double r = floor(__dadd_rn(fabs(v), 0.5));
      r = copysign(r, v);
      r = fmin(fmax(r, lo), hi);
      c = static_cast<int>(r);
    }
    out[i] = static_cast<uint8_t>(c & 0xFF);
  }
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
  const bool vec = aligned16(x) && (reinterpret_cast<uintptr_t>(out) & 3u) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  if (n4 > 0)
    k_quant8_vec<<<grid_for(n4, kThreads), kThreads, 0, s>>>(
        reinterpret_cast<const float4*>(x), reinterpret_cast<uint32_t*>(out), n4, scale, lo, hi);
  if (n4 * 4 < n)
    k_quant8_scalar<<<grid_for(n - n4 * 4, kThreads), kThreads, 0, s>>>(x, out, n4 * 4, n, scale,
                                                                       lo, hi);
  return check_launch();
}

int sf_quantize_f64(const double* x, void* codes, int64_t n, int bits, int fb, int is_signed,
                    void* stream) {
  if (n < 0 || (bits != 4 && bits != 8) || fb < 0 || fb > bits || (n > 0 && (!x || !codes)))
    return SF_EINVAL;
  if (n == 0) return SF_OK;
  const double lo = is_signed ? -static_cast<double>(1 << (bits - 1)) : 0.0;
  const double hi = is_signed ? static_cast<double>((1 << (bits - 1)) - 1) : static_cast<double>((1 << bits) - 1);
  k_quant_f64<<<grid_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
      x, static_cast<uint8_t*>(codes), n, static_cast<double>(1 << fb), lo, hi);
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
  const bool vec = aligned16(y) && (reinterpret_cast<uintptr_t>(c) & 3u) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  const uint32_t* c4 = reinterpret_cast<const uint32_t*>(c);
  float4* y4 = reinterpret_cast<float4*>(y);
  if (is_signed) {
    if (n4 > 0) k_dequant8_vec<true><<<grid_for(n4, kThreads), kThreads, 0, s>>>(c4, y4, n4, inv);
    if (n4 * 4 < n)
      k_dequant8_scalar<true><<<grid_for(n - n4 * 4, kThreads), kThreads, 0, s>>>(c, y, n4 * 4, n,
                                                                                 inv);
  } else {
    if (n4 > 0) k_dequant8_vec<false><<<grid_for(n4, kThreads), kThreads, 0, s>>>(c4, y4, n4, inv);
    if (n4 * 4 < n)
      k_dequant8_scalar<false><<<grid_for(n - n4 * 4, kThreads), kThreads, 0, s>>>(c, y, n4 * 4, n,
                                                                                  inv);
  }
  return check_launch();
}

}  // extern "C"
