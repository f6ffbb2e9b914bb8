// Attention head layout moves with the projection bias fused in.
//
// Reference: the encoder splits the q/k/v projections into heads and merges
// the context back (model.py:202-238 via reshape/transpose), after
// `x @ W + b` (tensor.py:337-379).  Here the projections run as plain GEMMs
// and one pass adds the bias while moving (B, T, h, dh) -> (B, h, T, dh),
// optionally emitting the Q4.4 codes the matmul cache stores (the codes of
// exactly the values written, as `quantize` would produce them).  The merge
// is the inverse move.  Both are pure HBM streams: 8 B/elt (+1 with codes).
#include <cub/device/device_radix_sort.cuh>

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

// Embedding backward: dW[v] = sum of g rows whose token id is v, added in
// position order (numpy's np.add.at order, tensor.py:497-520).  The ids
// are stable-sorted on the device beforehand (perm = positions in id
// order, starts[v] .. starts[v + 1] = the occurrences of v), so no host
// round trip is needed to size anything -- torch's embedding backward
// synchronises the host to count the unique ids.  One warp per table row;
// rows without occurrences are written as zeros (the dense gradient).
template <int VPL>
__global__ void __launch_bounds__(256) k_embedding_bwd(const float* __restrict__ g,
                                                       const int64_t* __restrict__ perm,
                                                       const int64_t* __restrict__ starts, float* __restrict__ dw,
                                                       int64_t V, int H) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t v = warp0; v < V; v += nwarps) {
    const int64_t a = __ldg(starts + v), b = __ldg(starts + v + 1);
    float4 acc[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = a; p < b; ++p) {
      const float4* gr = reinterpret_cast<const float4*>(g + __ldg(perm + p) * H);
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int c = lane + 32 * j;
        if (4 * c < H) {
          const float4 x = __ldg(gr + c);
          acc[j] = make_float4(acc[j].x + x.x, acc[j].y + x.y, acc[j].z + x.z, acc[j].w + x.w);
        }
      }
    }
    float4* out = reinterpret_cast<float4*>(dw + v * H);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) out[c] = acc[j];
    }
  }
}

__global__ void k_ids_to_keys(const int64_t* __restrict__ ids, int64_t n, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ pos) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    keys[i] = static_cast<uint32_t>(ids[i]);
    pos[i] = static_cast<uint32_t>(i);
  }
}

// starts[v] = first index in the sorted keys with key >= v (v = 0..V)
__global__ void k_segment_starts(const uint32_t* __restrict__ skeys, int64_t n, int64_t V,
                                 int64_t* __restrict__ starts) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v <= V;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(skeys[mid]) < v) lo = mid + 1; else hi = mid;
    }
    starts[v] = lo;
  }
}

template <int VPL>
__global__ void __launch_bounds__(256) k_embedding_bwd32(const float* __restrict__ g,
                                                         const uint32_t* __restrict__ perm,
                                                         const int64_t* __restrict__ starts,
                                                         float* __restrict__ dw, int64_t V, int H) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t v = warp0; v < V; v += nwarps) {
    const int64_t a = __ldg(starts + v), b = __ldg(starts + v + 1);
    float4 acc[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t p = a; p < b; ++p) {
      const float4* gr = reinterpret_cast<const float4*>(g + static_cast<int64_t>(__ldg(perm + p)) * H);
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int c = lane + 32 * j;
        if (4 * c < H) {
          const float4 x = __ldg(gr + c);
          acc[j] = make_float4(acc[j].x + x.x, acc[j].y + x.y, acc[j].z + x.z, acc[j].w + x.w);
        }
      }
    }
    float4* out = reinterpret_cast<float4*>(dw + v * H);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) out[c] = acc[j];
    }
  }
}

inline int end_bit_for(int64_t V) {
  int b = 1;
  while ((int64_t(1) << b) < V) ++b;
  return b;
}

inline size_t a256h(size_t b) { return (b + 255) & ~size_t(255); }

inline size_t cub_sort_bytes(int64_t n, int end_bit) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<int>(n), 0, end_bit);
  return tmp;
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

int sf_embedding_bwd(const float* g, const int64_t* perm, const int64_t* starts, float* dw, int64_t V,
                     int64_t H, void* stream) {
  if (V <= 0 || H < 4 || H % 4 || H > 1024 || !g || !perm || !starts || !dw || !aligned16(g) || !aligned16(dw))
    return SF_EINVAL;
  const unsigned grid = grid_for(V * 32, 256, 8);
  cudaStream_t s = as_stream(stream);
  const int h = static_cast<int>(H);
  if (H <= 128) k_embedding_bwd<1><<<grid, 256, 0, s>>>(g, perm, starts, dw, V, h);
  else if (H <= 256) k_embedding_bwd<2><<<grid, 256, 0, s>>>(g, perm, starts, dw, V, h);
  else if (H <= 512) k_embedding_bwd<4><<<grid, 256, 0, s>>>(g, perm, starts, dw, V, h);
  else if (H <= 768) k_embedding_bwd<6><<<grid, 256, 0, s>>>(g, perm, starts, dw, V, h);
  else k_embedding_bwd<8><<<grid, 256, 0, s>>>(g, perm, starts, dw, V, h);
  return check_launch();
}

size_t sf_embedding_grad_workspace_bytes(int64_t n, int64_t V) {
  if (n <= 0 || V <= 0) return 256;
  return 4 * a256h(static_cast<size_t>(n) * 4) + a256h(static_cast<size_t>(V + 1) * 8) +
         a256h(cub_sort_bytes(n, end_bit_for(V)));
}

int sf_embedding_grad(const int64_t* ids, int64_t n, const float* g, float* dw, int64_t V, int64_t H, void* ws,
                      void* stream) {
  if (n <= 0 || n > 0x7FFFFFFF || V <= 0 || V > 0x7FFFFFFF || H < 4 || H % 4 || H > 1024 || !ids || !g ||
      !dw || !ws || !aligned16(g) || !aligned16(dw))
    return SF_EINVAL;
  cudaStream_t s = as_stream(stream);
  char* w = static_cast<char*>(ws);
  uint32_t* keys = reinterpret_cast<uint32_t*>(w);
  w += a256h(static_cast<size_t>(n) * 4);
  uint32_t* pos = reinterpret_cast<uint32_t*>(w);
  w += a256h(static_cast<size_t>(n) * 4);
  uint32_t* skeys = reinterpret_cast<uint32_t*>(w);
  w += a256h(static_cast<size_t>(n) * 4);
  uint32_t* spos = reinterpret_cast<uint32_t*>(w);
  w += a256h(static_cast<size_t>(n) * 4);
  int64_t* starts = reinterpret_cast<int64_t*>(w);
  w += a256h(static_cast<size_t>(V + 1) * 8);
  const int eb = end_bit_for(V);
  size_t tmp = cub_sort_bytes(n, eb);
  k_ids_to_keys<<<grid_for(n, 256, 4), 256, 0, s>>>(ids, n, keys, pos);
  // LSD radix sort: stable, so each id's positions stay in increasing order
  if (cub::DeviceRadixSort::SortPairs(w, tmp, keys, skeys, pos, spos, static_cast<int>(n), 0, eb, s) !=
      cudaSuccess)
    return check_launch();
  k_segment_starts<<<grid_for(V + 1, 256, 4), 256, 0, s>>>(skeys, n, V, starts);
  const unsigned grid = grid_for(V * 32, 256, 8);
  const int h = static_cast<int>(H);
  if (H <= 128) k_embedding_bwd32<1><<<grid, 256, 0, s>>>(g, spos, starts, dw, V, h);
  else if (H <= 256) k_embedding_bwd32<2><<<grid, 256, 0, s>>>(g, spos, starts, dw, V, h);
  else if (H <= 512) k_embedding_bwd32<4><<<grid, 256, 0, s>>>(g, spos, starts, dw, V, h);
  else if (H <= 768) k_embedding_bwd32<6><<<grid, 256, 0, s>>>(g, spos, starts, dw, V, h);
  else k_embedding_bwd32<8><<<grid, 256, 0, s>>>(g, spos, starts, dw, V, h);
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
