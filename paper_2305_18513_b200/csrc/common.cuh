// Shared helpers for the sm_100a kernels behind include/slimfit_b200.h.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "slimfit_b200.h"

namespace sf {

// Thread-local last CUDA error (sf_last_cuda_error); defined in capi.cu.
void set_cuda_error(cudaError_t e);

inline int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_cuda_error(e);
    return SF_ECUDA;
  }
  return SF_OK;
}

// SM count of the current device, cached per device ordinal.
int num_sms();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// Grid for a grid-stride loop over `work` items: enough CTAs to keep
// ~`per_sm` resident per SM, never more than the work needs.
inline unsigned grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t need = (work + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
  if (need < 1) need = 1;
  return static_cast<unsigned>(need < cap ? need : cap);
}

// Streaming 128-bit load that does not allocate in L1 (data read once).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  // not volatile: read-only data, so the compiler may hoist and batch these
  // loads (volatile asm kept them serialized behind the arithmetic)
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Dynamic shared memory above 48 KB must be opted into per function and
// per device; `flags` is a per-call-site bitmask of devices already done.
template <typename K>
inline void smem_optin(K kernel, size_t bytes, unsigned long long& flags) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  const unsigned long long bit = 1ull << dev;
  if (flags & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  flags |= bit;
}

// ---- Programmatic dependent launch (PDL).  A kernel launched with
// launch_pdl() may be scheduled while its predecessor on the stream is still
// draining; it must call pdl_wait() before it reads anything the
// predecessor writes (work before that -- loads of inputs produced earlier,
// shared-memory setup -- overlaps the predecessor's tail).  A predecessor
// calls pdl_trigger() once its remaining CTAs no longer need to be
// scheduled ahead of the dependent's.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Round half away from zero, exactly (compression.py:61-63 computes
// copysign(floor(|v| + 0.5), v) in float64, which is exact for float32 v).
// v - trunc(v) is exact in float32, so no double rounding can occur.
__device__ __forceinline__ float round_half_away(float v) {
  float t = truncf(v);
  if (fabsf(v - t) >= 0.5f) t += copysignf(1.0f, v);
  return t;
}

// Saturating fixed-point code; NaN -> 0 as the reference's cast yields.
__device__ __forceinline__ int fixed_code(float x, float scale, float lo, float hi) {
  float v = x * scale;                 // exact: scale is a power of two
  if (v != v) return 0;
  float r = round_half_away(v);
  r = fminf(fmaxf(r, lo), hi);
  return static_cast<int>(r);
}

// ---- GEMM operand planes written by the producing kernel.  x = hi + mid +
// lo exactly, each term the round-to-nearest bf16 of what is left (the split
// of `sf_split3_bf16`, gemm_tc.cu, bit for bit); planes [3][rows][cols] with
// plane stride `plane` elements, so the next product reads them instead of
// running a split pass over its A operand.
__device__ __forceinline__ uint32_t bf16x2_rn(float lo_elem, float hi_elem) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}

__device__ __forceinline__ void split_pair3(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
  h = bf16x2_rn(x0, x1);
  float r0 = x0 - __uint_as_float(h << 16), r1 = x1 - __uint_as_float(h & 0xFFFF0000u);   // exact
  m = bf16x2_rn(r0, r1);
  r0 -= __uint_as_float(m << 16);                                                          // exact
  r1 -= __uint_as_float(m & 0xFFFF0000u);
  l = bf16x2_rn(r0, r1);
}

// four consecutive values at element offset o (o % 4 == 0)
__device__ __forceinline__ void planes_store4(float4 v, __nv_bfloat16* __restrict__ planes, int64_t plane,
                                              int64_t o) {
  uint32_t h0, m0, l0, h1, m1, l1;
  split_pair3(v.x, v.y, h0, m0, l0);
  split_pair3(v.z, v.w, h1, m1, l1);
  *reinterpret_cast<uint2*>(planes + o) = make_uint2(h0, h1);
  *reinterpret_cast<uint2*>(planes + plane + o) = make_uint2(m0, m1);
  *reinterpret_cast<uint2*>(planes + 2 * plane + o) = make_uint2(l0, l1);
}

// two consecutive values at element offset o (o % 2 == 0)
__device__ __forceinline__ void planes_store2(float a, float b, __nv_bfloat16* __restrict__ planes, int64_t plane,
                                              int64_t o) {
  uint32_t h, m, l;
  split_pair3(a, b, h, m, l);
  *reinterpret_cast<uint32_t*>(planes + o) = h;
  *reinterpret_cast<uint32_t*>(planes + plane + o) = m;
  *reinterpret_cast<uint32_t*>(planes + 2 * plane + o) = l;
}

// one value at element offset o
__device__ __forceinline__ void planes_store1(float a, __nv_bfloat16* __restrict__ planes, int64_t plane,
                                              int64_t o) {
  const __nv_bfloat16 h = __float2bfloat16_rn(a);
  const float r = a - __bfloat162float(h);
  const __nv_bfloat16 m = __float2bfloat16_rn(r);
  planes[o] = h;
  planes[plane + o] = m;
  planes[2 * plane + o] = __float2bfloat16_rn(r - __bfloat162float(m));
}


// ---- f16x3 operand planes: x = hi + 2^-11 lo with hi = RN_f16(x),
// lo = RN_f16((x - hi) * 2^11) (x - hi exact, |x - hi| <= 2^-11 |x|): two
// fp16 planes [2][rows][cols], the forward products' operands
// (sf_split2_f16, gemm_tc.cu, bit for bit).
__device__ __forceinline__ uint32_t f16x2_rn(float lo_elem, float hi_elem) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}

__device__ __forceinline__ float f16_lo_f32(uint32_t h) { return __half2float(__ushort_as_half(static_cast<unsigned short>(h & 0xFFFFu))); }
__device__ __forceinline__ float f16_hi_f32(uint32_t h) { return __half2float(__ushort_as_half(static_cast<unsigned short>(h >> 16))); }

__device__ __forceinline__ void split_pair2h(float x0, float x1, uint32_t& h, uint32_t& l) {
  h = f16x2_rn(x0, x1);
  l = f16x2_rn((x0 - f16_lo_f32(h)) * 2048.0f, (x1 - f16_hi_f32(h)) * 2048.0f);
}

__device__ __forceinline__ void planes_store4h(float4 v, __half* __restrict__ planes, int64_t plane, int64_t o) {
  uint32_t h0, l0, h1, l1;
  split_pair2h(v.x, v.y, h0, l0);
  split_pair2h(v.z, v.w, h1, l1);
  *reinterpret_cast<uint2*>(planes + o) = make_uint2(h0, h1);
  *reinterpret_cast<uint2*>(planes + plane + o) = make_uint2(l0, l1);
}

__device__ __forceinline__ void planes_store2h(float a, float b, __half* __restrict__ planes, int64_t plane,
                                               int64_t o) {
  uint32_t h, l;
  split_pair2h(a, b, h, l);
  *reinterpret_cast<uint32_t*>(planes + o) = h;
  *reinterpret_cast<uint32_t*>(planes + plane + o) = l;
}

__device__ __forceinline__ void planes_store1h(float a, __half* __restrict__ planes, int64_t plane, int64_t o) {
  const __half h = __float2half_rn(a);
  planes[o] = h;
  planes[plane + o] = __float2half_rn((a - __half2float(h)) * 2048.0f);
}

// Row scale of the row-scaled fp16 planes (pf 2): e = 15 - (exponent of
// amax) so that amax 2^e lies in [2^14, 2^15); returns 2^e (1 for a zero or
// non-finite row).  The product's row is multiplied by 2^-e (exact).
__device__ __forceinline__ float row_scale_exp(float amax, int& e) {
  e = 0;
  if (amax > 0.0f && amax <= 3.0e38f) {
    int ex;
    frexpf(amax, &ex);                     // amax = f 2^ex, f in [0.5, 1)
    e = 15 - ex;
    e = e < -126 ? -126 : (e > 126 ? 126 : e);
  }
  return __int_as_float((127 + e) << 23);
}

__device__ __forceinline__ float pow2i(int e) { return __int_as_float((127 + e) << 23); }   // |e| <= 126

__device__ __forceinline__ float max4abs(float4 v) {
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

// where a producer writes the next product's A-operand planes
struct PlanesOut {
  __nv_bfloat16* p;     // planes base, nullptr: none
  int pf;               // 0 three bf16 planes, 1 two fp16 planes, 2 two fp16 planes scaled per row
  float* rsc;           // pf 2: 2^-e per row
};

// producer planes in either form: pf 0 = three bf16 planes (sf_split3_bf16),
// pf 1 = two fp16 planes (sf_split2_f16); `planes` typed as the bf16 form
__device__ __forceinline__ void planes_store4f(float4 v, __nv_bfloat16* planes, int64_t plane, int64_t o, int pf) {
  if (pf) planes_store4h(v, reinterpret_cast<__half*>(planes), plane, o);
  else planes_store4(v, planes, plane, o);
}
__device__ __forceinline__ void planes_store2f(float a, float b, __nv_bfloat16* planes, int64_t plane, int64_t o,
                                               int pf) {
  if (pf) planes_store2h(a, b, reinterpret_cast<__half*>(planes), plane, o);
  else planes_store2(a, b, planes, plane, o);
}
__device__ __forceinline__ void planes_store1f(float a, __nv_bfloat16* planes, int64_t plane, int64_t o, int pf) {
  if (pf) planes_store1h(a, reinterpret_cast<__half*>(planes), plane, o);
  else planes_store1(a, planes, plane, o);
}

}  // namespace sf
