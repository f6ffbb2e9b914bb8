// LayerNorm forward/backward owning the semi-static x~ cache, and the
// softmax forward/backward owning the 8-bit probability cache.
//
// Reference: layernorm (tensor.py:447-494), softmax (:413-444) with
// _save_maybe_quant8 (:280-283), scale (:583-593).
//
// One warp per row; a row lives in registers (float4 per lane, VPL of them),
// so x is read once and y (+ x~) written once.  The frozen+pruned backward
// consumes the pruned x~ (values, ascending flat indices) directly: a
// row-pointer pass over the k indices gives each row its slice, which the
// warp scatters into a shared-memory row, so the dense restore (K7) never
// touches HBM.
// Column sums for dgamma/dbeta are deterministic: per-CTA partials in a
// fixed order, then one reduction kernel.
#include "common.cuh"

namespace sf {

constexpr int kLT = 256;          // 8 warps per CTA
constexpr int kWarps = kLT / 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// RES: the row is r + (x + bias) (the residual add after a projection whose
// bias was left out of the GEMM, rounded in the reference's order); the sum
// is written to `sum` when non-null (pre-norm keeps the residual stream).
template <int VPL, bool RES>
__global__ void __launch_bounds__(kLT, 4) k_ln_fwd(const float* __restrict__ x,
                                                const float* __restrict__ gamma,
                                                const float* __restrict__ beta,
                                                float* __restrict__ y, float* __restrict__ xt,
                                                float* __restrict__ rstd, int64_t rows, int H,
                                                float eps, const float* __restrict__ res,
                                                const float* __restrict__ bias,
                                                float* __restrict__ sum,
                                                __nv_bfloat16* __restrict__ yp = nullptr, int pf = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t plane = rows * H;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const float invH = 1.0f / static_cast<float>(H);
  (void)invH;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float4* xr = reinterpret_cast<const float4*>(x + r * H);
    float4 v[VPL];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      int c = lane + 32 * j;
      v[j] = (4 * c < H) ? __ldg(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (RES && 4 * c < H) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bias) + c);
        const float4 rr = __ldg(reinterpret_cast<const float4*>(res + r * H) + c);
        v[j] = make_float4(__fadd_rn(rr.x, __fadd_rn(v[j].x, bb.x)), __fadd_rn(rr.y, __fadd_rn(v[j].y, bb.y)),
                           __fadd_rn(rr.z, __fadd_rn(v[j].z, bb.z)), __fadd_rn(rr.w, __fadd_rn(v[j].w, bb.w)));
        if (sum) reinterpret_cast<float4*>(sum + r * H)[c] = v[j];
      }
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    const float mean = __fdiv_rn(warp_sum(s), static_cast<float>(H));
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      int c = lane + 32 * j;
      if (4 * c < H) {
        float a = v[j].x - mean, b = v[j].y - mean, cc = v[j].z - mean, d = v[j].w - mean;
        q += (__fmul_rn(a, a) + __fmul_rn(b, b)) + (__fmul_rn(cc, cc) + __fmul_rn(d, d));
      }
    }
    const float var = __fdiv_rn(warp_sum(q), static_cast<float>(H));
    const float rs = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, eps)));
    if (lane == 0) rstd[r] = rs;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      int c = lane + 32 * j;
      if (4 * c < H) {
        float4 g = __ldg(reinterpret_cast<const float4*>(gamma) + c);
        float4 b = __ldg(reinterpret_cast<const float4*>(beta) + c);
        float4 t = make_float4(__fmul_rn(v[j].x - mean, rs), __fmul_rn(v[j].y - mean, rs),
                               __fmul_rn(v[j].z - mean, rs), __fmul_rn(v[j].w - mean, rs));
        if (xt) reinterpret_cast<float4*>(xt + r * H)[c] = t;
        const float4 yv =
            make_float4(__fadd_rn(__fmul_rn(t.x, g.x), b.x), __fadd_rn(__fmul_rn(t.y, g.y), b.y),
                        __fadd_rn(__fmul_rn(t.z, g.z), b.z), __fadd_rn(__fmul_rn(t.w, g.w), b.w));
        reinterpret_cast<float4*>(y + r * H)[c] = yv;
        if (yp) planes_store4f(yv, yp, plane, r * H + 4 * c, pf);
      }
    }
  }
}

// row_ptr[r] = first j with indices[j] >= r*H (CSR row pointers of the
// pruned x~, indices ascending); row_ptr[rows] = k.
__global__ void k_rowptr(const int32_t* __restrict__ idx, int64_t k, int H, int64_t rows,
                         int32_t* __restrict__ row_ptr) {
  // indices < 2^31 (int32), so 32-bit unsigned division suffices
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const uint32_t h = static_cast<uint32_t>(H);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j <= k;
       j += stride) {
    const int64_t r = j < k ? static_cast<int64_t>(static_cast<uint32_t>(__ldg(idx + j)) / h) : rows;
    const int64_t rp =
        j > 0 ? static_cast<int64_t>(static_cast<uint32_t>(__ldg(idx + j - 1)) / h) : -1;
    for (int64_t q = rp + 1; q <= r; ++q) row_ptr[q] = static_cast<int32_t>(j);
  }
}

// Backward without dgamma/dbeta (the frozen LayerNorm: dense x~ when the
// prune codec is off, pruned x~ otherwise).  Two sweeps over the row: the
// first accumulates the row sums, the second recomputes gg from g and x~
// re-read through L1 (the row was just loaded) and writes dx, so nothing
// row-sized stays in registers and occupancy stays high.
// Row-scaled fp16 planes of one row held by a warp (VPL float4 per lane):
// the row's maximum, then x 2^e split into the two planes, 2^-e per row.
template <int VPL>
__device__ __forceinline__ void ln_row_planes(const float4 (&o)[VPL], float mx, const PlanesOut& po, int64_t plane,
                                              int64_t r, int H, int lane) {
#pragma unroll
  for (int k = 16; k; k >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, k));
  int e;
  const float sc = row_scale_exp(mx, e);
  if (lane == 0) po.rsc[r] = pow2i(-e);
  __half* hp = reinterpret_cast<__half*>(po.p);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int c = lane + 32 * j;
    if (4 * c < H)
      planes_store4h(make_float4(o[j].x * sc, o[j].y * sc, o[j].z * sc, o[j].w * sc), hp, plane, r * H + 4 * c);
  }
}

template <int VPL, bool SPARSE>
__global__ void __launch_bounds__(kLT) k_ln_bwd_lean(const float* __restrict__ g,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ xt,
                                                     const float* __restrict__ values,
                                                     const int32_t* __restrict__ indices,
                                                     const int32_t* __restrict__ row_ptr,
                                                     const float* __restrict__ rstd,
                                                     float* __restrict__ dx, int64_t rows, int H,
                                                     PlanesOut po = {}) {
  const int64_t plane = rows * H;
  // The row of g stays in registers (one HBM read, every load issued before
  // any arithmetic); x~ comes from a shared-memory row (sparse: zeroed, then
  // the kept values scattered into it) or is re-read through L1.
  // gg = gamma * g * rs / H elementwise as numpy rounds it (tensor.py:485),
  // computed once per element and kept in registers for the second sweep.
  extern __shared__ float sh_rows[];      // kWarps * H floats (sparse rows)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float* myrow = sh_rows + wid * H;
  const float fH = static_cast<float>(H);
  const float4* gm4 = reinterpret_cast<const float4*>(gamma);
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float4* g4 = reinterpret_cast<const float4*>(g + r * H);
    float4 gv[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      gv[j] = 4 * c < H ? ld_stream(g4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float rs = __ldg(rstd + r);
    const float4* t4 = SPARSE ? reinterpret_cast<const float4*>(myrow)
                              : reinterpret_cast<const float4*>(xt + r * H);
    if (SPARSE) {
      const int64_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);   // int32 CSR
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int c = lane + 32 * j;
        if (4 * c < H) reinterpret_cast<float4*>(myrow)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncwarp();
      // scatter the row's kept (index, value) pairs: the loads of several
      // iterations are issued together (rows can hold up to H pairs -- a
      // serial loop would pay one memory latency per 32 of them)
      const int32_t rH = static_cast<int32_t>(r * H);
      int32_t j = static_cast<int32_t>(a) + lane;
      const int32_t jb = static_cast<int32_t>(b);
      for (; j + 96 < jb; j += 128) {
        const int32_t i0 = __ldg(indices + j), i1 = __ldg(indices + j + 32);
        const int32_t i2 = __ldg(indices + j + 64), i3 = __ldg(indices + j + 96);
        const float v0 = __ldg(values + j), v1 = __ldg(values + j + 32);
        const float v2 = __ldg(values + j + 64), v3 = __ldg(values + j + 96);
        myrow[i0 - rH] = v0;
        myrow[i1 - rH] = v1;
        myrow[i2 - rH] = v2;
        myrow[i3 - rH] = v3;
      }
      for (; j < jb; j += 32) myrow[__ldg(indices + j) - rH] = __ldg(values + j);
      __syncwarp();
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) {
        const float4 gm = __ldg(gm4 + c);
        const float4 tv = SPARSE ? t4[c] : __ldg(t4 + c);
        gv[j].x = __fdiv_rn(__fmul_rn(__fmul_rn(gm.x, gv[j].x), rs), fH);   // gg
        gv[j].y = __fdiv_rn(__fmul_rn(__fmul_rn(gm.y, gv[j].y), rs), fH);
        gv[j].z = __fdiv_rn(__fmul_rn(__fmul_rn(gm.z, gv[j].z), rs), fH);
        gv[j].w = __fdiv_rn(__fmul_rn(__fmul_rn(gm.w, gv[j].w), rs), fH);
        s1 += (gv[j].x + gv[j].y) + (gv[j].z + gv[j].w);
        s2 += (__fmul_rn(gv[j].x, tv.x) + __fmul_rn(gv[j].y, tv.y)) +
              (__fmul_rn(gv[j].z, tv.z) + __fmul_rn(gv[j].w, tv.w));
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) {
        const float4 tv = SPARSE ? t4[c] : __ldg(t4 + c);
        float4 o;
        o.x = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].x), s1), __fmul_rn(tv.x, s2));
        o.y = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].y), s1), __fmul_rn(tv.y, s2));
        o.z = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].z), s1), __fmul_rn(tv.z, s2));
        o.w = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].w), s1), __fmul_rn(tv.w, s2));
        reinterpret_cast<float4*>(dx + r * H)[c] = o;
        gv[j] = o;
        mx = fmaxf(mx, max4abs(o));
        if (po.p && po.pf != 2) planes_store4f(o, po.p, plane, r * H + 4 * c, po.pf);
      }
    }
    if (po.p && po.pf == 2) ln_row_planes<VPL>(gv, mx, po, plane, r, H, lane);
    if (SPARSE) __syncwarp();
  }
}

template <int VPL, bool SPARSE, bool COLS>
__global__ void __launch_bounds__(kLT, 3) k_ln_bwd(const float* __restrict__ g,
                                                   const float* __restrict__ gamma,
                                                   const float* __restrict__ xt,
                                                   const float* __restrict__ values,
                                                   const int32_t* __restrict__ indices,
                                                   const int32_t* __restrict__ row_ptr,
                                                   const float* __restrict__ rstd,
                                                   float* __restrict__ dx, float* __restrict__ part,
                                                   int64_t rows, int H,
                                                   PlanesOut po = {}) {
  const int64_t plane = rows * H;
  pdl_trigger();                          // the column finish may launch and wait
  // [SPARSE: kWarps * H floats, the sparse rows] [COLS: kWarps * 2H floats, each
  // warp's column sums of g x~ and g, in its rows' order].  The column sums
  // live in shared memory, not registers: 3 CTAs per SM instead of 2.
  extern __shared__ float sh_rows[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  float* myrow = sh_rows + wid * H;
  float* acc_s = sh_rows + (SPARSE ? kWarps * H : 0);
  float4* acc_g4 = reinterpret_cast<float4*>(acc_s + wid * 2 * H);
  float4* acc_b4 = reinterpret_cast<float4*>(acc_s + wid * 2 * H + H);
  if (COLS) {
    for (int c = lane; c < H / 2; c += 32) acc_g4[c] = make_float4(0.f, 0.f, 0.f, 0.f);   // both halves
    __syncwarp();
  }
  const float fH = static_cast<float>(H);

  for (int64_t r = warp0; r < rows; r += nwarps) {
    float4 gv[VPL], tv[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) gv[j] = ld_stream(reinterpret_cast<const float4*>(g + r * H) + c);
    }
    if (SPARSE) {
      for (int c = lane; c < H / 4; c += 32)
        reinterpret_cast<float4*>(myrow)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
      const int64_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);   // int32 CSR
      // scatter the row's kept (index, value) pairs: the loads of several
      // iterations are issued together (rows can hold up to H pairs -- a
      // serial loop would pay one memory latency per 32 of them)
      const int32_t rH = static_cast<int32_t>(r * H);
      int32_t j = static_cast<int32_t>(a) + lane;
      const int32_t jb = static_cast<int32_t>(b);
      for (; j + 96 < jb; j += 128) {
        const int32_t i0 = __ldg(indices + j), i1 = __ldg(indices + j + 32);
        const int32_t i2 = __ldg(indices + j + 64), i3 = __ldg(indices + j + 96);
        const float v0 = __ldg(values + j), v1 = __ldg(values + j + 32);
        const float v2 = __ldg(values + j + 64), v3 = __ldg(values + j + 96);
        myrow[i0 - rH] = v0;
        myrow[i1 - rH] = v1;
        myrow[i2 - rH] = v2;
        myrow[i3 - rH] = v3;
      }
      for (; j < jb; j += 32) myrow[__ldg(indices + j) - rH] = __ldg(values + j);
      __syncwarp();
    }
    const float rs = __ldg(rstd + r);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) {
        const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma) + c);
        tv[j] = SPARSE ? reinterpret_cast<const float4*>(myrow)[c]
                       : ld_stream(reinterpret_cast<const float4*>(xt + r * H) + c);
        if (COLS) {                                   // this lane's columns: no other lane touches them
          float4 ag = acc_g4[c], ab = acc_b4[c];
          ag.x += tv[j].x * gv[j].x;
          ag.y += tv[j].y * gv[j].y;
          ag.z += tv[j].z * gv[j].z;
          ag.w += tv[j].w * gv[j].w;
          ab.x += gv[j].x;
          ab.y += gv[j].y;
          ab.z += gv[j].z;
          ab.w += gv[j].w;
          acc_g4[c] = ag;
          acc_b4[c] = ab;
        }
        // gg = gamma * g * rs / H  (left to right, as numpy evaluates it); gv <- gg
        gv[j] = make_float4(__fdiv_rn(__fmul_rn(__fmul_rn(gm.x, gv[j].x), rs), fH),
                            __fdiv_rn(__fmul_rn(__fmul_rn(gm.y, gv[j].y), rs), fH),
                            __fdiv_rn(__fmul_rn(__fmul_rn(gm.z, gv[j].z), rs), fH),
                            __fdiv_rn(__fmul_rn(__fmul_rn(gm.w, gv[j].w), rs), fH));
        s1 += (gv[j].x + gv[j].y) + (gv[j].z + gv[j].w);
        s2 += (__fmul_rn(gv[j].x, tv[j].x) + __fmul_rn(gv[j].y, tv[j].y)) +
              (__fmul_rn(gv[j].z, tv[j].z) + __fmul_rn(gv[j].w, tv[j].w));
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int c = lane + 32 * j;
      if (4 * c < H) {
        float4 o;
        o.x = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].x), s1), __fmul_rn(tv[j].x, s2));
        o.y = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].y), s1), __fmul_rn(tv[j].y, s2));
        o.z = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].z), s1), __fmul_rn(tv[j].z, s2));
        o.w = __fsub_rn(__fsub_rn(__fmul_rn(fH, gv[j].w), s1), __fmul_rn(tv[j].w, s2));
        reinterpret_cast<float4*>(dx + r * H)[c] = o;
        gv[j] = o;
        mx = fmaxf(mx, max4abs(o));
        if (po.p && po.pf != 2) planes_store4f(o, po.p, plane, r * H + 4 * c, po.pf);
      }
    }
    if (po.p && po.pf == 2) ln_row_planes<VPL>(gv, mx, po, plane, r, H, lane);
    if (SPARSE) __syncwarp();
  }
  if (!COLS) return;
  // CTA reduction of the per-warp column sums, fixed order -> deterministic
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass)
    for (int c = threadIdx.x; c < H; c += blockDim.x) {
      float t = 0.f;
      for (int w = 0; w < kWarps; ++w) t += acc_s[w * 2 * H + pass * H + c];
      part[(static_cast<int64_t>(blockIdx.x) * 2 + pass) * H + c] = t;
    }
}

// dgamma / dbeta = column sums of the per-CTA partials.  One CTA per 32
// columns: lane = column, the 8 warps stride the partial rows and their
// sums combine in shared memory in a fixed order (deterministic), so the
// 2 x nparts loads per column are spread over 8 warps x H/32 CTAs instead
// of one serial loop per thread.
constexpr int kCF = 256;
__global__ void __launch_bounds__(kCF) k_col_finish(const float* __restrict__ part, int nparts, int H,
                                                   float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ float sa[kCF / 32][32], sb[kCF / 32][32];
  pdl_wait();                                  // the partials of the backward kernel
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float a = 0.f, b = 0.f;
  if (c < H) {
#pragma unroll 4
    for (int p = w; p < nparts; p += kCF / 32) {
      a += __ldg(part + (static_cast<int64_t>(p) * 2) * H + c);
      b += __ldg(part + (static_cast<int64_t>(p) * 2 + 1) * H + c);
    }
  }
  sa[w][lane] = a;
  sb[w][lane] = b;
  __syncthreads();
  if (w == 0 && c < H) {
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int q = 0; q < kCF / 32; ++q) {
      ta += sa[q][lane];
      tb += sb[q][lane];
    }
    if (dgamma) dgamma[c] = ta;
    if (dbeta) dbeta[c] = tb;
  }
}

// ---------------------------------------------------------------- softmax

template <int MAXI>
__global__ void __launch_bounds__(kLT) k_softmax_fwd_q8(const float* __restrict__ s,
                                                        float* __restrict__ probs,
                                                        uint8_t* __restrict__ codes, int64_t rows,
                                                        int W, float scale, float qscale, float lo,
                                                        float hi) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float* sr = s + r * W;
    float v[MAXI];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      int c = lane + 32 * i;
      v[i] = c < W ? __fmul_rn(__ldg(sr + c), scale) : -INFINITY;   // scale op, tensor.py:583
      m = fmaxf(m, v[i]);
    }
    m = warp_max(m);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      int c = lane + 32 * i;
      v[i] = c < W ? expf(v[i] - m) : 0.f;
      sum += v[i];
    }
    sum = warp_sum(sum);
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      int c = lane + 32 * i;
      if (c < W) {
        float p = __fdiv_rn(v[i], sum);
        if (probs) probs[r * W + c] = p;
        codes[r * W + c] = static_cast<uint8_t>(fixed_code(p, qscale, lo, hi) & 0xFF);
      }
    }
  }
}

template <int MAXI, bool SIGNED>
__global__ void __launch_bounds__(kLT) k_softmax_bwd_q8(const float* __restrict__ g,
                                                        const uint8_t* __restrict__ codes,
                                                        float* __restrict__ ds, int64_t rows,
                                                        int W, float inv, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    float p[MAXI], gv[MAXI];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      int c = lane + 32 * i;
      if (c < W) {
        uint32_t b = codes[r * W + c];
        int code = SIGNED ? static_cast<int>(static_cast<int8_t>(b)) : static_cast<int>(b);
        p[i] = static_cast<float>(code) * inv;
        gv[i] = __ldg(g + r * W + c);
        dot += __fmul_rn(gv[i], p[i]);
      } else {
        p[i] = gv[i] = 0.f;
      }
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int i = 0; i < MAXI; ++i) {
      int c = lane + 32 * i;
      if (c < W) ds[r * W + c] = __fmul_rn(__fmul_rn(p[i], __fsub_rn(gv[i], dot)), scale);
    }
  }
}

// float4 path (W % 4 == 0): lane owns float4 c = lane + 32 j of the row;
// one 16 B load, one 16 B probs store and one 4 B codes store per float4.
template <int MV>
__global__ void __launch_bounds__(kLT) k_softmax_fwd_q8_v4(const float* __restrict__ s,
                                                           float* __restrict__ probs,
                                                           uint8_t* __restrict__ codes,
                                                           int64_t rows, int W4, float scale,
                                                           float qscale, float lo, float hi) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float4* sr = reinterpret_cast<const float4*>(s) + r * W4;
    float4 v[MV];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < MV; ++j) {
      const int c = lane + 32 * j;
      if (c < W4) {
        float4 t = ld_stream(sr + c);
        v[j] = make_float4(__fmul_rn(t.x, scale), __fmul_rn(t.y, scale), __fmul_rn(t.z, scale),
                           __fmul_rn(t.w, scale));
        m = fmaxf(m, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
      }
    }
    m = warp_max(m);
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < MV; ++j) {
      const int c = lane + 32 * j;
      if (c < W4) {
        v[j] = make_float4(expf(v[j].x - m), expf(v[j].y - m), expf(v[j].z - m), expf(v[j].w - m));
        sum += (v[j].x + v[j].y) + (v[j].z + v[j].w);
      }
    }
    sum = warp_sum(sum);
#pragma unroll
    for (int j = 0; j < MV; ++j) {
      const int c = lane + 32 * j;
      if (c < W4) {
        float4 p = make_float4(__fdiv_rn(v[j].x, sum), __fdiv_rn(v[j].y, sum),
                               __fdiv_rn(v[j].z, sum), __fdiv_rn(v[j].w, sum));
        if (probs) reinterpret_cast<float4*>(probs)[r * W4 + c] = p;
        const uint32_t w = (static_cast<uint32_t>(fixed_code(p.x, qscale, lo, hi)) & 0xFFu) |
                           ((static_cast<uint32_t>(fixed_code(p.y, qscale, lo, hi)) & 0xFFu) << 8) |
                           ((static_cast<uint32_t>(fixed_code(p.z, qscale, lo, hi)) & 0xFFu) << 16) |
                           ((static_cast<uint32_t>(fixed_code(p.w, qscale, lo, hi)) & 0xFFu) << 24);
        reinterpret_cast<uint32_t*>(codes)[r * W4 + c] = w;
      }
    }
  }
}

template <bool SIGNED>
__device__ __forceinline__ float dec8(uint32_t b, float inv) {
  return static_cast<float>(SIGNED ? static_cast<int>(static_cast<int8_t>(b & 0xFF))
                                   : static_cast<int>(b & 0xFF)) * inv;
}

template <int MV, bool SIGNED>
__global__ void __launch_bounds__(kLT) k_softmax_bwd_q8_v4(const float* __restrict__ g,
                                                           const uint8_t* __restrict__ codes,
                                                           float* __restrict__ ds, int64_t rows,
                                                           int W4, float inv, float scale) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    float4 p[MV], gv[MV];
    float dot = 0.f;
#pragma unroll
    for (int j = 0; j < MV; ++j) {
      const int c = lane + 32 * j;
      if (c < W4) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(codes) + r * W4 + c);
        p[j] = make_float4(dec8<SIGNED>(w, inv), dec8<SIGNED>(w >> 8, inv),
                           dec8<SIGNED>(w >> 16, inv), dec8<SIGNED>(w >> 24, inv));
        gv[j] = ld_stream(reinterpret_cast<const float4*>(g) + r * W4 + c);
        dot += (__fmul_rn(gv[j].x, p[j].x) + __fmul_rn(gv[j].y, p[j].y)) +
               (__fmul_rn(gv[j].z, p[j].z) + __fmul_rn(gv[j].w, p[j].w));
      }
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int j = 0; j < MV; ++j) {
      const int c = lane + 32 * j;
      if (c < W4)
        reinterpret_cast<float4*>(ds)[r * W4 + c] =
            make_float4(__fmul_rn(__fmul_rn(p[j].x, __fsub_rn(gv[j].x, dot)), scale),
                        __fmul_rn(__fmul_rn(p[j].y, __fsub_rn(gv[j].y, dot)), scale),
                        __fmul_rn(__fmul_rn(p[j].z, __fsub_rn(gv[j].z, dot)), scale),
                        __fmul_rn(__fmul_rn(p[j].w, __fsub_rn(gv[j].w, dot)), scale));
    }
  }
}

template <int VPL>
int launch_ln_fwd(const float* x, const float* gamma, const float* beta, float* y, float* xt,
                  float* rstd, int64_t rows, int H, float eps, cudaStream_t s,
                  const float* res = nullptr, const float* bias = nullptr, float* sum = nullptr,
                  __nv_bfloat16* yp = nullptr, int pf = 0) {
  unsigned grid = grid_for(rows * 32, kLT, 8);
  if (res)
    k_ln_fwd<VPL, true><<<grid, kLT, 0, s>>>(x, gamma, beta, y, xt, rstd, rows, H, eps, res, bias, sum, yp, pf);
  else
    k_ln_fwd<VPL, false><<<grid, kLT, 0, s>>>(x, gamma, beta, y, xt, rstd, rows, H, eps, nullptr,
                                              nullptr, nullptr, yp, pf);
  return check_launch();
}

inline unsigned ln_bwd_grid(int64_t rows) { return grid_for(rows * 32, kLT, 3); }

inline size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

template <int VPL, bool SPARSE, bool COLS>
void launch_ln_bwd_kernel(unsigned grid, size_t smem, cudaStream_t s, const float* g,
                          const float* gamma, const float* xt, const float* values,
                          const int32_t* indices, const int32_t* row_ptr, const float* rstd,
                          float* dx, float* part, int64_t rows, int H, PlanesOut po) {
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_ln_bwd<VPL, SPARSE, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  k_ln_bwd<VPL, SPARSE, COLS><<<grid, kLT, smem, s>>>(g, gamma, xt, values, indices, row_ptr, rstd,
                                                      dx, part, rows, H, po);
}

template <int VPL>
int launch_ln_bwd(const float* g, const float* gamma, const float* xt, const float* values,
                  const int32_t* indices, int64_t k, const int32_t* row_ptr_in, const float* rstd,
                  float* dx, float* dgamma, float* dbeta, int64_t rows, int H, void* ws,
                  cudaStream_t s, PlanesOut po = {}) {
  const unsigned grid = ln_bwd_grid(rows);
  const bool cols = dgamma || dbeta;
  const size_t smem = static_cast<size_t>(kWarps) * H * sizeof(float);
  char* w = static_cast<char*>(ws);
  float* part = reinterpret_cast<float*>(w);
  int32_t* row_ptr = reinterpret_cast<int32_t*>(w + a256(static_cast<size_t>(grid) * 2 * H * 4));
  if (!xt) {
    if (row_ptr_in)
      row_ptr = const_cast<int32_t*>(row_ptr_in);     // CSR produced by the prune pass
    else
      k_rowptr<<<grid_for(k + 1, 256, 4), 256, 0, s>>>(indices, k, H, rows, row_ptr);
    const unsigned lgrid = grid_for(rows * 32, kLT, 8);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_ln_bwd_lean<VPL, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
    k_ln_bwd_lean<VPL, true><<<lgrid, kLT, smem, s>>>(g, gamma, nullptr, values, indices, row_ptr,
                                                      rstd, dx, rows, H, po);
  } else if (cols) {
    launch_ln_bwd_kernel<VPL, false, true>(grid, 2 * smem, s, g, gamma, xt, nullptr, nullptr, nullptr,
                                           rstd, dx, part, rows, H, po);
    launch_pdl(k_col_finish, dim3((H + 31) / 32), dim3(kCF), 0, s, static_cast<const float*>(part), grid, H,
               dgamma, dbeta);
  } else {
    k_ln_bwd_lean<VPL, false><<<grid_for(rows * 32, kLT, 8), kLT, 0, s>>>(
        g, gamma, xt, nullptr, nullptr, nullptr, rstd, dx, rows, H, po);
  }
  return check_launch();
}

template <int MAXI>
int launch_softmax_fwd(const float* sc, float* probs, uint8_t* codes, int64_t rows, int W,
                       float scale, float qs, float lo, float hi, cudaStream_t s) {
  k_softmax_fwd_q8<MAXI><<<grid_for(rows * 32, kLT, 8), kLT, 0, s>>>(sc, probs, codes, rows, W,
                                                                      scale, qs, lo, hi);
  return check_launch();
}

template <int MAXI>
int launch_softmax_bwd(const float* g, const uint8_t* codes, float* ds, int64_t rows, int W,
                       float inv, bool sgn, float scale, cudaStream_t s) {
  unsigned grid = grid_for(rows * 32, kLT, 8);
  if (sgn)
    k_softmax_bwd_q8<MAXI, true><<<grid, kLT, 0, s>>>(g, codes, ds, rows, W, inv, scale);
  else
    k_softmax_bwd_q8<MAXI, false><<<grid, kLT, 0, s>>>(g, codes, ds, rows, W, inv, scale);
  return check_launch();
}

}  // namespace sf

using namespace sf;

extern "C" {

int sf_layernorm_fwd_p(const float* x, const float* gamma, const float* beta, float* y,
                       float* xtilde, float* rstd, int64_t rows, int64_t H, float eps, void* y_planes,
                       void* stream) {
  return sf_layernorm_fwd_pf(x, gamma, beta, y, xtilde, rstd, rows, H, eps, y_planes, 0, stream);
}

int sf_layernorm_fwd_pf(const float* x, const float* gamma, const float* beta, float* y,
                        float* xtilde, float* rstd, int64_t rows, int64_t H, float eps, void* y_planes,
                        int planes_format, void* stream) {
  if (planes_format < 0 || planes_format > 1) return SF_EINVAL;
  if (rows < 0 || H < 4 || H % 4 || H > 1024 || !x || !gamma || !beta || !y || !rstd)
    return SF_EINVAL;
  if (!aligned16(x) || !aligned16(y) || !aligned16(gamma) || !aligned16(beta) ||
      (xtilde && !aligned16(xtilde)) || (reinterpret_cast<uintptr_t>(y_planes) & 7u))
    return SF_EINVAL;
  if (rows == 0) return SF_OK;
  cudaStream_t s = as_stream(stream);
  const int h = static_cast<int>(H);
  __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(y_planes);
#define SF_LNF(V) launch_ln_fwd<V>(x, gamma, beta, y, xtilde, rstd, rows, h, eps, s, nullptr, nullptr, nullptr, yp, \
                                   planes_format)
  if (H <= 128) return SF_LNF(1);
  if (H <= 256) return SF_LNF(2);
  if (H <= 512) return SF_LNF(4);
  if (H <= 768) return SF_LNF(6);
  return SF_LNF(8);
#undef SF_LNF
}

int sf_layernorm_fwd(const float* x, const float* gamma, const float* beta, float* y,
                     float* xtilde, float* rstd, int64_t rows, int64_t H, float eps,
                     void* stream) {
  return sf_layernorm_fwd_p(x, gamma, beta, y, xtilde, rstd, rows, H, eps, nullptr, stream);
}

int sf_layernorm_fwd_residual_p(const float* res, const float* x, const float* bias, const float* gamma,
                                const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                                int64_t rows, int64_t H, float eps, void* y_planes, void* stream) {
  return sf_layernorm_fwd_residual_pf(res, x, bias, gamma, beta, y, sum, xtilde, rstd, rows, H, eps, y_planes, 0,
                                      stream);
}

int sf_layernorm_fwd_residual_pf(const float* res, const float* x, const float* bias, const float* gamma,
                                 const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                                 int64_t rows, int64_t H, float eps, void* y_planes, int planes_format,
                                 void* stream) {
  if (planes_format < 0 || planes_format > 1) return SF_EINVAL;
  if (rows < 0 || H < 4 || H % 4 || H > 1024 || !res || !x || !bias || !gamma || !beta || !y || !rstd)
    return SF_EINVAL;
  if (!aligned16(res) || !aligned16(x) || !aligned16(bias) || !aligned16(y) || !aligned16(gamma) ||
      !aligned16(beta) || (xtilde && !aligned16(xtilde)) || (sum && !aligned16(sum)) ||
      (reinterpret_cast<uintptr_t>(y_planes) & 7u))
    return SF_EINVAL;
  if (rows == 0) return SF_OK;
  cudaStream_t s = as_stream(stream);
  const int h = static_cast<int>(H);
  __nv_bfloat16* yp = static_cast<__nv_bfloat16*>(y_planes);
#define SF_LNF(V) launch_ln_fwd<V>(x, gamma, beta, y, xtilde, rstd, rows, h, eps, s, res, bias, sum, yp, planes_format)
  if (H <= 128) return SF_LNF(1);
  if (H <= 256) return SF_LNF(2);
  if (H <= 512) return SF_LNF(4);
  if (H <= 768) return SF_LNF(6);
  return SF_LNF(8);
#undef SF_LNF
}

int sf_layernorm_fwd_residual(const float* res, const float* x, const float* bias, const float* gamma,
                              const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                              int64_t rows, int64_t H, float eps, void* stream) {
  return sf_layernorm_fwd_residual_p(res, x, bias, gamma, beta, y, sum, xtilde, rstd, rows, H, eps, nullptr,
                                     stream);
}

size_t sf_layernorm_bwd_workspace_bytes(int64_t rows, int64_t H) {
  const int64_t r = rows > 0 ? rows : 1;
  return a256(static_cast<size_t>(ln_bwd_grid(r)) * 2 * H * sizeof(float)) +
         a256(static_cast<size_t>(r + 1) * sizeof(int32_t));
}

int sf_layernorm_bwd_p(const float* g, const float* gamma, const float* xtilde,
                       const float* values, const int32_t* indices, int64_t k,
                       const int32_t* row_ptr, const float* rstd,
                       float* dx, float* dgamma, float* dbeta, int64_t rows, int64_t H, void* ws,
                       void* dx_planes, void* stream) {
  return sf_layernorm_bwd_pf(g, gamma, xtilde, values, indices, k, row_ptr, rstd, dx, dgamma, dbeta, rows, H, ws,
                             dx_planes, 0, nullptr, stream);
}

int sf_layernorm_bwd_pf(const float* g, const float* gamma, const float* xtilde,
                        const float* values, const int32_t* indices, int64_t k,
                        const int32_t* row_ptr, const float* rstd,
                        float* dx, float* dgamma, float* dbeta, int64_t rows, int64_t H, void* ws,
                        void* dx_planes, int planes_format, float* dx_row_scale, void* stream) {
  if (planes_format < 0 || planes_format > 2 || (planes_format == 2 && dx_planes && !dx_row_scale))
    return SF_EINVAL;
  if (rows < 0 || H < 4 || H % 4 || H > 1024 || !g || !gamma || !rstd || !dx) return SF_EINVAL;
  if (!xtilde && (k < 0 || (k > 0 && (!values || !indices)))) return SF_EINVAL;
  if (!ws) return SF_EINVAL;
  if (!aligned16(g) || !aligned16(dx) || !aligned16(gamma) || (xtilde && !aligned16(xtilde)) ||
      (reinterpret_cast<uintptr_t>(dx_planes) & 7u))
    return SF_EINVAL;
  if (rows == 0) return SF_OK;
  cudaStream_t s = as_stream(stream);
  const int h = static_cast<int>(H);
  const PlanesOut po{static_cast<__nv_bfloat16*>(dx_planes), planes_format, dx_row_scale};
#define SF_LNB(V) \
  launch_ln_bwd<V>(g, gamma, xtilde, values, indices, k, row_ptr, rstd, dx, dgamma, dbeta, rows, h, ws, \
                   s, po)
  if (H <= 128) return SF_LNB(1);
  if (H <= 256) return SF_LNB(2);
  if (H <= 512) return SF_LNB(4);
  if (H <= 768) return SF_LNB(6);
  return SF_LNB(8);
#undef SF_LNB
}

int sf_layernorm_bwd(const float* g, const float* gamma, const float* xtilde,
                     const float* values, const int32_t* indices, int64_t k,
                     const int32_t* row_ptr, const float* rstd,
                     float* dx, float* dgamma, float* dbeta, int64_t rows, int64_t H, void* ws,
                     void* stream) {
  return sf_layernorm_bwd_p(g, gamma, xtilde, values, indices, k, row_ptr, rstd, dx, dgamma, dbeta, rows, H, ws,
                            nullptr, stream);
}

int sf_softmax_fwd_q8(const float* sc, float* probs, void* codes, int64_t rows, int64_t W,
                      float scale, int fb, int is_signed, void* stream) {
  if (rows < 0 || W < 1 || W > 1024 || fb < 0 || fb > 8 || !sc || !codes) return SF_EINVAL;
  if (rows == 0) return SF_OK;
  cudaStream_t s = as_stream(stream);
  const float qs = static_cast<float>(1 << fb);
  const float lo = is_signed ? -128.f : 0.f, hi = is_signed ? 127.f : 255.f;
  uint8_t* c = static_cast<uint8_t*>(codes);
  const int w = static_cast<int>(W);
  if (W % 4 == 0 && aligned16(sc) && (!probs || aligned16(probs)) &&
      (reinterpret_cast<uintptr_t>(c) & 3u) == 0) {
    const unsigned grid = grid_for(rows * 32, kLT, 8);
    const int w4 = w / 4;
#define SF_SMV(MV) \
  k_softmax_fwd_q8_v4<MV><<<grid, kLT, 0, s>>>(sc, probs, c, rows, w4, scale, qs, lo, hi)
    if (w4 <= 32) SF_SMV(1);
    else if (w4 <= 64) SF_SMV(2);
    else if (w4 <= 128) SF_SMV(4);
    else SF_SMV(8);
#undef SF_SMV
    return check_launch();
  }
  if (W <= 128) return launch_softmax_fwd<4>(sc, probs, c, rows, w, scale, qs, lo, hi, s);
  if (W <= 256) return launch_softmax_fwd<8>(sc, probs, c, rows, w, scale, qs, lo, hi, s);
  if (W <= 512) return launch_softmax_fwd<16>(sc, probs, c, rows, w, scale, qs, lo, hi, s);
  return launch_softmax_fwd<32>(sc, probs, c, rows, w, scale, qs, lo, hi, s);
}

int sf_softmax_bwd_q8(const float* g, const void* codes, float* ds, int64_t rows, int64_t W,
                      int fb, int is_signed, float scale, void* stream) {
  if (rows < 0 || W < 1 || W > 1024 || fb < 0 || fb > 8 || !g || !codes || !ds) return SF_EINVAL;
  if (rows == 0) return SF_OK;
  cudaStream_t s = as_stream(stream);
  const float inv = 1.0f / static_cast<float>(1 << fb);
  const uint8_t* c = static_cast<const uint8_t*>(codes);
  const int w = static_cast<int>(W);
  const bool sg = is_signed != 0;
  if (W % 4 == 0 && aligned16(g) && aligned16(ds) && (reinterpret_cast<uintptr_t>(c) & 3u) == 0) {
    const unsigned grid = grid_for(rows * 32, kLT, 8);
    const int w4 = w / 4;
#define SF_SMB(MV)                                                                        \
  (sg ? (k_softmax_bwd_q8_v4<MV, true><<<grid, kLT, 0, s>>>(g, c, ds, rows, w4, inv, scale), 0) \
      : (k_softmax_bwd_q8_v4<MV, false><<<grid, kLT, 0, s>>>(g, c, ds, rows, w4, inv, scale), 0))
    if (w4 <= 32) SF_SMB(1);
    else if (w4 <= 64) SF_SMB(2);
    else if (w4 <= 128) SF_SMB(4);
    else SF_SMB(8);
#undef SF_SMB
    return check_launch();
  }
  if (W <= 128) return launch_softmax_bwd<4>(g, c, ds, rows, w, inv, sg, scale, s);
  if (W <= 256) return launch_softmax_bwd<8>(g, c, ds, rows, w, inv, sg, scale, s);
  if (W <= 512) return launch_softmax_bwd<16>(g, c, ds, rows, w, inv, sg, scale, s);
  return launch_softmax_bwd<32>(g, c, ds, rows, w, inv, sg, scale, s);
}

}  // extern "C"
