// Fused self-attention core with the SlimFit matsoft8 caches, fp32 SIMT.
//
// Reference (pure numpy, float32): per head
//   scores = q @ k^T                     (matmul, tensor.py:290-334; caches
//                                         q and k^T as 8-bit codes)
//   probs  = softmax(scores * scale)     (softmax, tensor.py:413-444; caches
//                                         probs as 8-bit codes, shared with
//                                         the context matmul)
//   ctx    = probs @ v                   (matmul; caches v as 8-bit codes)
// with q/k/v = x @ W + b split into heads (model.py:202-238).  The backward
// pass decodes every operand from those codes (SavedValue.get,
// tensor.py:132-135):
//   dP = g @ v~^T,  dv = p~^T @ g,  dS = p~ (dP - rowsum(dP p~)) scale,
//   dq = dS @ k~,   dk = dS^T @ q~.
//
// Unfused, that is three batched SGEMMs + softmax + head split/merge + four
// 8-bit encoders forward and four SGEMMs + softmax backward + decoders
// backward, each round-tripping (B, h, T, T) fp32 through HBM.  Here one CTA
// keeps a head's tiles in shared memory: forward reads the q/k/v projection
// rows straight from the GEMM output (bias added in registers, exactly as
// the split kernel rounds it), writes the four code caches and the context
// in the merged (B, T, H) layout -- scores and probabilities never reach
// HBM.  Backward reads g in the merged layout and the codes, and writes
// dq | dk | dv side by side into the (B*T, 3H) operand of the q/k/v
// input-gradient GEMM (tensor.py's _QKV convention).
//
// Arithmetic is fp32 FMA on the CUDA cores (the reference's precision; the
// products are 128x128x64, too short for a split-bf16 tensor-core scheme to
// pay for its extra passes here).  Scale, exp, division and the code
// rounding are the same operations, in the same order, as the unfused
// kernels (layernorm.cu softmax, codec8.cu quantize).
//
// Limits: head dim 64; T <= 128 with T % 4 == 0 runs the one-head kernels,
// any other T <= 384 the query-tiled ("wide") kernels below (ViT T = 197,
// BERT-large T = 384); the host keeps the unfused path beyond.
#include <cuda_bf16.h>

#include "common.cuh"
#include <algorithm>

namespace sf {
namespace {

constexpr int kDH = 64;       // head dim
constexpr int kTM = 128;      // max sequence length
constexpr int kFT = 256;      // forward threads
constexpr int kBT = 512;      // backward threads
constexpr int kVS = kDH + 4;  // Q / K / V / G / Pt row stride (see below)
constexpr int kSS = kTM + 4;  // dS row stride

__device__ __forceinline__ float4 ld4s(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4s(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

__device__ __forceinline__ uint32_t codes4(float4 v, float qs, float lo, float hi) {
  const uint32_t c0 = static_cast<uint8_t>(fixed_code(v.x, qs, lo, hi));
  const uint32_t c1 = static_cast<uint8_t>(fixed_code(v.y, qs, lo, hi));
  const uint32_t c2 = static_cast<uint8_t>(fixed_code(v.z, qs, lo, hi));
  const uint32_t c3 = static_cast<uint8_t>(fixed_code(v.w, qs, lo, hi));
  return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

// four signed 8-bit codes -> code * inv (exact: inv is a power of two)
__device__ __forceinline__ float4 decode4(uint32_t w, float inv) {
  return make_float4(static_cast<float>(static_cast<int8_t>(w & 0xFFu)) * inv,
                     static_cast<float>(static_cast<int8_t>((w >> 8) & 0xFFu)) * inv,
                     static_cast<float>(static_cast<int8_t>((w >> 16) & 0xFFu)) * inv,
                     static_cast<float>(static_cast<int8_t>(w >> 24)) * inv);
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ float comp(const float4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// Shared-memory tiles are row-major with a 68-float row stride: a float4 at
// (row, d4) sits in 16-byte bank group (17 row + d4) mod 8 = (row + d4) mod
// 8, so eight lanes reading the same d4 of eight consecutive rows, or eight
// consecutive d4 of one row, never conflict.  The global loads are fully
// coalesced (16 lanes per 256-byte head row).  In the products over the key
// axis a thread owns the eight keys lc + 8e (e = 0..7), again eight
// consecutive rows per quarter-warp.

// ------------------------------------------------------------------ forward
// grid (ceil(T / 64), B * h); CTA = 64 query rows of one head.
// smem: [Q 64 x kVS | K 128 x kVS]  (reused as Pt 128 x kVS after the scores)
//       V 128 x kVS, row max/sum exchange.
__global__ void __launch_bounds__(kFT, 2) k_attn_fwd(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint32_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ __align__(16) float sm[];
  float* Q = sm;                               // [r][kVS]
  float* K = sm + 64 * kVS;                    // [j][kVS]
  float* Pt = sm;                              // [j][kVS]  (after the scores)
  float* V = sm + (64 + kTM) * kVS;            // [j][kVS]
  float* redm = V + kTM * kVS;                 // [2][64]
  float* reds = redm + 128;                    // [2][64]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int row0 = blockIdx.x * 64;
  const int H = h * kDH;
  const int64_t M = static_cast<int64_t>(gridDim.y / h) * T;     // B * T
  const int64_t MH = M * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;             // first row of this sequence
  const int hoff = hh * kDH;

  // ---- loads: 16 lanes per head row (float4 d4 = tid & 15), coalesced
  {
    const int d4 = tid & 15;
    const float4 bqv = __ldg(reinterpret_cast<const float4*>(bq + hoff) + d4);
    const float4 bkv = __ldg(reinterpret_cast<const float4*>(bk + hoff) + d4);
    const float4 bvv = __ldg(reinterpret_cast<const float4*>(bv + hoff) + d4);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = tid >> 4; r < 64; r += kFT / 16) {              // q: this CTA's rows
      const int t = row0 + r;
      float4 v = z;
      if (t < T) {
        v = add4(__ldg(reinterpret_cast<const float4*>(y3 + (rbase + t) * H + hoff) + d4), bqv);
        qc[((static_cast<int64_t>(bh) * T + t) * kDH) / 4 + d4] = codes4(v, qs, lo, hi);
      }
      st4s(Q + r * kVS + 4 * d4, v);
    }
    for (int t = tid >> 4; t < kTM; t += kFT / 16) {             // k, v: all rows
      float4 kv = z, vv = z;
      if (t < T) {
        kv = add4(__ldg(reinterpret_cast<const float4*>(y3 + MH + (rbase + t) * H + hoff) + d4), bkv);
        vv = add4(__ldg(reinterpret_cast<const float4*>(y3 + 2 * MH + (rbase + t) * H + hoff) + d4), bvv);
        if (t >= row0 && t < row0 + 64) {                          // each row coded once
          const int64_t o = ((static_cast<int64_t>(bh) * T + t) * kDH) / 4 + d4;
          kc[o] = codes4(kv, qs, lo, hi);
          vc[o] = codes4(vv, qs, lo, hi);
        }
      }
      st4s(K + t * kVS + 4 * d4, kv);
      st4s(V + t * kVS + 4 * d4, vv);
    }
  }
  __syncthreads();

  // ---- scores: thread = 4 rows x 8 keys (kb + lc + 8e)
  const int rbw = w >> 1, cbw = w & 1, lr = lane >> 3, lc = lane & 7;
  const int rl = rbw * 16 + lr * 4;                 // first local row
  const int kb = cbw * 64 + lc;                     // first key; keys kb + 8e
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
#pragma unroll 2
  for (int d4 = 0; d4 < kDH / 4; ++d4) {
    float4 a[4], k[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = ld4s(Q + (rl + i) * kVS + 4 * d4);
#pragma unroll
    for (int e = 0; e < 8; ++e) k[e] = ld4s(K + (kb + 8 * e) * kVS + 4 * d4);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc[i][e] = fmaf(a[i].x, k[e].x, acc[i][e]);
        acc[i][e] = fmaf(a[i].y, k[e].y, acc[i][e]);
        acc[i][e] = fmaf(a[i].z, k[e].z, acc[i][e]);
        acc[i][e] = fmaf(a[i].w, k[e].w, acc[i][e]);
      }
  }

  // ---- softmax over keys (scale, max, exp, sum, divide as k_softmax_fwd_q8)
  float m[4], ssum[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[i] = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[i][e] = kb + 8 * e < T ? __fmul_rn(acc[i][e], scale) : -INFINITY;
      m[i] = fmaxf(m[i], acc[i][e]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) m[i] = fmaxf(m[i], __shfl_xor_sync(0xFFFFFFFFu, m[i], o));
  }
  if (lc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) redm[cbw * 64 + rl + i] = m[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[i] = fmaxf(redm[rl + i], redm[64 + rl + i]);
    ssum[i] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[i][e] = kb + 8 * e < T ? expf(acc[i][e] - m[i]) : 0.f;
      ssum[i] += acc[i][e];
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) ssum[i] += __shfl_xor_sync(0xFFFFFFFFu, ssum[i], o);
  }
  if (lc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) reds[cbw * 64 + rl + i] = ssum[i];
  }
  __syncthreads();                                  // also: Q/K reads are done
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float tot = reds[rl + i] + reds[64 + rl + i];
    const int t = row0 + rl + i;
    uint8_t* prow = reinterpret_cast<uint8_t*>(pc) + (static_cast<int64_t>(bh) * T + t) * T;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[i][e] = __fdiv_rn(acc[i][e], tot);
      if (t < T && kb + 8 * e < T) prow[kb + 8 * e] = static_cast<uint8_t>(fixed_code(acc[i][e], qs, lo, hi));
    }
  }
  // probabilities, transposed, over the (now free) Q/K region
#pragma unroll
  for (int e = 0; e < 8; ++e)
    st4s(Pt + (kb + 8 * e) * kVS + rl, make_float4(acc[0][e], acc[1][e], acc[2][e], acc[3][e]));
  __syncthreads();

  // ---- context = P @ V: thread = 4 rows x 4 dims
  const int dc = cbw * 32 + lc * 4;
  float o[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[i][e] = 0.f;
#pragma unroll 4
  for (int j = 0; j < T; ++j) {
    const float4 p = ld4s(Pt + j * kVS + rl);
    const float4 v = ld4s(V + j * kVS + dc);
    const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[i][0] = fmaf(pv[i], v.x, o[i][0]);
      o[i][1] = fmaf(pv[i], v.y, o[i][1]);
      o[i][2] = fmaf(pv[i], v.z, o[i][2]);
      o[i][3] = fmaf(pv[i], v.w, o[i][3]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = row0 + rl + i;
    if (t < T)
      st4s(ctx + (rbase + t) * H + hoff + dc, make_float4(o[i][0], o[i][1], o[i][2], o[i][3]));
      if (xp) planes_store4f(make_float4(o[i][0], o[i][1], o[i][2], o[i][3]), xp, MH, (rbase + t) * H + hoff + dc, pf);
  }
}

// ------------------------------------------------------------------ backward
// grid (B * h); CTA = one head, 512 threads.
// smem: region A = [G 128 x kVS | V~ 128 x kVS]  (reused as dS 128 x kSS)
//       Pc 128 x 128 bytes, Qc / Kc 128 x 64 bytes, row dots.
__global__ void __launch_bounds__(kBT, 1) k_attn_bwd(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
    const uint32_t* __restrict__ vc, const uint32_t* __restrict__ pc, int T, int h, float scale,
    float inv, float* __restrict__ gcat, __nv_bfloat16* __restrict__ xp) {
  extern __shared__ __align__(16) float sm[];
  float* G = sm;                               // [r][kVS]
  float* V = sm + kTM * kVS;                   // [j][kVS]
  float* dS = sm;                              // [r][kSS] (after dP / dV)
  uint32_t* Pc = reinterpret_cast<uint32_t*>(sm + 2 * kTM * kVS);   // [r][kTM/4] words
  uint32_t* Qc = Pc + kTM * (kTM / 4);                              // [r][16] words
  uint32_t* Kc = Qc + kTM * (kDH / 4);
  float* redd = reinterpret_cast<float*>(Kc + kTM * (kDH / 4));     // [2][128]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t P3 = static_cast<int64_t>(gridDim.x / h) * T * 3 * H;   // gcat planes' stride
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;            // code rows of this head

  // ---- loads (coalesced: 16 lanes per row)
  {
    const int d4 = tid & 15;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = tid >> 4; t < kTM; t += kBT / 16) {
      float4 gv = z, vv = z;
      uint32_t qw = 0, kw = 0;
      if (t < T) {
        gv = __ldg(reinterpret_cast<const float4*>(g + (rbase + t) * H + hoff) + d4);
        vv = decode4(__ldg(vc + (cbase + t) * (kDH / 4) + d4), inv);
        qw = __ldg(qc + (cbase + t) * (kDH / 4) + d4);
        kw = __ldg(kc + (cbase + t) * (kDH / 4) + d4);
      }
      st4s(G + t * kVS + 4 * d4, gv);
      st4s(V + t * kVS + 4 * d4, vv);
      Qc[t * (kDH / 4) + d4] = qw;
      Kc[t * (kDH / 4) + d4] = kw;
    }
  }
  const int T4w = T / 4;
  for (int idx = tid; idx < kTM * (kTM / 4); idx += kBT) {
    const int t = idx >> 5, c4 = idx & 31;
    Pc[idx] = (t < T && c4 < T4w) ? __ldg(pc + (cbase + t) * T4w + c4) : 0u;
  }
  __syncthreads();

  const int lr = lane >> 3, lc = lane & 7;
  const int rb = (w >> 1) * 16 + lr * 4;        // 4 rows (dP, dQ) / 4 keys (dV, dK)
  const int cbw = w & 1;
  const int kb = cbw * 64 + lc;                 // dP keys kb + 8e
  const uint8_t* Pb = reinterpret_cast<const uint8_t*>(Pc);

  // ---- dP = g @ v~^T : thread = 4 rows x 8 keys
  float dp[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) dp[i][e] = 0.f;
#pragma unroll 2
  for (int d4 = 0; d4 < kDH / 4; ++d4) {
    float4 a[4], v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = ld4s(G + (rb + i) * kVS + 4 * d4);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = ld4s(V + (kb + 8 * e) * kVS + 4 * d4);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        dp[i][e] = fmaf(a[i].x, v[e].x, dp[i][e]);
        dp[i][e] = fmaf(a[i].y, v[e].y, dp[i][e]);
        dp[i][e] = fmaf(a[i].z, v[e].z, dp[i][e]);
        dp[i][e] = fmaf(a[i].w, v[e].w, dp[i][e]);
      }
  }

  // ---- dv = p~^T @ g : thread = 4 keys x 4 dims, reduction over rows
  const int dc = cbw * 32 + lc * 4;
  {
    float o[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[i][e] = 0.f;
#pragma unroll 4
    for (int r = 0; r < T; ++r) {
      const float4 p = decode4(Pc[r * (kTM / 4) + rb / 4], inv);    // keys rb..rb+3
      const float4 gv = ld4s(G + r * kVS + dc);
      const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o[i][0] = fmaf(pv[i], gv.x, o[i][0]);
        o[i][1] = fmaf(pv[i], gv.y, o[i][1]);
        o[i][2] = fmaf(pv[i], gv.z, o[i][2]);
        o[i][3] = fmaf(pv[i], gv.w, o[i][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = rb + i;
      if (j < T) {
        st4s(gcat + (rbase + j) * (3 * H) + 2 * H + hoff + dc,
             make_float4(o[i][0], o[i][1], o[i][2], o[i][3]));
        if (xp) planes_store4(make_float4(o[i][0], o[i][1], o[i][2], o[i][3]), xp, P3,
                              (rbase + j) * (3 * H) + 2 * H + hoff + dc);
      }
    }
  }

  // ---- dS = p~ (dP - sum_j dP p~) scale  (as k_softmax_bwd_q8)
  float pr[4][8], dot[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = rb + i;
    dot[i] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      pr[i][e] = static_cast<float>(static_cast<int8_t>(Pb[r * kTM + kb + 8 * e])) * inv;
      dot[i] += __fmul_rn(dp[i][e], pr[i][e]);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) dot[i] += __shfl_xor_sync(0xFFFFFFFFu, dot[i], o);
  }
  if (lc == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) redd[cbw * kTM + rb + i] = dot[i];
  }
  __syncthreads();                                 // dot partials visible; G/V reads done
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float dt = redd[rb + i] + redd[kTM + rb + i];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      dS[(rb + i) * kSS + kb + 8 * e] = __fmul_rn(__fmul_rn(pr[i][e], __fsub_rn(dp[i][e], dt)), scale);
  }
  __syncthreads();

  // ---- dq = dS @ k~ : thread = 4 rows x 4 dims;  dk = dS^T @ q~ : 4 keys x 4 dims
  float oq[4][4], ok[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) oq[i][e] = ok[i][e] = 0.f;
#pragma unroll 2
  for (int j = 0; j < T; j += 4) {
    // dq: rows rb..rb+3, keys j..j+3
    float4 srow[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) srow[i] = ld4s(dS + (rb + i) * kSS + j);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 kv = decode4(Kc[(j + u) * (kDH / 4) + dc / 4], inv);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float sv = comp(srow[i], u);
        oq[i][0] = fmaf(sv, kv.x, oq[i][0]);
        oq[i][1] = fmaf(sv, kv.y, oq[i][1]);
        oq[i][2] = fmaf(sv, kv.z, oq[i][2]);
        oq[i][3] = fmaf(sv, kv.w, oq[i][3]);
      }
    }
    // dk: keys rb..rb+3, rows j..j+3
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 sk = ld4s(dS + (j + u) * kSS + rb);
      const float4 qv = decode4(Qc[(j + u) * (kDH / 4) + dc / 4], inv);
      const float sv[4] = {sk.x, sk.y, sk.z, sk.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ok[i][0] = fmaf(sv[i], qv.x, ok[i][0]);
        ok[i][1] = fmaf(sv[i], qv.y, ok[i][1]);
        ok[i][2] = fmaf(sv[i], qv.z, ok[i][2]);
        ok[i][3] = fmaf(sv[i], qv.w, ok[i][3]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = rb + i;
    if (t < T) {
      float* row = gcat + (rbase + t) * (3 * H) + hoff + dc;
      st4s(row, make_float4(oq[i][0], oq[i][1], oq[i][2], oq[i][3]));
      st4s(row + H, make_float4(ok[i][0], ok[i][1], ok[i][2], ok[i][3]));
      if (xp) {
        const int64_t o0 = (rbase + t) * (3 * H) + hoff + dc;
        planes_store4(make_float4(oq[i][0], oq[i][1], oq[i][2], oq[i][3]), xp, P3, o0);
        planes_store4(make_float4(ok[i][0], ok[i][1], ok[i][2], ok[i][3]), xp, P3, o0 + H);
      }
    }
  }
}

// ------------------------------------------------------------------ tensor cores
// mma.sync m16n8k16 bf16 -> fp32 (measured on B200: ~550 TFLOP/s, 8x the
// FP32 FMA rate).  fp32 operands are split exactly into three bf16 terms
// x = hi + mid + lo (8 + 8 + 8 significand bits); 8-bit cached codes times
// 2^-fb are exact in bf16.  A code-operand x fp32-operand product is thus
// three MMAs of exact bf16 x bf16 products accumulated in fp32 -- the
// backward's four products all have one code operand.
__device__ __forceinline__ uint32_t bf2(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void split3(float x, float& h, float& m, float& l) {
  h = __bfloat162float(__float2bfloat16_rn(x));
  float r = x - h;                              // exact
  m = __bfloat162float(__float2bfloat16_rn(r));
  r = r - m;                                    // exact
  l = __bfloat162float(__float2bfloat16_rn(r));
}

// (x0, x1) adjacent fragment elements -> hi / mid / lo packed pairs: one
// paired cvt.rn.bf16x2 per term, the bf16 -> fp32 widening is a shift
__device__ __forceinline__ void split_pair(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
  h = bf2(x0, x1);
  float r0 = x0 - __uint_as_float(h << 16), r1 = x1 - __uint_as_float(h & 0xFFFF0000u);   // exact
  m = bf2(r0, r1);
  r0 -= __uint_as_float(m << 16);                                                          // exact
  r1 -= __uint_as_float(m & 0xFFFF0000u);
  l = bf2(r0, r1);
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float code_f(int8_t c, float inv) { return static_cast<float>(c) * inv; }

// Backward on the tensor cores.  grid (B * h), 256 threads (8 warps); warp
// w owns rows [16w, 16w + 16) of dP / dS / dQ and keys [16w, 16w + 16) of
// dK / dV.  Fragment conventions (PTX m16n8k16): g = lane >> 2, t = lane & 3.
constexpr int kTB = 256;
constexpr int kGS = kDH + 8;            // G fp32 row stride (72: conflict-free float2 A loads)
constexpr int kPS = kTM + 4;            // Pc byte row stride (132: rows spread over banks)
constexpr int kVB = kDH + 8;            // Vb bf16 row stride (72): [j][d]
constexpr int kTS = kTM + 8;            // Kb / Qb [d][*] and Pt [j][r] bf16 row stride (136)
constexpr size_t kTcG = size_t(kTM) * kGS * 4;
constexpr size_t kTcVb = size_t(kTM) * kVB * 2;
constexpr size_t kTcKb = size_t(kDH) * kTS * 2;
constexpr size_t kTcPt = size_t(kTM) * kTS * 2;
constexpr size_t kTcPc = size_t(kTM) * kPS;
constexpr size_t kTcDS = size_t(kTM) * kSS * 4;
constexpr size_t kBwdTcSmem = kTcG + kTcVb + 2 * kTcKb + kTcPt + kTcPc + kTcDS;
static_assert(3 * size_t(kDH) * kTS * 2 <= kTcG + kTcVb, "g planes fit over G | Vb");

__global__ void __launch_bounds__(kTB, 1) k_attn_bwd_tc(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
    const uint32_t* __restrict__ vc, const uint32_t* __restrict__ pc, int T, int h, float scale,
    float inv, float* __restrict__ gcat, __nv_bfloat16* __restrict__ xp) {
  extern __shared__ __align__(16) unsigned char smb[];
  float* G = reinterpret_cast<float*>(smb);                                   // [r][kGS]
  __nv_bfloat16* Vb = reinterpret_cast<__nv_bfloat16*>(smb + kTcG);          // [j][kVB]
  __nv_bfloat16* Kb = reinterpret_cast<__nv_bfloat16*>(smb + kTcG + kTcVb);  // [d][kTS] (k~^T)
  __nv_bfloat16* Qb = Kb + kDH * kTS;                                          // [d][kTS] (q~^T)
  __nv_bfloat16* Pt = Qb + kDH * kTS;                                          // [j][kTS] (p~^T)
  int8_t* Pc = reinterpret_cast<int8_t*>(Pt + kTM * kTS);                      // [r][kTM]
  float* dS = reinterpret_cast<float*>(Pc + kTcPc);                            // [r][kSS]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t P3 = static_cast<int64_t>(gridDim.x / h) * T * 3 * H;   // gcat planes' stride
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const __nv_bfloat16 zb = __float2bfloat16_rn(0.f);

  // ---- loads: fixed trip counts, every global load of a loop issued before
  // its shared-memory stores
  {
    const int d4 = tid & 15;
    float4 gv[kTM / 16];
    uint32_t vw[kTM / 16];
#pragma unroll
    for (int q = 0; q < kTM / 16; ++q) {                          // g rows, v~ rows (coalesced)
      const int t = (tid >> 4) + 16 * q;
      gv[q] = t < T ? __ldg(reinterpret_cast<const float4*>(g + (rbase + t) * H + hoff) + d4)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      vw[q] = t < T ? __ldg(vc + (cbase + t) * (kDH / 4) + d4) : 0u;
    }
    uint32_t kw[kTM * (kDH / 4) / kTB], qw[kTM * (kDH / 4) / kTB];
#pragma unroll
    for (int q = 0; q < kTM * (kDH / 4) / kTB; ++q) {             // k~, q~ code words
      const int idx = tid + q * kTB;
      const int t = idx & (kTM - 1), c4 = idx >> 7;
      kw[q] = t < T ? __ldg(kc + (cbase + t) * (kDH / 4) + c4) : 0u;
      qw[q] = t < T ? __ldg(qc + (cbase + t) * (kDH / 4) + c4) : 0u;
    }
    const int T4w = T / 4;
    uint32_t pw[kTM * (kTM / 4) / kTB];
#pragma unroll
    for (int q = 0; q < kTM * (kTM / 4) / kTB; ++q) {             // p code rows (coalesced)
      const int idx = tid + q * kTB;
      const int r = idx >> 5, c4 = idx & 31;
      pw[q] = (r < T && c4 < T4w) ? __ldg(pc + (cbase + r) * T4w + c4) : 0u;
    }
#pragma unroll
    for (int q = 0; q < kTM / 16; ++q) {
      const int t = (tid >> 4) + 16 * q;
      *reinterpret_cast<float4*>(G + t * kGS + 4 * d4) = gv[q];
      const float4 vv = decode4(vw[q], inv);
      uint32_t* vrow = reinterpret_cast<uint32_t*>(Vb + t * kVB + 4 * d4);
      vrow[0] = bf2(vv.x, vv.y);
      vrow[1] = bf2(vv.z, vv.w);
    }
#pragma unroll
    for (int q = 0; q < kTM * (kDH / 4) / kTB; ++q) {             // k~^T, q~^T (transposed)
      const int idx = tid + q * kTB;
      const int t = idx & (kTM - 1), c4 = idx >> 7;
      const float4 kv = decode4(kw[q], inv), qv = decode4(qw[q], inv);
      Kb[(4 * c4 + 0) * kTS + t] = __float2bfloat16_rn(kv.x);
      Kb[(4 * c4 + 1) * kTS + t] = __float2bfloat16_rn(kv.y);
      Kb[(4 * c4 + 2) * kTS + t] = __float2bfloat16_rn(kv.z);
      Kb[(4 * c4 + 3) * kTS + t] = __float2bfloat16_rn(kv.w);
      Qb[(4 * c4 + 0) * kTS + t] = __float2bfloat16_rn(qv.x);
      Qb[(4 * c4 + 1) * kTS + t] = __float2bfloat16_rn(qv.y);
      Qb[(4 * c4 + 2) * kTS + t] = __float2bfloat16_rn(qv.z);
      Qb[(4 * c4 + 3) * kTS + t] = __float2bfloat16_rn(qv.w);
    }
#pragma unroll
    for (int q = 0; q < kTM * (kTM / 4) / kTB; ++q) {
      const int idx = tid + q * kTB;
      const int r = idx >> 5, c4 = idx & 31;
      *reinterpret_cast<uint32_t*>(Pc + r * kPS + 4 * c4) = pw[q];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < kTM * (kTM / 2); idx += kTB) {       // p~^T: Pt[j][r, r+1]
    const int j = idx & (kTM - 1), r2 = idx >> 7;
    reinterpret_cast<uint32_t*>(Pt + j * kTS)[r2] =
        bf2(code_f(Pc[(2 * r2) * kPS + j], inv), code_f(Pc[(2 * r2 + 1) * kPS + j], inv));
  }
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int R0 = 16 * w;
  const uint32_t* Vb32 = reinterpret_cast<const uint32_t*>(Vb);
  const uint32_t* Kb32 = reinterpret_cast<const uint32_t*>(Kb);
  const uint32_t* Qb32 = reinterpret_cast<const uint32_t*>(Qb);
  const uint32_t* Pt32 = reinterpret_cast<const uint32_t*>(Pt);

  // ---- dP = g v~^T: rows R0.., all 128 keys (16 n-tiles), k = d
  float acc[16][4];
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < kDH / 16; ++kb) {
    uint32_t ah[4], am[4], al[4];
    {
      const float2 x0 = *reinterpret_cast<const float2*>(G + (R0 + gq) * kGS + 16 * kb + 2 * tq);
      const float2 x1 = *reinterpret_cast<const float2*>(G + (R0 + gq + 8) * kGS + 16 * kb + 2 * tq);
      const float2 x2 = *reinterpret_cast<const float2*>(G + (R0 + gq) * kGS + 16 * kb + 8 + 2 * tq);
      const float2 x3 = *reinterpret_cast<const float2*>(G + (R0 + gq + 8) * kGS + 16 * kb + 8 + 2 * tq);
      split_pair(x0.x, x0.y, ah[0], am[0], al[0]);
      split_pair(x1.x, x1.y, ah[1], am[1], al[1]);
      split_pair(x2.x, x2.y, ah[2], am[2], al[2]);
      split_pair(x3.x, x3.y, ah[3], am[3], al[3]);
    }
    uint32_t b0[16], b1[16];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      b0[nt] = Vb32[(8 * nt + gq) * (kVB / 2) + 8 * kb + tq];
      b1[nt] = Vb32[(8 * nt + gq) * (kVB / 2) + 8 * kb + 4 + tq];
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) mma16816(acc[nt], al, b0[nt], b1[nt]);
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) mma16816(acc[nt], am, b0[nt], b1[nt]);
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) mma16816(acc[nt], ah, b0[nt], b1[nt]);
  }

  // ---- dS = p~ (dP - rowsum(dP p~)) scale, rows R0 + gq (c0, c1) and + 8 (c2, c3)
  {
    float dot0 = 0.f, dot1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int j = 8 * nt + 2 * tq;
      const int8_t* p0 = Pc + (R0 + gq) * kPS + j;
      const int8_t* p1 = Pc + (R0 + gq + 8) * kPS + j;
      dot0 += __fmul_rn(acc[nt][0], code_f(p0[0], inv)) + __fmul_rn(acc[nt][1], code_f(p0[1], inv));
      dot1 += __fmul_rn(acc[nt][2], code_f(p1[0], inv)) + __fmul_rn(acc[nt][3], code_f(p1[1], inv));
    }
    dot0 += __shfl_xor_sync(0xFFFFFFFFu, dot0, 1);
    dot0 += __shfl_xor_sync(0xFFFFFFFFu, dot0, 2);
    dot1 += __shfl_xor_sync(0xFFFFFFFFu, dot1, 1);
    dot1 += __shfl_xor_sync(0xFFFFFFFFu, dot1, 2);
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int j = 8 * nt + 2 * tq;
      const int8_t* p0 = Pc + (R0 + gq) * kPS + j;
      const int8_t* p1 = Pc + (R0 + gq + 8) * kPS + j;
      acc[nt][0] = __fmul_rn(__fmul_rn(code_f(p0[0], inv), __fsub_rn(acc[nt][0], dot0)), scale);
      acc[nt][1] = __fmul_rn(__fmul_rn(code_f(p0[1], inv), __fsub_rn(acc[nt][1], dot0)), scale);
      acc[nt][2] = __fmul_rn(__fmul_rn(code_f(p1[0], inv), __fsub_rn(acc[nt][2], dot1)), scale);
      acc[nt][3] = __fmul_rn(__fmul_rn(code_f(p1[1], inv), __fsub_rn(acc[nt][3], dot1)), scale);
      *reinterpret_cast<float2*>(dS + (R0 + gq) * kSS + j) = make_float2(acc[nt][0], acc[nt][1]);
      *reinterpret_cast<float2*>(dS + (R0 + gq + 8) * kSS + j) = make_float2(acc[nt][2], acc[nt][3]);
    }
  }

  // ---- dq = dS k~: A = dS from registers (C -> A fragments), k = key
  {
    float oq[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) oq[nt][0] = oq[nt][1] = oq[nt][2] = oq[nt][3] = 0.f;
#pragma unroll
    for (int kb = 0; kb < kTM / 16; ++kb) {
      uint32_t ah[4], am[4], al[4];
      split_pair(acc[2 * kb][0], acc[2 * kb][1], ah[0], am[0], al[0]);
      split_pair(acc[2 * kb][2], acc[2 * kb][3], ah[1], am[1], al[1]);
      split_pair(acc[2 * kb + 1][0], acc[2 * kb + 1][1], ah[2], am[2], al[2]);
      split_pair(acc[2 * kb + 1][2], acc[2 * kb + 1][3], ah[3], am[3], al[3]);
      uint32_t b0[8], b1[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        b0[nt] = Kb32[(8 * nt + gq) * (kTS / 2) + 8 * kb + tq];
        b1[nt] = Kb32[(8 * nt + gq) * (kTS / 2) + 8 * kb + 4 + tq];
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(oq[nt], al, b0[nt], b1[nt]);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(oq[nt], am, b0[nt], b1[nt]);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(oq[nt], ah, b0[nt], b1[nt]);
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int d = 8 * nt + 2 * tq;
      const int r0 = R0 + gq, r1 = R0 + gq + 8;
      if (r0 < T) {
        *reinterpret_cast<float2*>(gcat + (rbase + r0) * (3 * H) + hoff + d) = make_float2(oq[nt][0], oq[nt][1]);
        if (xp) planes_store2(oq[nt][0], oq[nt][1], xp, P3, (rbase + r0) * (3 * H) + hoff + d);
      }
      if (r1 < T) {
        *reinterpret_cast<float2*>(gcat + (rbase + r1) * (3 * H) + hoff + d) = make_float2(oq[nt][2], oq[nt][3]);
        if (xp) planes_store2(oq[nt][2], oq[nt][3], xp, P3, (rbase + r1) * (3 * H) + hoff + d);
      }
    }
  }
  // g split once into bf16 planes gT_{h,m,l}[d][r] (the dv B operand,
  // pairs along r) over the G | Vb region, which dP no longer needs
  __syncthreads();                                   // dS complete; every dP read of G / Vb done
  {
    float2 gv[16];
    // item (d, r2): lane bits pick d & 7 and r2 & 3, so both the G reads
    // (bank 8 r2 + d) and the plane writes (bank 4 d + r2) are conflict-free
    auto item = [&](int q, int& d, int& r2) {
      const int it = tid + q * kTB, ln = it & 31, rest = it >> 5;
      d = (ln & 7) + 8 * (rest & 7);
      r2 = (ln >> 3) + 4 * (rest >> 3);
    };
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int d, r2;
      item(q, d, r2);
      gv[q] = make_float2(G[(2 * r2) * kGS + d], G[(2 * r2 + 1) * kGS + d]);
    }
    __syncthreads();
    uint32_t* P3 = reinterpret_cast<uint32_t*>(smb);          // 3 planes of [d][kTS/2] words
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int d, r2;
      item(q, d, r2);
      uint32_t hh, mm, ll;
      split_pair(gv[q].x, gv[q].y, hh, mm, ll);
      P3[0 * kDH * (kTS / 2) + d * (kTS / 2) + r2] = hh;
      P3[1 * kDH * (kTS / 2) + d * (kTS / 2) + r2] = mm;
      P3[2 * kDH * (kTS / 2) + d * (kTS / 2) + r2] = ll;
    }
    __syncthreads();
  }
  const uint32_t* GH = reinterpret_cast<const uint32_t*>(smb);
  const uint32_t* GM = GH + kDH * (kTS / 2);
  const uint32_t* GL = GM + kDH * (kTS / 2);

  // ---- dk = dS^T q~ (A = dS^T from smem, split) and dv = p~^T g (A = p~^T exact, B = g planes)
  {
    float ok[8][4], ov[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      ok[nt][0] = ok[nt][1] = ok[nt][2] = ok[nt][3] = 0.f;
      ov[nt][0] = ov[nt][1] = ov[nt][2] = ov[nt][3] = 0.f;
    }
    const int J0 = R0;
#pragma unroll 2
    for (int kb = 0; kb < kTM / 16; ++kb) {
      const int r = 16 * kb + 2 * tq;
      uint32_t ah[4], am[4], al[4];
      split_pair(dS[r * kSS + J0 + gq], dS[(r + 1) * kSS + J0 + gq], ah[0], am[0], al[0]);
      split_pair(dS[r * kSS + J0 + gq + 8], dS[(r + 1) * kSS + J0 + gq + 8], ah[1], am[1], al[1]);
      split_pair(dS[(r + 8) * kSS + J0 + gq], dS[(r + 9) * kSS + J0 + gq], ah[2], am[2], al[2]);
      split_pair(dS[(r + 8) * kSS + J0 + gq + 8], dS[(r + 9) * kSS + J0 + gq + 8], ah[3], am[3], al[3]);
      uint32_t ap[4];
      ap[0] = Pt32[(J0 + gq) * (kTS / 2) + 8 * kb + tq];
      ap[1] = Pt32[(J0 + gq + 8) * (kTS / 2) + 8 * kb + tq];
      ap[2] = Pt32[(J0 + gq) * (kTS / 2) + 8 * kb + 4 + tq];
      ap[3] = Pt32[(J0 + gq + 8) * (kTS / 2) + 8 * kb + 4 + tq];
      uint32_t b0[8], b1[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        b0[nt] = Qb32[(8 * nt + gq) * (kTS / 2) + 8 * kb + tq];
        b1[nt] = Qb32[(8 * nt + gq) * (kTS / 2) + 8 * kb + 4 + tq];
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(ok[nt], al, b0[nt], b1[nt]);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(ok[nt], am, b0[nt], b1[nt]);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(ok[nt], ah, b0[nt], b1[nt]);
      // dv: B[k = r][n = d] = g[r][d] from the split planes
      const uint32_t* GP[3] = {GL, GM, GH};
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        uint32_t c0[8], c1[8];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const int o = (8 * nt + gq) * (kTS / 2) + 8 * kb + tq;
          c0[nt] = GP[p][o];
          c1[nt] = GP[p][o + 4];
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) mma16816(ov[nt], ap, c0[nt], c1[nt]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int d = 8 * nt + 2 * tq;
      const int j0 = J0 + gq, j1 = J0 + gq + 8;
      if (j0 < T) {
        float* row = gcat + (rbase + j0) * (3 * H) + hoff + d;
        *reinterpret_cast<float2*>(row + H) = make_float2(ok[nt][0], ok[nt][1]);
        *reinterpret_cast<float2*>(row + 2 * H) = make_float2(ov[nt][0], ov[nt][1]);
        if (xp) {
          const int64_t o0 = (rbase + j0) * (3 * H) + hoff + d;
          planes_store2(ok[nt][0], ok[nt][1], xp, P3, o0 + H);
          planes_store2(ov[nt][0], ov[nt][1], xp, P3, o0 + 2 * H);
        }
      }
      if (j1 < T) {
        float* row = gcat + (rbase + j1) * (3 * H) + hoff + d;
        *reinterpret_cast<float2*>(row + H) = make_float2(ok[nt][2], ok[nt][3]);
        *reinterpret_cast<float2*>(row + 2 * H) = make_float2(ov[nt][2], ov[nt][3]);
        if (xp) {
          const int64_t o0 = (rbase + j1) * (3 * H) + hoff + d;
          planes_store2(ok[nt][2], ok[nt][3], xp, P3, o0 + H);
          planes_store2(ov[nt][2], ov[nt][3], xp, P3, o0 + 2 * H);
        }
      }
    }
  }
}

// Forward on the tensor cores.  grid (B * h); one CTA = one whole head
// (k / v staged once), 512 threads = 16 warps: warp w owns rows
// [16 (w >> 1), +16) and keys [64 (w & 1), +64).  q, k, v (fp32, bias added
// as the split kernel does) are stored as three bf16 planes each, row-major
// [row][d]; S = q k^T and ctx = p v each take the six split products that
// carry fp32 accuracy (hh, hm, mh, mm, hl, lh; the dropped ml, lm, ll are
// below 2^-24 relative), smallest first.
constexpr int kTF = 512;
constexpr size_t kPlane = size_t(kTM) * kVB;                 // bf16 elements per plane
constexpr size_t kFwdTcSmem = 9 * kPlane * 2 + 4 * kTM * sizeof(float) +
                              size_t(8) * 16 * (kDH + 4) * sizeof(float);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ldsm_x2_trans(uint32_t& r0, uint32_t& r1, const void* row_addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(row_addr)));
}

__global__ void __launch_bounds__(kTF, 1) k_attn_fwd_tc(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint16_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ __align__(16) unsigned char smb[];
  __nv_bfloat16* Qp = reinterpret_cast<__nv_bfloat16*>(smb);   // [3][kTM][kVB]
  __nv_bfloat16* Kp = Qp + 3 * kPlane;
  __nv_bfloat16* Vp = Kp + 3 * kPlane;
  float* redm = reinterpret_cast<float*>(Vp + 3 * kPlane);     // [2][kTM]
  float* reds = redm + 2 * kTM;                                 // [2][kTM]
  float* part = reds + 2 * kTM;                                 // [8][16][kDH + 4]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.x / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  // ---- loads: (row, d4) items, 16 lanes per row (coalesced); bias, codes, split planes
  {
    const int d4 = tid & 15;
    const float4 bias[3] = {__ldg(reinterpret_cast<const float4*>(bq + hoff) + d4),
                            __ldg(reinterpret_cast<const float4*>(bk + hoff) + d4),
                            __ldg(reinterpret_cast<const float4*>(bv + hoff) + d4)};
    uint32_t* codes[3] = {qc, kc, vc};
    __nv_bfloat16* planes[3] = {Qp, Kp, Vp};
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      float4 x[kTM * 16 / kTF];
#pragma unroll
      for (int q = 0; q < kTM * 16 / kTF; ++q) {
        const int t = (tid >> 4) + (kTF / 16) * q;
        x[q] = t < T ? add4(__ldg(reinterpret_cast<const float4*>(y3 + m * MH + (rbase + t) * H + hoff) + d4),
                            bias[m])
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < kTM * 16 / kTF; ++q) {
        const int t = (tid >> 4) + (kTF / 16) * q;
        if (t < T) codes[m][(cbase + t) * (kDH / 4) + d4] = codes4(x[q], qs, lo, hi);
        uint32_t h0, m0, l0, h1, m1, l1;
        split_pair(x[q].x, x[q].y, h0, m0, l0);
        split_pair(x[q].z, x[q].w, h1, m1, l1);
        const size_t o = (static_cast<size_t>(t) * kVB + 4 * d4) / 2;   // word offset in a plane
        uint32_t* P = reinterpret_cast<uint32_t*>(planes[m]);
        P[o] = h0; P[o + 1] = h1;
        P[kPlane / 2 + o] = m0; P[kPlane / 2 + o + 1] = m1;
        P[kPlane + o] = l0; P[kPlane + o + 1] = l1;
      }
    }
  }
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int rg = w >> 1, kh = w & 1;
  const int R0 = 16 * rg, J0 = 64 * kh;
  const uint32_t* Q32 = reinterpret_cast<const uint32_t*>(Qp);
  const uint32_t* K32 = reinterpret_cast<const uint32_t*>(Kp);
  constexpr int PW = int(kPlane / 2);       // words per plane
  constexpr int RW = kVB / 2;               // words per row

  // ---- S = q k^T: rows R0.., keys J0.. (8 n-tiles), k = d
  float acc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < kDH / 16; ++kb) {
    uint32_t a[3][4];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      a[p][0] = Q32[p * PW + (R0 + gq) * RW + 8 * kb + tq];
      a[p][1] = Q32[p * PW + (R0 + gq + 8) * RW + 8 * kb + tq];
      a[p][2] = Q32[p * PW + (R0 + gq) * RW + 8 * kb + 4 + tq];
      a[p][3] = Q32[p * PW + (R0 + gq + 8) * RW + 8 * kb + 4 + tq];
    }
    uint32_t b0[3][8], b1[3][8];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        b0[p][nt] = K32[p * PW + (J0 + 8 * nt + gq) * RW + 8 * kb + tq];
        b1[p][nt] = K32[p * PW + (J0 + 8 * nt + gq) * RW + 8 * kb + 4 + tq];
      }
    // product-major, n-tile-minor: consecutive MMAs hit different
    // accumulators, so the tensor pipe never waits on its own result
    constexpr int PA[6] = {2, 0, 1, 1, 0, 0}, PB[6] = {0, 2, 1, 0, 1, 0};   // lh hl mm mh hm hh
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(acc[nt], a[PA[q]], b0[PB[q]][nt], b1[PB[q]][nt]);
  }

  // ---- softmax over keys, rows R0 + gq (c0, c1) and R0 + gq + 8 (c2, c3)
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    const bool v0 = j < T, v1 = j + 1 < T;
    acc[nt][0] = v0 ? __fmul_rn(acc[nt][0], scale) : -INFINITY;
    acc[nt][1] = v1 ? __fmul_rn(acc[nt][1], scale) : -INFINITY;
    acc[nt][2] = v0 ? __fmul_rn(acc[nt][2], scale) : -INFINITY;
    acc[nt][3] = v1 ? __fmul_rn(acc[nt][3], scale) : -INFINITY;
    m0 = fmaxf(m0, fmaxf(acc[nt][0], acc[nt][1]));
    m1 = fmaxf(m1, fmaxf(acc[nt][2], acc[nt][3]));
  }
  m0 = fmaxf(m0, __shfl_xor_sync(0xFFFFFFFFu, m0, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xFFFFFFFFu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xFFFFFFFFu, m1, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xFFFFFFFFu, m1, 2));
  if (tq == 0) {
    redm[kh * kTM + R0 + gq] = m0;
    redm[kh * kTM + R0 + gq + 8] = m1;
  }
  __syncthreads();
  m0 = fmaxf(redm[R0 + gq], redm[kTM + R0 + gq]);
  m1 = fmaxf(redm[R0 + gq + 8], redm[kTM + R0 + gq + 8]);
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    acc[nt][0] = j < T ? expf(acc[nt][0] - m0) : 0.f;
    acc[nt][1] = j + 1 < T ? expf(acc[nt][1] - m0) : 0.f;
    acc[nt][2] = j < T ? expf(acc[nt][2] - m1) : 0.f;
    acc[nt][3] = j + 1 < T ? expf(acc[nt][3] - m1) : 0.f;
    s0 += acc[nt][0] + acc[nt][1];
    s1 += acc[nt][2] + acc[nt][3];
  }
  s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, 1);
  s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, 2);
  s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, 1);
  s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, 2);
  if (tq == 0) {
    reds[kh * kTM + R0 + gq] = s0;
    reds[kh * kTM + R0 + gq + 8] = s1;
  }
  __syncthreads();
  s0 = reds[R0 + gq] + reds[kTM + R0 + gq];
  s1 = reds[R0 + gq + 8] + reds[kTM + R0 + gq + 8];
  const int r0 = R0 + gq, r1 = R0 + gq + 8;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    acc[nt][0] = __fdiv_rn(acc[nt][0], s0);
    acc[nt][1] = __fdiv_rn(acc[nt][1], s0);
    acc[nt][2] = __fdiv_rn(acc[nt][2], s1);
    acc[nt][3] = __fdiv_rn(acc[nt][3], s1);
    if (j < T) {                                           // T % 4 == 0: j + 1 < T too
      const uint32_t c00 = static_cast<uint8_t>(fixed_code(acc[nt][0], qs, lo, hi));
      const uint32_t c01 = static_cast<uint8_t>(fixed_code(acc[nt][1], qs, lo, hi));
      const uint32_t c10 = static_cast<uint8_t>(fixed_code(acc[nt][2], qs, lo, hi));
      const uint32_t c11 = static_cast<uint8_t>(fixed_code(acc[nt][3], qs, lo, hi));
      if (r0 < T) pc[((cbase + r0) * T + j) / 2] = static_cast<uint16_t>(c00 | (c01 << 8));
      if (r1 < T) pc[((cbase + r1) * T + j) / 2] = static_cast<uint16_t>(c10 | (c11 << 8));
    }
  }

  // ---- ctx partial = p v over this warp's 64 keys: A = p (registers, split), B = v planes (ldmatrix.trans)
  float o[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    uint32_t a[3][4];
    split_pair(acc[2 * kb][0], acc[2 * kb][1], a[0][0], a[1][0], a[2][0]);
    split_pair(acc[2 * kb][2], acc[2 * kb][3], a[0][1], a[1][1], a[2][1]);
    split_pair(acc[2 * kb + 1][0], acc[2 * kb + 1][1], a[0][2], a[1][2], a[2][2]);
    split_pair(acc[2 * kb + 1][2], acc[2 * kb + 1][3], a[0][3], a[1][3], a[2][3]);
    const int jrow = J0 + 16 * kb + (lane & 15);           // ldmatrix row address (lanes 0..15)
    uint32_t b0[3][8], b1[3][8];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int p = 0; p < 3; ++p) ldsm_x2_trans(b0[p][nt], b1[p][nt], Vp + p * kPlane + jrow * kVB + 8 * nt);
    constexpr int PA[6] = {2, 0, 1, 1, 0, 0}, PB[6] = {0, 2, 1, 0, 1, 0};
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mma16816(o[nt], a[PA[q]], b0[PB[q]][nt], b1[PB[q]][nt]);
  }
  // ---- combine the two key halves, write the merged context
  float* my = part + rg * 16 * (kDH + 4);
  if (kh == 1) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int d = 8 * nt + 2 * tq;
      *reinterpret_cast<float2*>(my + gq * (kDH + 4) + d) = make_float2(o[nt][0], o[nt][1]);
      *reinterpret_cast<float2*>(my + (gq + 8) * (kDH + 4) + d) = make_float2(o[nt][2], o[nt][3]);
    }
  }
  __syncthreads();
  if (kh == 0) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int d = 8 * nt + 2 * tq;
      const float2 u = *reinterpret_cast<const float2*>(my + gq * (kDH + 4) + d);
      const float2 v = *reinterpret_cast<const float2*>(my + (gq + 8) * (kDH + 4) + d);
      if (r0 < T)
      {
        *reinterpret_cast<float2*>(ctx + (rbase + r0) * H + hoff + d) = make_float2(o[nt][0] + u.x, o[nt][1] + u.y);
        if (xp) planes_store2f(o[nt][0] + u.x, o[nt][1] + u.y, xp, MH, (rbase + r0) * H + hoff + d, pf);
      }
      if (r1 < T)
      {
        *reinterpret_cast<float2*>(ctx + (rbase + r1) * H + hoff + d) = make_float2(o[nt][2] + v.x, o[nt][3] + v.y);
        if (xp) planes_store2f(o[nt][2] + v.x, o[nt][3] + v.y, xp, MH, (rbase + r1) * H + hoff + d, pf);
      }
    }
  }
}

// ------------------------------------------------------------------ tcgen05 forward (T <= 128)
// grid (B * h); one CTA = one head, 256 threads.  q, k, v (fp32 + bias) are
// split into three bf16 planes each straight into shared memory in the
// canonical no-swizzle layouts the tensor core reads through descriptors:
// q, k K-major (8-row x 16-byte core matrices, K chunks 128 B apart, row
// groups 1 KB apart), v MN-major (8-key x 8-dim core matrices: head dims
// contiguous, so a thread's 8 dims are one 16-byte store).  One thread issues
// S = q k^T as 4 K-steps x the six split products that carry fp32 accuracy,
// `tcgen05.mma` M = 128, N = 128, K = 16, into two TMEM accumulators (hh
// alone, the five small terms together, as the dense GEMM); every thread
// then owns one row of S (TMEM lane = row; warps w and w + 4 the two column
// halves): scale, max, exp, sum, IEEE divide and code rounding as the
// one-head kernels, probability codes stored 16 bytes at a time, p split
// into planes over the q | k space, and ctx = p v as 8 K-steps x 6 products
// (M = 128, N = 64) into two more accumulators, read back row by row.
constexpr int kT5 = 512;                     // 16 warps: lanes 32 (w % 4).., column quarter w / 4
constexpr uint32_t kQKPlane = 128 * kDH * 2;             // 16 KB: 128 rows x 64 bf16
constexpr uint32_t kVPlane = kDH * 128 * 2;              // 16 KB: 64 dims x 128 keys
constexpr uint32_t kPPlane = 128 * 128 * 2;              // 32 KB: 128 rows x 128 keys
constexpr size_t kFwd5Smem = 1024 + 9 * size_t(kQKPlane) + 8 * 128 * sizeof(float) + 64;

// fixed_code for a probability (>= 0, or NaN -> 0): round half away from
// zero of v >= 0 is t + (v - t >= 0.5) with t = trunc(v) (v - t exact)
__device__ __forceinline__ uint32_t prob_code(float p, float qs, float hi) {
  const float v = p * qs;
  const float t = truncf(v);
  const float r = fminf(t + ((v - t >= 0.5f) ? 1.f : 0.f), hi);
  return v >= 0.f ? static_cast<uint32_t>(r) : 0u;
}

__device__ __forceinline__ uint32_t prob_codes4(float a, float b, float c, float d, float qs, float hi) {
  return prob_code(a, qs, hi) | (prob_code(b, qs, hi) << 8) | (prob_code(c, qs, hi) << 16) |
         (prob_code(d, qs, hi) << 24);
}

__device__ __forceinline__ uint64_t desc_nosw(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (static_cast<uint64_t>(1) << 46);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait5(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void tmem_ld32x(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 8 consecutive fp32 values -> three 16-byte bf16 plane chunks at smem byte
// offsets o, o + plane, o + 2 plane
__device__ __forceinline__ void split8_smem(const float* v, unsigned char* base, uint32_t o, uint32_t plane) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split_pair(v[2 * j], v[2 * j + 1], h[j], m[j], l[j]);
  *reinterpret_cast<uint4*>(base + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + plane + o) = make_uint4(m[0], m[1], m[2], m[3]);
  *reinterpret_cast<uint4*>(base + 2 * plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void __launch_bounds__(kT5, 1) k_attn_fwd_tc5(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint8_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (sbase - raw);
  // [Q 3 planes | K 3 planes | V 3 planes] (P's 3 planes later over Q | K), reductions, barriers
  const uint32_t sQ = sbase, sK = sbase + 3 * kQKPlane, sV = sbase + 6 * kQKPlane, sP = sbase;
  unsigned char* gQ = gbase;
  unsigned char* gK = gbase + 3 * kQKPlane;
  unsigned char* gV = gbase + 6 * kQKPlane;
  unsigned char* gP = gbase;
  float* redm = reinterpret_cast<float*>(gbase + 9 * kQKPlane);   // [4][128]
  float* reds = redm + 512;                                       // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reds + 512);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const uint32_t barS = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  const uint32_t barC = barS + 8;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.x / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barS));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barC));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- loads: thread = (row t = tid & 127, head dims [16 (tid >> 7), +16)); bias, codes, planes
  {
    const int t = tid & 127, d0 = 16 * (tid >> 7);
    const bool ok = t < T;
    float4 raw[3][4];                                    // every load of the thread in flight at once
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float* src = y3 + m * MH + (rbase + t) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        raw[m][c] = ok ? __ldg(reinterpret_cast<const float4*>(src) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float* bsrc = (m == 0 ? bq : m == 1 ? bk : bv) + hoff + d0;
      float x[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bsrc) + c);
        const float4 v = raw[m][c];
        x[4 * c] = ok ? v.x + bb.x : 0.f;
        x[4 * c + 1] = ok ? v.y + bb.y : 0.f;
        x[4 * c + 2] = ok ? v.z + bb.z : 0.f;
        x[4 * c + 3] = ok ? v.w + bb.w : 0.f;
      }
      if (ok) {
        uint32_t* codes = (m == 0 ? qc : m == 1 ? kc : vc) + (cbase + t) * (kDH / 4) + d0 / 4;
        *reinterpret_cast<uint4*>(codes) =
            make_uint4(codes4(make_float4(x[0], x[1], x[2], x[3]), qs, lo, hi),
                       codes4(make_float4(x[4], x[5], x[6], x[7]), qs, lo, hi),
                       codes4(make_float4(x[8], x[9], x[10], x[11]), qs, lo, hi),
                       codes4(make_float4(x[12], x[13], x[14], x[15]), qs, lo, hi));
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {                      // 8 dims per chunk
        const int d = d0 + 8 * c;
        if (m < 2) {                                     // K-major: (row/8) 1 KB, (d/8) 128 B, (row%8) 16 B
          const uint32_t o = (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u;
          split8_smem(x + 8 * c, m == 0 ? gQ : gK, o, kQKPlane);
        } else {                                         // MN-major: (d/8) 2 KB, (key/8) 128 B, (key%8) 16 B
          const uint32_t o = (d >> 3) * 2048u + (t >> 3) * 128u + (t & 7) * 16u;
          split8_smem(x + 8 * c, gV, o, kVPlane);
        }
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t accS0 = tmem, accS1 = tmem + 128, accC0 = tmem + 256, accC1 = tmem + 320;
  constexpr uint32_t kIdS = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t kIdC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
    // S = q k^T: K = 64 head dims in 4 steps of 16 (two 128-byte K chunks each)
#pragma unroll
    for (int ks = 0; ks < kDH / 16; ++ks) {
      const uint32_t off = ks * 256u;
      uint64_t a[3], bb[3];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        a[p] = desc_nosw(sQ + p * kQKPlane + off, 128, 1024);
        bb[p] = desc_nosw(sK + p * kQKPlane + off, 128, 1024);
      }
      const uint32_t acc = ks != 0;
      umma(accS0, a[0], bb[0], kIdS, acc);
      umma(accS1, a[0], bb[1], kIdS, acc);
      umma(accS1, a[1], bb[0], kIdS, 1);
      umma(accS1, a[1], bb[1], kIdS, 1);
      umma(accS1, a[0], bb[2], kIdS, 1);
      umma(accS1, a[2], bb[0], kIdS, 1);
    }
    umma_commit(barS);
  }
  __syncwarp();
  mbar_wait5(barS, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- softmax: thread = row r (TMEM lane), columns [32 qt, +32)
  const int r = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;
  const uint32_t lane_addr = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  float s[32];
  {
    float a1[32];
    tmem_ld32x(accS0 + lane_addr + 32 * qt, s);
    tmem_ld32x(accS1 + lane_addr + 32 * qt, a1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) s[j] += a1[j];
  }
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int key = 32 * qt + j;
    s[j] = key < T ? __fmul_rn(s[j], scale) : -INFINITY;
    mx = fmaxf(mx, s[j]);
  }
  redm[qt * 128 + r] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(redm[r], redm[128 + r]), fmaxf(redm[256 + r], redm[384 + r]));
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int key = 32 * qt + j;
    s[j] = key < T ? expf(s[j] - mx) : 0.f;
    sum += s[j];
  }
  reds[qt * 128 + r] = sum;
  __syncthreads();
  sum = (reds[r] + reds[128 + r]) + (reds[256 + r] + reds[384 + r]);
  // p, its codes (16 bytes per store when the row allows), its planes over q | k
  // (the S products are complete: barS)
#pragma unroll
  for (int j = 0; j < 32; ++j) s[j] = __fdiv_rn(s[j], sum);
  if (r < T) {
    uint8_t* prow = pc + (cbase + r) * T + 32 * qt;
    const int nk = min(32, T - 32 * qt);
    if ((T & 15) == 0 && nk == 32) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t w4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w4[q] = prob_codes4(s[16 * c + 4 * q], s[16 * c + 4 * q + 1], s[16 * c + 4 * q + 2],
                              s[16 * c + 4 * q + 3], qs, hi);
        *reinterpret_cast<uint4*>(prow + 16 * c) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)                           // static indices: s stays in registers
        if (j < nk) prow[j] = static_cast<uint8_t>(prob_code(s[j], qs, hi));
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {                              // K-major P: (row/8) 2 KB, (key/8) 128 B
    const int key = 32 * qt + 8 * c;
    const uint32_t o = (r >> 3) * 2048u + (key >> 3) * 128u + (r & 7) * 16u;
    split8_smem(s + 8 * c, gP, o, kPPlane);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    // ctx = p v: K = 128 keys in 8 steps of 16
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t off = ks * 256u;
      uint64_t a[3], bb[3];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        a[p] = desc_nosw(sP + p * kPPlane + off, 128, 2048);
        bb[p] = desc_nosw(sV + p * kVPlane + off, 128, 2048);
      }
      const uint32_t acc = ks != 0;
      umma(accC0, a[0], bb[0], kIdC, acc);
      umma(accC1, a[0], bb[1], kIdC, acc);
      umma(accC1, a[1], bb[0], kIdC, 1);
      umma(accC1, a[1], bb[1], kIdC, 1);
      umma(accC1, a[0], bb[2], kIdC, 1);
      umma(accC1, a[2], bb[0], kIdC, 1);
    }
    umma_commit(barC);
  }
  __syncwarp();
  mbar_wait5(barC, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ctx rows through shared memory (over the P planes: the products are
  // complete) so that warps store whole 256-byte rows, fp32 and planes
  float* cs = reinterpret_cast<float*>(gP);                 // [128][kDH + 4]
  {
    uint32_t u0[16], u1[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u0[0]), "=r"(u0[1]), "=r"(u0[2]), "=r"(u0[3]), "=r"(u0[4]), "=r"(u0[5]), "=r"(u0[6]), "=r"(u0[7]),
          "=r"(u0[8]), "=r"(u0[9]), "=r"(u0[10]), "=r"(u0[11]), "=r"(u0[12]), "=r"(u0[13]), "=r"(u0[14]), "=r"(u0[15])
        : "r"(accC0 + lane_addr + 16 * qt));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u1[0]), "=r"(u1[1]), "=r"(u1[2]), "=r"(u1[3]), "=r"(u1[4]), "=r"(u1[5]), "=r"(u1[6]), "=r"(u1[7]),
          "=r"(u1[8]), "=r"(u1[9]), "=r"(u1[10]), "=r"(u1[11]), "=r"(u1[12]), "=r"(u1[13]), "=r"(u1[14]), "=r"(u1[15])
        : "r"(accC1 + lane_addr + 16 * qt));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 16 * qt + j) =
          make_float4(__uint_as_float(u0[j]) + __uint_as_float(u1[j]), __uint_as_float(u0[j + 1]) + __uint_as_float(u1[j + 1]),
                      __uint_as_float(u0[j + 2]) + __uint_as_float(u1[j + 2]), __uint_as_float(u0[j + 3]) + __uint_as_float(u1[j + 3]));
  }
  __syncthreads();
  // warp w stores rows w, w + 16, ...: lane l writes dims [4 (l & 15), +4) of row (l >> 4)
  for (int rr = 2 * warp + ((tid & 31) >> 4); rr < T; rr += 2 * (kT5 / 32)) {
    const int d = 4 * (tid & 15);
    const float4 o = *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
    const int64_t go = (rbase + rr) * H + hoff + d;
    *reinterpret_cast<float4*>(ctx + go) = o;
    if (xp) planes_store4f(o, xp, MH, go, pf);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------ tcgen05 forward, fp16 planes (T <= 128)
// The one-head forward with the f16x3 operand form of the dense products:
// q, k, v (+ bias) and p split into two fp16 planes each (x = hi + 2^-11 lo,
// 22 significant bits; q/k/v/p are far below fp16's range), S = q k^T and
// ctx = p v as three MMAs per K step (hh into one TMEM accumulator, hl + lh
// into the other).  Half the shared memory of the bf16 form (100 KB) and
// 256 TMEM columns (the context accumulators reuse the score columns once
// every thread holds its row of S in registers), so two CTAs share an SM
// and one head's loads and MMA waits overlap the other's softmax.  256
// threads: warp w owns TMEM lanes 32 (w % 4).. (rows) and column half w / 4.
constexpr int kTH = 256;
constexpr uint32_t kHPlane = 128 * kDH * 2;               // 16 KB: 128 rows x 64 fp16
constexpr uint32_t kHPPlane = 128 * 128 * 2;              // 32 KB: p, 128 rows x 128 keys
constexpr size_t kFwdHSmem = 1024 + 6 * size_t(kHPlane) + 4 * 128 * sizeof(float) + 64;
static_assert(2 * kHPPlane <= 4 * kHPlane, "p planes fit over q | k");

__device__ __forceinline__ void split8_smem_h(const float* v, unsigned char* base, uint32_t o, uint32_t plane) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split_pair2h(v[2 * j], v[2 * j + 1], h[j], l[j]);
  *reinterpret_cast<uint4*>(base + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void __launch_bounds__(kTH, 2) k_attn_fwd_tc5h(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint8_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (sbase - raw);
  // [Q 2 planes | K 2 planes | V 2 planes] (P's 2 planes later over Q | K), reductions, barriers
  const uint32_t sQ = sbase, sK = sbase + 2 * kHPlane, sV = sbase + 4 * kHPlane, sP = sbase;
  unsigned char* gQ = gbase;
  unsigned char* gK = gbase + 2 * kHPlane;
  unsigned char* gV = gbase + 4 * kHPlane;
  unsigned char* gP = gbase;
  float* redm = reinterpret_cast<float*>(gbase + 6 * kHPlane);   // [2][128]
  float* reds = redm + 256;                                      // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reds + 256);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const uint32_t barS = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  const uint32_t barC = barS + 8;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.x / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barS));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barC));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- loads: thread = (row t = tid & 127, head dims [32 (tid >> 7), +32)); bias, codes, planes
  {
    const int t = tid & 127, d0 = 32 * (tid >> 7);
    const bool ok = t < T;
#pragma unroll 1
    for (int m = 0; m < 3; ++m) {
      const float* src = y3 + m * MH + (rbase + t) * H + hoff + d0;
      const float* bsrc = (m == 0 ? bq : m == 1 ? bk : bv) + hoff + d0;
      float x[32];
      float4 raw4[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        raw4[c] = ok ? __ldg(reinterpret_cast<const float4*>(src) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(bsrc) + c);
        x[4 * c] = ok ? raw4[c].x + bb.x : 0.f;
        x[4 * c + 1] = ok ? raw4[c].y + bb.y : 0.f;
        x[4 * c + 2] = ok ? raw4[c].z + bb.z : 0.f;
        x[4 * c + 3] = ok ? raw4[c].w + bb.w : 0.f;
      }
      if (ok) {
        uint32_t* codes = (m == 0 ? qc : m == 1 ? kc : vc) + (cbase + t) * (kDH / 4) + d0 / 4;
#pragma unroll
        for (int c = 0; c < 2; ++c)
          *reinterpret_cast<uint4*>(codes + 4 * c) =
              make_uint4(codes4(make_float4(x[16 * c], x[16 * c + 1], x[16 * c + 2], x[16 * c + 3]), qs, lo, hi),
                         codes4(make_float4(x[16 * c + 4], x[16 * c + 5], x[16 * c + 6], x[16 * c + 7]), qs, lo, hi),
                         codes4(make_float4(x[16 * c + 8], x[16 * c + 9], x[16 * c + 10], x[16 * c + 11]), qs, lo, hi),
                         codes4(make_float4(x[16 * c + 12], x[16 * c + 13], x[16 * c + 14], x[16 * c + 15]), qs, lo,
                                hi));
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {                      // 8 dims per chunk
        const int d = d0 + 8 * c;
        if (m < 2) {                                     // K-major: (row/8) 1 KB, (d/8) 128 B, (row%8) 16 B
          const uint32_t o = (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u;
          split8_smem_h(x + 8 * c, m == 0 ? gQ : gK, o, kHPlane);
        } else {                                         // MN-major: (d/8) 2 KB, (key/8) 128 B, (key%8) 16 B
          const uint32_t o = (d >> 3) * 2048u + (t >> 3) * 128u + (t & 7) * 16u;
          split8_smem_h(x + 8 * c, gV, o, kHPlane);
        }
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t accS0 = tmem, accS1 = tmem + 128, accC0 = tmem, accC1 = tmem + 64;
  // kind::f16 with fp16 A and B (formats 0)
  constexpr uint32_t kIdS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  constexpr uint32_t kIdC = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  if (tid == 0) {
#pragma unroll
    for (int ks = 0; ks < kDH / 16; ++ks) {
      const uint32_t off = ks * 256u;
      const uint64_t ah = desc_nosw(sQ + off, 128, 1024), al = desc_nosw(sQ + kHPlane + off, 128, 1024);
      const uint64_t bh_ = desc_nosw(sK + off, 128, 1024), bl = desc_nosw(sK + kHPlane + off, 128, 1024);
      const uint32_t acc = ks != 0;
      umma(accS0, ah, bh_, kIdS, acc);
      umma(accS1, ah, bl, kIdS, acc);
      umma(accS1, al, bh_, kIdS, 1);
    }
    umma_commit(barS);
  }
  __syncwarp();
  mbar_wait5(barS, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- softmax: thread = row r (TMEM lane), columns [64 ch, +64)
  const int r = 32 * (warp & 3) + (tid & 31), ch = warp >> 2;
  const uint32_t lane_addr = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  float s[64];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float a0[32], a1[32];
    tmem_ld32x(accS0 + lane_addr + 64 * ch + 32 * half, a0);
    tmem_ld32x(accS1 + lane_addr + 64 * ch + 32 * half, a1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) s[32 * half + j] = __fmaf_rn(0x1p-11f, a1[j], a0[j]);
  }
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const int key = 64 * ch + j;
    s[j] = key < T ? __fmul_rn(s[j], scale) : -INFINITY;
    mx = fmaxf(mx, s[j]);
  }
  redm[ch * 128 + r] = mx;
  __syncthreads();
  mx = fmaxf(redm[r], redm[128 + r]);
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const int key = 64 * ch + j;
    s[j] = key < T ? expf(s[j] - mx) : 0.f;
    if (j < 32) sum0 += s[j];
    else sum1 += s[j];
  }
  reds[ch * 128 + r] = sum0 + sum1;
  __syncthreads();
  const float sum = reds[r] + reds[128 + r];
#pragma unroll
  for (int j = 0; j < 64; ++j) s[j] = __fdiv_rn(s[j], sum);
  if (r < T) {
    uint8_t* prow = pc + (cbase + r) * T + 64 * ch;
    const int nk = min(64, T - 64 * ch);
    if ((T & 15) == 0 && nk == 64) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t w4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w4[q] = prob_codes4(s[16 * c + 4 * q], s[16 * c + 4 * q + 1], s[16 * c + 4 * q + 2],
                              s[16 * c + 4 * q + 3], qs, hi);
        *reinterpret_cast<uint4*>(prow + 16 * c) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 64; ++j)                           // static indices: s stays in registers
        if (j < nk) prow[j] = static_cast<uint8_t>(prob_code(s[j], qs, hi));
    }
  }
  // every thread's S reads are complete (its wait::ld above); the barrier
  // below also orders them before the context MMAs reuse the columns
#pragma unroll
  for (int c = 0; c < 8; ++c) {                              // K-major P: (row/8) 2 KB, (key/8) 128 B
    const int key = 64 * ch + 8 * c;
    const uint32_t o = (r >> 3) * 2048u + (key >> 3) * 128u + (r & 7) * 16u;
    split8_smem_h(s + 8 * c, gP, o, kHPPlane);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const uint32_t off = ks * 256u;
      const uint64_t ah = desc_nosw(sP + off, 128, 2048), al = desc_nosw(sP + kHPPlane + off, 128, 2048);
      const uint64_t bh_ = desc_nosw(sV + off, 128, 2048), bl = desc_nosw(sV + kHPlane + off, 128, 2048);
      const uint32_t acc = ks != 0;
      umma(accC0, ah, bh_, kIdC, acc);
      umma(accC1, ah, bl, kIdC, acc);
      umma(accC1, al, bh_, kIdC, 1);
    }
    umma_commit(barC);
  }
  __syncwarp();
  mbar_wait5(barC, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ctx rows through shared memory (over the P planes: the products are
  // complete) so that warps store whole 256-byte rows, fp32 and planes
  float* cs = reinterpret_cast<float*>(gP);                 // [128][kDH + 4]
  {
    float u0[32], u1[32];
    tmem_ld32x(accC0 + lane_addr + 32 * ch, u0);
    tmem_ld32x(accC1 + lane_addr + 32 * ch, u1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 32 * ch + j) =
          make_float4(__fmaf_rn(0x1p-11f, u1[j], u0[j]), __fmaf_rn(0x1p-11f, u1[j + 1], u0[j + 1]),
                      __fmaf_rn(0x1p-11f, u1[j + 2], u0[j + 2]), __fmaf_rn(0x1p-11f, u1[j + 3], u0[j + 3]));
  }
  __syncthreads();
  // warp w stores rows w, w + 16, ...: lane l writes dims [4 (l & 15), +4) of row (l >> 4)
  for (int rr = 2 * warp + ((tid & 31) >> 4); rr < T; rr += 2 * (kTH / 32)) {
    const int d = 4 * (tid & 15);
    const float4 o = *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
    const int64_t go = (rbase + rr) * H + hoff + d;
    if (ctx) *reinterpret_cast<float4*>(ctx + go) = o;   // NULL: planes only
    if (xp) planes_store4f(o, xp, MH, go, pf);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ------------------------------------------------------------------ tcgen05 forward, query-tiled (T <= 384)
// grid (ceil(T / 128), B * h); one CTA = 128 query rows of one head, 512
// threads.  Shared memory: the q tile's three bf16 planes (48 KB) and all
// keys' planes (T16 = T rounded up to 16 keys; K-major as the one-head
// kernel, 16 KB per 128 keys and plane).  S = q k^T runs in key blocks of
// 128: the hi x hi product into the block's TMEM columns [128 j, +N_j), the
// five small terms into a 128-column scratch at [384, 512); every thread
// then adds its row's quarter of the scratch onto the block (tcgen05.ld /
// tcgen05.st), scaled and masked, tracking the row maximum -- TMEM ends up
// holding the whole 128 x T16 score tile in fp32 with the same two-
// accumulator precision as the one-head kernel.  Exp-sum is a second pass
// over TMEM; the third pass recomputes each probability (same expf, IEEE
// divide), stores its code and writes p's planes for 32 keys at a time into
// one of two 24 KB buffers over the q planes, and one thread runs
// ctx += p v for those keys (v's planes MN-major over the k planes) while
// the next 32 keys are prepared.  ctx accumulators (hh | small terms) take
// the scratch columns once S is complete.  Codes: every CTA writes q, k, v
// codes for the rows of its own tile range.
constexpr int kT5W = 384;                                  // max T of the query-tiled tcgen05 forward
constexpr uint32_t kW5PPlane = 128 * 32 * 2;               // p planes for 32 keys: 8 KB
__host__ __device__ constexpr size_t fwd5w_smem(int t16) {
  return 1024 + 3 * size_t(kQKPlane) + 3 * size_t(t16) * 128 + 8 * 128 * sizeof(float) + 64;
}

__device__ __forceinline__ void tmem_st32x(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t u[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(u[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t u[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(u[i]);
}

__device__ __forceinline__ void tc_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// one (row, 16-dim quarter) item of projection m: fp32 + bias -> codes (rows
// in [c0, c1)) and three bf16 planes; K-major (q, k) or MN-major (v, key
// groups `vsbo` bytes apart per 8 dims)
__device__ __forceinline__ void stage5_item(const float4 (&raw)[4], const float* __restrict__ bias, int row,
                                            bool ok, bool code, uint32_t* __restrict__ codes, float qs, float lo,
                                            float hi, int d0, unsigned char* base, uint32_t plane, bool mn,
                                            uint32_t vsbo) {
  float x[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 bb = __ldg(reinterpret_cast<const float4*>(bias) + c);
    x[4 * c] = ok ? raw[c].x + bb.x : 0.f;
    x[4 * c + 1] = ok ? raw[c].y + bb.y : 0.f;
    x[4 * c + 2] = ok ? raw[c].z + bb.z : 0.f;
    x[4 * c + 3] = ok ? raw[c].w + bb.w : 0.f;
  }
  if (ok && code)
    *reinterpret_cast<uint4*>(codes) =
        make_uint4(codes4(make_float4(x[0], x[1], x[2], x[3]), qs, lo, hi),
                   codes4(make_float4(x[4], x[5], x[6], x[7]), qs, lo, hi),
                   codes4(make_float4(x[8], x[9], x[10], x[11]), qs, lo, hi),
                   codes4(make_float4(x[12], x[13], x[14], x[15]), qs, lo, hi));
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int d = d0 + 8 * c;
    const uint32_t o = mn ? (d >> 3) * vsbo + (row >> 3) * 128u + (row & 7) * 16u
                          : (row >> 3) * 1024u + (d >> 3) * 128u + (row & 7) * 16u;
    split8_smem(x + 8 * c, base, o, plane);
  }
}

__global__ void __launch_bounds__(kT5, 1) k_attn_fwd_tc5w(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint8_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (sbase - raw);
  const int T16 = (T + 15) & ~15;
  const uint32_t KPL = static_cast<uint32_t>(T16) * 128u;            // one k (or v) plane
  const uint32_t sQ = sbase, sK = sbase + 3 * kQKPlane;
  unsigned char* gQ = gbase;
  unsigned char* gK = gbase + 3 * kQKPlane;
  float* redm = reinterpret_cast<float*>(gK + 3 * KPL);              // [4][128]
  float* reds = redm + 512;                                          // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reds + 512);          // S, P0, P1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
  const uint32_t barS = static_cast<uint32_t>(__cvta_generic_to_shared(bars));

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int q0 = blockIdx.x * 128;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.y / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const int c1 = min(T, q0 + 128);                                   // code rows [q0, c1)

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barS + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- q tile and all keys: thread = (row 128 m + (tid & 127), dims [16 (tid >> 7), +16))
  const int t7 = tid & 127, d0 = 16 * (tid >> 7);
  const int nkm = (T16 + 127) >> 7;                                  // 128-row groups of keys (<= 3)
  {
    float4 rq[4], rk[3][4];
    const int tq = q0 + t7;
    {
      const float* src = y3 + (rbase + tq) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rq[c] = tq < T ? __ldg(reinterpret_cast<const float4*>(src) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      const float* src = y3 + MH + (rbase + t) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rk[m][c] = (m < nkm && t < T) ? __ldg(reinterpret_cast<const float4*>(src) + c)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < nkm && t < T) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + MH));   // v, later
    }
    stage5_item(rq, bq + hoff + d0, t7, tq < T, true, qc + (cbase + tq) * (kDH / 4) + d0 / 4, qs, lo, hi, d0,
                gQ, kQKPlane, false, 0);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm && t < T16)
        stage5_item(rk[m], bk + hoff + d0, t, t < T, t >= q0 && t < c1, kc + (cbase + t) * (kDH / 4) + d0 / 4, qs,
                    lo, hi, d0, gK, KPL, false, 0);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t accX = tmem + 384;                                  // S small terms, then ctx
  const uint32_t accC0 = tmem + 384, accC1 = tmem + 448;
  constexpr uint32_t kIdC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const int r = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;        // TMEM lane = row; column quarter
  const uint32_t lane_addr = static_cast<uint32_t>(32 * (warp & 3)) << 16;

  // ---- S in key blocks of 128, two accumulators, combined in place
  float mx = -INFINITY;
  for (int j = 0; j < nkm; ++j) {
    const int nj = min(128, T16 - 128 * j);
    if (tid == 0) {
      const uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(nj) >> 3) << 17) |
                           ((128u >> 4) << 24);
#pragma unroll
      for (int ks = 0; ks < kDH / 16; ++ks) {
        const uint32_t off = ks * 256u;
        uint64_t a[3], bb[3];
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          a[p] = desc_nosw(sQ + p * kQKPlane + off, 128, 1024);
          bb[p] = desc_nosw(sK + p * KPL + j * 16384u + off, 128, 1024);
        }
        const uint32_t acc = ks != 0;
        umma(tmem + 128 * j, a[0], bb[0], idS, acc);
        umma(accX, a[0], bb[1], idS, acc);
        umma(accX, a[1], bb[0], idS, 1);
        umma(accX, a[1], bb[1], idS, 1);
        umma(accX, a[0], bb[2], idS, 1);
        umma(accX, a[2], bb[0], idS, 1);
      }
      umma_commit(barS);
    }
    __syncwarp();
    mbar_wait5(barS, j & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (32 * qt < nj) {                                              // warp-uniform
      float a0[32], a1[32];
      tmem_ld32x(tmem + lane_addr + 128 * j + 32 * qt, a0);
      tmem_ld32x(accX + lane_addr + 32 * qt, a1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int key = 128 * j + 32 * qt + i;
        a0[i] = key < T ? __fmul_rn(a0[i] + a1[i], scale) : -INFINITY;
        mx = fmaxf(mx, a0[i]);
      }
      tmem_st32x(tmem + lane_addr + 128 * j + 32 * qt, a0);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_sync();                                                       // scratch free for the next block
  }
  // ---- row max and exp-sum over the four column quarters
  redm[qt * 128 + r] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(redm[r], redm[128 + r]), fmaxf(redm[256 + r], redm[384 + r]));
  float sum = 0.f;
  for (int j = 0; j < nkm; ++j) {
    if (32 * qt < min(128, T16 - 128 * j)) {
      float a0[32];
      tmem_ld32x(tmem + lane_addr + 128 * j + 32 * qt, a0);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int key = 128 * j + 32 * qt + i;
        sum += key < T ? expf(a0[i] - mx) : 0.f;
      }
    }
  }
  reds[qt * 128 + r] = sum;
  // ---- v planes over the k planes (S is complete: its last wait above)
  {
    const uint32_t vsbo = static_cast<uint32_t>(T16) * 16u;
    float4 rv[3][4];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      const float* src = y3 + 2 * MH + (rbase + t) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rv[m][c] = (m < nkm && t < T) ? __ldg(reinterpret_cast<const float4*>(src) + c)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm && t < T16)
        stage5_item(rv[m], bv + hoff + d0, t, t < T, t >= q0 && t < c1, vc + (cbase + t) * (kDH / 4) + d0 / 4, qs,
                    lo, hi, d0, gK, KPL, true, vsbo);
    }
  }
  __syncthreads();
  sum = (reds[r] + reds[128 + r]) + (reds[256 + r] + reds[384 + r]);
  // ---- p: codes, planes for 32 keys at a time, ctx += p v on the tensor cores
  const int rg = q0 + r;
  uint8_t* prow = pc + (cbase + rg) * T;
  const int nch = (T16 + 31) >> 5;
  for (int c = 0; c < nch; ++c) {
    const int key0 = 32 * c + 8 * qt;
    float p[8];
    tmem_ld8(tmem + lane_addr + key0, p);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = key0 + i < T ? __fdiv_rn(expf(p[i] - mx), sum) : 0.f;
    if (rg < T) {
      if ((T & 7) == 0 && key0 + 8 <= T) {
        *reinterpret_cast<uint2*>(prow + key0) =
            make_uint2(prob_codes4(p[0], p[1], p[2], p[3], qs, hi), prob_codes4(p[4], p[5], p[6], p[7], qs, hi));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (key0 + i < T) prow[key0 + i] = static_cast<uint8_t>(prob_code(p[i], qs, hi));
      }
    }
    const int buf = c & 1;
    if (c >= 2) mbar_wait5(barS + 8 * (1 + buf), ((c - 2) >> 1) & 1);   // chunk c - 2's MMAs read this buffer
    split8_smem(p, gQ + buf * 3 * kW5PPlane, (r >> 3) * 512u + qt * 128u + (r & 7) * 16u, kW5PPlane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_sync();
    if (tid == 0) {
      const int nks = min(2, (T16 - 32 * c) >> 4);
      for (int ks = 0; ks < nks; ++ks) {
        uint64_t a[3], bb[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          a[q] = desc_nosw(sQ + buf * 3 * kW5PPlane + q * kW5PPlane + ks * 256u, 128, 512);
          bb[q] = desc_nosw(sK + q * KPL + c * 512u + ks * 256u, 128, static_cast<uint32_t>(T16) * 16u);
        }
        const uint32_t acc = (c | ks) != 0;
        umma(accC0, a[0], bb[0], kIdC, acc);
        umma(accC1, a[0], bb[1], kIdC, acc);
        umma(accC1, a[1], bb[0], kIdC, 1);
        umma(accC1, a[1], bb[1], kIdC, 1);
        umma(accC1, a[0], bb[2], kIdC, 1);
        umma(accC1, a[2], bb[0], kIdC, 1);
      }
      umma_commit(barS + 8 * (1 + buf));
    }
    __syncwarp();
  }
  mbar_wait5(barS + 8 * (1 + ((nch - 1) & 1)), ((nch - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- ctx rows through shared memory (over the p buffers) as whole 256-byte rows
  float* cs = reinterpret_cast<float*>(gQ);                          // [128][kDH + 4]
  {
    float u0[16], u1[16];
    tmem_ld16(accC0 + lane_addr + 16 * qt, u0);
    tmem_ld16(accC1 + lane_addr + 16 * qt, u1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 16 * qt + j) =
          make_float4(u0[j] + u1[j], u0[j + 1] + u1[j + 1], u0[j + 2] + u1[j + 2], u0[j + 3] + u1[j + 3]);
  }
  __syncthreads();
  for (int rr = 2 * warp + ((tid & 31) >> 4); rr < 128 && q0 + rr < T; rr += 2 * (kT5 / 32)) {
    const int d = 4 * (tid & 15);
    const float4 o = *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
    const int64_t go = (rbase + q0 + rr) * H + hoff + d;
    *reinterpret_cast<float4*>(ctx + go) = o;
    if (xp) planes_store4f(o, xp, MH, go, pf);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------ tcgen05 backward (T <= 128)
// grid (B * h); one CTA = one head, 512 threads.  Shared memory holds g
// split into three bf16 planes and q~, k~, v~, p~ as exact bf16 (8-bit codes
// times 2^-fb), all in no-swizzle layouts built from 8 x 16-byte core
// matrices -- the same bytes read K-major by one descriptor and MN-major by
// another (the two strides swapped), so g serves as the A operand of
// dP = g v~^T and the B operand of dv = p~^T g, and so on.  MMAs (one
// thread; every product two TMEM accumulators: the hi term alone and the
// smaller terms together, as the dense GEMM):
//   dP = g v~^T (M 128 rows, N 128 keys, K 64)  and  dv = p~^T g (M 128 keys, N 64, K 128 rows),
// then every thread owns a quarter row: dS = p~ (dP - sum_j dP p~) scale
// (row sums over the four quarters in shared memory), split into planes
// over the g | v~ | p~ space, then
//   dq = dS k~ (M 128 rows) and dk = dS^T q~ (M 128 keys), N 64, K 128.
// dq, dk, dv leave through shared memory as whole rows of the (B*T, 3H)
// operand.
constexpr uint32_t kB5G = 3 * 128 * kDH * 2;            // g planes (48 KB)
constexpr uint32_t kB5C = 128 * kDH * 2;                // one 128 x 64 bf16 operand (16 KB)
constexpr uint32_t kB5P = 128 * 128 * 2;                // one 128 x 128 bf16 operand (32 KB)
constexpr size_t kBwd5Smem = 1024 + size_t(kB5G) + 3 * kB5C + kB5P + 4 * 128 * sizeof(float) + 64;
static_assert(3 * kB5P <= kB5G + kB5C + kB5P, "dS planes fit over g | v~ | p~");

__device__ __forceinline__ uint64_t desc_ns(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (static_cast<uint64_t>(1) << 46);
}

// 8 consecutive int8 codes -> 16 bytes of exact bf16 (code * inv)
__device__ __forceinline__ uint4 codes8_bf16(uint2 w, float inv) {
  const float4 a = decode4(w.x, inv), b = decode4(w.y, inv);
  return make_uint4(bf2(a.x, a.y), bf2(a.z, a.w), bf2(b.x, b.y), bf2(b.z, b.w));
}

// Persistent: grid min(B h, #SMs), each CTA loops over heads; every thread
// prefetches its own slice of the next head (g row quarter, q~/k~/v~ code
// quarters, p~ code run: 144 bytes) with cp.async into a private staging
// slot while the current head computes (T % 16 == 0; other T load directly).
constexpr int kB5Stage = 144;                               // staged bytes per thread
constexpr size_t kBwd5SmemP = kBwd5Smem + size_t(kT5) * kB5Stage;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

__device__ __forceinline__ void bwd5_prefetch(unsigned char* slot, const float* __restrict__ g,
                                              const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
                                              const uint32_t* __restrict__ vc, const uint8_t* __restrict__ pc,
                                              int T, int h, int bh) {
  const int tid = threadIdx.x, t = tid & 127, qt = tid >> 7;
  const bool ok = t < T;
  const int b = bh / h, hh = bh - b * h, H = h * kDH;
  const int64_t rbase = static_cast<int64_t>(b) * T, cbase = static_cast<int64_t>(bh) * T;
  const int tt = ok ? t : 0;
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(slot));
  const float* gs = g + (rbase + tt) * H + hh * kDH + 16 * qt;
#pragma unroll
  for (int c = 0; c < 4; ++c) cp_async16(d + 16 * c, gs + 4 * c, ok);
#pragma unroll
  for (int m = 0; m < 3; ++m)
    cp_async16(d + 64 + 16 * m, (m == 0 ? qc : m == 1 ? kc : vc) + (cbase + tt) * (kDH / 4) + 4 * qt, ok);
  const bool p0 = ok && 32 * qt + 16 <= T, p1 = ok && 32 * qt + 32 <= T;   // T % 16 == 0: whole chunks
  const uint8_t* prow = pc + (cbase + tt) * T;
  cp_async16(d + 112, prow + (p0 ? 32 * qt : 0), p0);
  cp_async16(d + 128, prow + (p1 ? 32 * qt + 16 : 0), p1);
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(kT5, 1) k_attn_bwd_tc5(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
    const uint32_t* __restrict__ vc, const uint8_t* __restrict__ pc, int T, int h, float scale, float inv,
    float* __restrict__ gcat, int nbh) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gb = smem_raw + (sbase - raw);
  // [ G planes | V | P ] (later the dS planes, later the output staging) | K | Q | row sums | barriers | staging
  const uint32_t sG = sbase, sV = sbase + kB5G, sP = sV + kB5C, sK = sP + kB5P, sQ = sK + kB5C;
  unsigned char* gG = gb;
  unsigned char* gV = gb + kB5G;
  unsigned char* gP = gV + kB5C;
  unsigned char* gK = gP + kB5P;
  unsigned char* gQ = gK + kB5C;
  const uint32_t sS = sbase;                               // dS planes (3 x 32 KB) over G | V | P
  unsigned char* gS = gb;
  float* redt = reinterpret_cast<float*>(gQ + kB5C);      // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(redt + 512);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  unsigned char* slot = gb + (kBwd5Smem - 1024) + static_cast<size_t>(threadIdx.x) * kB5Stage;
  const uint32_t bar1 = static_cast<uint32_t>(__cvta_generic_to_shared(bars)), bar2 = bar1 + 8;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int H = h * kDH;
  const bool staged = (T & 15) == 0;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar2));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (staged && static_cast<int>(blockIdx.x) < nbh) bwd5_prefetch(slot, g, qc, kc, vc, pc, T, h, blockIdx.x);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // instruction descriptors: D f32, A/B bf16, bit 15 A MN-major, bit 16 B MN-major
  constexpr uint32_t kBase = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 4) << 24);
  constexpr uint32_t kIdP = kBase | ((128u >> 3) << 17);                        // g v~^T
  constexpr uint32_t kIdV = kBase | (1u << 15) | (1u << 16) | ((64u >> 3) << 17);  // p~^T g
  constexpr uint32_t kIdQ = kBase | (1u << 16) | ((64u >> 3) << 17);             // dS k~
  constexpr uint32_t kIdK = kBase | (1u << 15) | (1u << 16) | ((64u >> 3) << 17);  // dS^T q~
  const uint32_t tP0 = tmem, tP1 = tmem + 128, tV0 = tmem + 256, tV1 = tmem + 320;
  const uint32_t tQ0 = tmem, tQ1 = tmem + 64, tK0 = tmem + 128, tK1 = tmem + 192;   // over dP, later
  constexpr uint32_t GPL = 128u * kDH * 2;                  // g plane stride (bytes)
  const int r = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;
  const uint32_t la = static_cast<uint32_t>(32 * (warp & 3)) << 16;

  int it = 0;
  for (int bh = blockIdx.x; bh < nbh; bh += gridDim.x, ++it) {
    const int b = bh / h, hh = bh - b * h;
    const int64_t rbase = static_cast<int64_t>(b) * T;
    const int hoff = hh * kDH;
    const int64_t cbase = static_cast<int64_t>(bh) * T;
    // ---- stage: thread = (row t = tid & 127, quarter qt = tid >> 7)
    {
      const int t = tid & 127, qs = tid >> 7;
      const bool ok = t < T;
      float x[16];
      uint4 cw[3];
      uint32_t pw[8];
      if (staged) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = *reinterpret_cast<const float4*>(slot + 16 * c);
          x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
#pragma unroll
        for (int m = 0; m < 3; ++m) cw[m] = *reinterpret_cast<const uint4*>(slot + 64 + 16 * m);
        const uint4 a = *reinterpret_cast<const uint4*>(slot + 112), a2 = *reinterpret_cast<const uint4*>(slot + 128);
        pw[0] = a.x; pw[1] = a.y; pw[2] = a.z; pw[3] = a.w; pw[4] = a2.x; pw[5] = a2.y; pw[6] = a2.z; pw[7] = a2.w;
        // the slot is consumed: the next head's slice flies while this head computes
        if (bh + static_cast<int>(gridDim.x) < nbh) bwd5_prefetch(slot, g, qc, kc, vc, pc, T, h, bh + gridDim.x);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(g + (rbase + t) * H + hoff + 16 * qs) + c)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const uint32_t* src = (m == 0 ? qc : m == 1 ? kc : vc) + (cbase + t) * (kDH / 4) + 4 * qs;
          cw[m] = ok ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0u, 0u, 0u, 0u);
        }
        const uint8_t* prow = pc + (cbase + t) * T + 32 * qs;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint32_t v = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = 32 * qs + 4 * q + e;
            if (ok && key < T) v |= static_cast<uint32_t>(__ldg(prow + 4 * q + e)) << (8 * e);
          }
          pw[q] = v;
        }
      }
      // g: head dims [16 qs, +16) -> planes (64-wide layout: row group 1 KB, dim group 128 B)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int d = 16 * qs + 8 * c;
        split8_smem(x + 8 * c, gG, (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u, 128u * kDH * 2);
      }
      // q~, k~, v~ rows: 16 codes each -> bf16, same 64-wide layout
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        unsigned char* dst = m == 0 ? gQ : m == 1 ? gK : gV;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int d = 16 * qs + 8 * c;
          *reinterpret_cast<uint4*>(dst + (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u) =
              codes8_bf16(c == 0 ? make_uint2(cw[m].x, cw[m].y) : make_uint2(cw[m].z, cw[m].w), inv);
        }
      }
      // p~ row t, keys [32 qs, +32) -> bf16 (128-wide layout: row group 2 KB, key group 128 B)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int key = 32 * qs + 8 * c;
        *reinterpret_cast<uint4*>(gP + (t >> 3) * 2048u + (key >> 3) * 128u + (t & 7) * 16u) =
            codes8_bf16(make_uint2(pw[2 * c], pw[2 * c + 1]), inv);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < kDH / 16; ++ks) {                  // dP: K = head dims
        const uint64_t bv = desc_ns(sV + 256u * ks, 128, 1024);
        umma(tP0, desc_ns(sG + 256u * ks, 128, 1024), bv, kIdP, ks != 0);
        umma(tP1, desc_ns(sG + 2 * GPL + 256u * ks, 128, 1024), bv, kIdP, ks != 0);
        umma(tP1, desc_ns(sG + GPL + 256u * ks, 128, 1024), bv, kIdP, 1);
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {                         // dv: K = rows (16 per step: 2 row groups)
        const uint64_t ap = desc_ns(sP + 4096u * ks, 2048, 128);  // MN-major: K groups 2 KB, M groups 128 B
        umma(tV0, ap, desc_ns(sG + 2048u * ks, 1024, 128), kIdV, ks != 0);
        umma(tV1, ap, desc_ns(sG + 2 * GPL + 2048u * ks, 1024, 128), kIdV, ks != 0);
        umma(tV1, ap, desc_ns(sG + GPL + 2048u * ks, 1024, 128), kIdV, 1);
      }
      umma_commit(bar1);
    }
    __syncwarp();
    mbar_wait5(bar1, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- dS: thread = row r, keys [32 qt, +32)
    float dp[32], pv[32];
    {
      float a0[16], a1[16];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld16(tP0 + la + 32 * qt + 16 * c, a0);
        tmem_ld16(tP1 + la + 32 * qt + 16 * c, a1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) dp[16 * c + j] = a0[j] + a1[j];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 w = *reinterpret_cast<const uint4*>(gP + (r >> 3) * 2048u + ((32 * qt + 8 * c) >> 3) * 128u + (r & 7) * 16u);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        pv[8 * c + 2 * q] = __uint_as_float(ww[q] << 16);
        pv[8 * c + 2 * q + 1] = __uint_as_float(ww[q] & 0xFFFF0000u);
      }
    }
    float part = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) part += __fmul_rn(dp[j], pv[j]);
    redt[qt * 128 + r] = part;
    __syncthreads();                                           // also: dP / dv products done reading g, v~, p~
    const float dt = (redt[r] + redt[128 + r]) + (redt[256 + r] + redt[384 + r]);
#pragma unroll
    for (int j = 0; j < 32; ++j) dp[j] = __fmul_rn(__fmul_rn(pv[j], __fsub_rn(dp[j], dt)), scale);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int key = 32 * qt + 8 * c;
      split8_smem(dp + 8 * c, gS, (r >> 3) * 2048u + (key >> 3) * 128u + (r & 7) * 16u, kB5P);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        // dq = dS k~: A K-major (key groups 128 B, row groups 2 KB); B = k~ MN-major (key groups 1 KB, dim groups 128 B)
        const uint64_t bk = desc_ns(sK + 2048u * ks, 1024, 128);
        umma(tQ0, desc_ns(sS + 256u * ks, 128, 2048), bk, kIdQ, ks != 0);
        umma(tQ1, desc_ns(sS + 2 * kB5P + 256u * ks, 128, 2048), bk, kIdQ, ks != 0);
        umma(tQ1, desc_ns(sS + kB5P + 256u * ks, 128, 2048), bk, kIdQ, 1);
        // dk = dS^T q~: A MN-major (row groups 2 KB, key groups 128 B); B = q~ MN-major
        const uint64_t bq = desc_ns(sQ + 2048u * ks, 1024, 128);
        umma(tK0, desc_ns(sS + 4096u * ks, 2048, 128), bq, kIdK, ks != 0);
        umma(tK1, desc_ns(sS + 2 * kB5P + 4096u * ks, 2048, 128), bq, kIdK, ks != 0);
        umma(tK1, desc_ns(sS + kB5P + 4096u * ks, 2048, 128), bq, kIdK, 1);
      }
      umma_commit(bar2);
    }
    __syncwarp();
    mbar_wait5(bar2, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- dq | dk | dv through shared memory (over the dS planes: the products are done)
    float* cs = reinterpret_cast<float*>(gS);                 // [128][kDH + 4]
#pragma unroll 1
    for (int o = 0; o < 3; ++o) {
      const uint32_t t0 = o == 0 ? tQ0 : o == 1 ? tK0 : tV0, t1 = o == 0 ? tQ1 : o == 1 ? tK1 : tV1;
      float a0[16], a1[16];
      tmem_ld16(t0 + la + 16 * qt, a0);
      tmem_ld16(t1 + la + 16 * qt, a1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 16 * qt + j) =
            make_float4(a0[j] + a1[j], a0[j + 1] + a1[j + 1], a0[j + 2] + a1[j + 2], a0[j + 3] + a1[j + 3]);
      __syncthreads();
      for (int rr = 2 * warp + ((tid & 31) >> 4); rr < T; rr += 2 * (kT5 / 32)) {
        const int d = 4 * (tid & 15);
        *reinterpret_cast<float4*>(gcat + (rbase + rr) * (3 * H) + o * H + hoff + d) =
            *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
      }
      __syncthreads();
    }
    // the next head's MMAs overwrite the accumulators these threads just read
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------ tcgen05 backward, fp16 planes (T <= 128)
// The one-head backward on two fp16 planes per fp32 operand, two CTAs per SM
// (97 KB shared memory, 256 TMEM columns, 256 threads).  g and dS span far
// more than fp16's range: each is scaled by one power of two per head (its
// maximum lands in [2^14, 2^15)) and split as hi = RN_f16(x 2^e), lo =
// RN_f16(x 2^e - hi) -- 22 bits for everything above 2^-14 of the head's
// maximum.  Code operands (q~, k~, v~, p~: 8-bit codes x 2^-fb) are exact in
// fp16.  Every product is two MMAs per K step into ONE accumulator, the
// small terms first: the lo chain over the whole K, then the hi chain on top
// of it -- the accumulator's truncation then acts on the hi additions only,
// as in the two-accumulator form.  Products are scaled back by 2^-e (exact).
// Shared memory: phase 1 [g hi | g lo | v~ | p~ (2 x 16 KB)] + k~ at 80 KB;
// phase 2 [dS hi | dS lo (2 x 32 KB)] + q~ at 64 KB (q~ staged through
// registers while phase 1 runs) + k~.
constexpr uint32_t kHB = 128 * kDH * 2;                   // 16 KB: 128 rows x 64 fp16
constexpr size_t kBwdHSmem = 1024 + 6 * size_t(kHB) + 4 * 128 * sizeof(float) + 64;

__device__ __forceinline__ uint32_t h2u(float a, float b) {   // two exact fp16 (codes) -> packed
  return f16x2_rn(a, b);
}

__device__ __forceinline__ uint4 codes8_f16(uint2 w, float inv) {
  const float4 a = decode4(w.x, inv), b = decode4(w.y, inv);
  return make_uint4(h2u(a.x, a.y), h2u(a.z, a.w), h2u(b.x, b.y), h2u(b.z, b.w));
}

// 8 values (already x 2^e) -> hi / lo (unscaled remainder) fp16 planes
__device__ __forceinline__ void split8_smem_hu(const float* v, unsigned char* base, uint32_t o, uint32_t plane) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    h[j] = f16x2_rn(v[2 * j], v[2 * j + 1]);
    l[j] = f16x2_rn(v[2 * j] - f16_lo_f32(h[j]), v[2 * j + 1] - f16_hi_f32(h[j]));
  }
  *reinterpret_cast<uint4*>(base + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(base + plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ float block_max256(float m, float* red) {
#pragma unroll
  for (int k = 16; k; k >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, k));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kTH, 2) k_attn_bwd_tc5h(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
    const uint32_t* __restrict__ vc, const uint8_t* __restrict__ pc, int T, int h, float scale, float inv,
    float* __restrict__ gcat) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gb = smem_raw + (sbase - raw);
  const uint32_t sG = sbase, sV = sbase + 2 * kHB, sP = sbase + 3 * kHB, sS = sbase;
  const uint32_t sQ = sbase + 4 * kHB, sK = sbase + 5 * kHB;
  unsigned char* gG = gb;
  unsigned char* gV = gb + 2 * kHB;
  unsigned char* gP = gb + 3 * kHB;
  unsigned char* gS = gb;
  unsigned char* gQ = gb + 4 * kHB;
  unsigned char* gK = gb + 5 * kHB;
  float* redt = reinterpret_cast<float*>(gb + 6 * kHB);    // [2][128] + 8 scratch
  uint64_t* bars = reinterpret_cast<uint64_t*>(redt + 512);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const uint32_t bar1 = static_cast<uint32_t>(__cvta_generic_to_shared(bars)), bar2 = bar1 + 8;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.x, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar2));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // ---- stage: thread = (row t = tid & 127, half hq = tid >> 7: dims [32 hq, +32), keys [64 hq, +64))
  const int t = tid & 127, hq = tid >> 7;
  const bool ok = t < T;
  uint4 qreg[2];                                           // q~ codes, staged after phase 1
  float eg_scale;
  {
    float x[32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(g + (rbase + t) * H + hoff + 32 * hq) + c)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
    }
    const uint32_t* qsrc = qc + (cbase + t) * (kDH / 4) + 8 * hq;
    qreg[0] = ok ? __ldg(reinterpret_cast<const uint4*>(qsrc)) : make_uint4(0u, 0u, 0u, 0u);
    qreg[1] = ok ? __ldg(reinterpret_cast<const uint4*>(qsrc) + 1) : make_uint4(0u, 0u, 0u, 0u);
    // k~, v~ rows: 32 codes each -> fp16 (64-wide K-major layout)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const uint32_t* src = (m == 0 ? kc : vc) + (cbase + t) * (kDH / 4) + 8 * hq;
      const uint4 w0 = ok ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0u, 0u, 0u, 0u);
      const uint4 w1 = ok ? __ldg(reinterpret_cast<const uint4*>(src) + 1) : make_uint4(0u, 0u, 0u, 0u);
      unsigned char* dst = m == 0 ? gK : gV;
      const uint2 ww[4] = {make_uint2(w0.x, w0.y), make_uint2(w0.z, w0.w), make_uint2(w1.x, w1.y), make_uint2(w1.z, w1.w)};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int d = 32 * hq + 8 * c;
        *reinterpret_cast<uint4*>(dst + (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u) = codes8_f16(ww[c], inv);
      }
    }
    // p~ row t, keys [64 hq, +64) -> fp16 (128-wide layout: row group 2 KB, key group 128 B)
    {
      const uint8_t* prow = pc + (cbase + t) * T + 64 * hq;
      uint32_t pw[16];
      if (ok && (T & 15) == 0 && 64 * hq + 64 <= T) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 a = __ldg(reinterpret_cast<const uint4*>(prow) + c);
          pw[4 * c] = a.x; pw[4 * c + 1] = a.y; pw[4 * c + 2] = a.z; pw[4 * c + 3] = a.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          uint32_t v = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = 64 * hq + 4 * q + e;
            if (ok && key < T) v |= static_cast<uint32_t>(__ldg(prow + 4 * q + e)) << (8 * e);
          }
          pw[q] = v;
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int key = 64 * hq + 8 * c;
        *reinterpret_cast<uint4*>(gP + (t >> 3) * 2048u + (key >> 3) * 128u + (t & 7) * 16u) =
            codes8_f16(make_uint2(pw[2 * c], pw[2 * c + 1]), inv);
      }
    }
    // g: one power of two per head, then hi / lo planes
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) m = fmaxf(m, fabsf(x[j]));
    int eg;
    eg_scale = row_scale_exp(block_max256(m, redt + 256), eg);
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] *= eg_scale;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int d = 32 * hq + 8 * c;
      split8_smem_hu(x + 8 * c, gG, (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u, kHB);
    }
  }
  const float ginv = 1.0f / eg_scale;                       // exact: a power of two
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // D f32, A/B fp16 (formats 0); bit 15 A MN-major, bit 16 B MN-major
  constexpr uint32_t kBase = (1u << 4) | ((128u >> 4) << 24);
  constexpr uint32_t kIdP = kBase | ((128u >> 3) << 17);                        // g v~^T
  constexpr uint32_t kIdV = kBase | (1u << 15) | (1u << 16) | ((64u >> 3) << 17);  // p~^T g
  constexpr uint32_t kIdQ = kBase | (1u << 16) | ((64u >> 3) << 17);             // dS k~
  constexpr uint32_t kIdK = kBase | (1u << 15) | (1u << 16) | ((64u >> 3) << 17);  // dS^T q~
  const uint32_t tP = tmem, tQ = tmem, tK = tmem + 64, tV = tmem + 128;
  if (tid == 0) {
    // dP: the lo chain over K = 64 head dims, then the hi chain on top
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int ks = 0; ks < kDH / 16; ++ks)
        umma(tP, desc_ns(sG + (pass == 0 ? kHB : 0u) + 256u * ks, 128, 1024), desc_ns(sV + 256u * ks, 128, 1024),
             kIdP, (pass | ks) != 0);
    // dv = p~^T g: K = 128 rows, 16 per step
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        umma(tV, desc_ns(sP + 4096u * ks, 2048, 128), desc_ns(sG + (pass == 0 ? kHB : 0u) + 2048u * ks, 1024, 128),
             kIdV, (pass | ks) != 0);
    umma_commit(bar1);
  }
  __syncwarp();
  mbar_wait5(bar1, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- dS: thread = row r (TMEM lane), keys [64 ch, +64) in two chunks of 32
  const int r = 32 * (warp & 3) + (tid & 31), ch = warp >> 2;
  const uint32_t la = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  auto load_chunk = [&](int c, float (&dp)[32], float (&pv)[32]) {
    tmem_ld32x(tP + la + 64 * ch + 32 * c, dp);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 w = *reinterpret_cast<const uint4*>(gP + (r >> 3) * 2048u + ((64 * ch + 32 * c + 8 * q) >> 3) * 128u +
                                                    (r & 7) * 16u);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        pv[8 * q + 2 * e] = f16_lo_f32(ww[e]);
        pv[8 * q + 2 * e + 1] = f16_hi_f32(ww[e]);
      }
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) dp[j] *= ginv;            // dP itself (exact rescale)
  };
  float part = 0.f;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    float dp[32], pv[32];
    load_chunk(c, dp, pv);
#pragma unroll
    for (int j = 0; j < 32; ++j) part += __fmul_rn(dp[j], pv[j]);
  }
  redt[ch * 128 + r] = part;
  __syncthreads();
  const float dt = redt[r] + redt[128 + r];
  float smax = 0.f;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    float dp[32], pv[32];
    load_chunk(c, dp, pv);
#pragma unroll
    for (int j = 0; j < 32; ++j) smax = fmaxf(smax, fabsf(__fmul_rn(__fmul_rn(pv[j], __fsub_rn(dp[j], dt)), scale)));
  }
  int es;
  const float es_scale = row_scale_exp(block_max256(smax, redt + 256), es);   // (also: p~ reads done)
  float dsv[2][32];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float pv[32];
    load_chunk(c, dsv[c], pv);
#pragma unroll
    for (int j = 0; j < 32; ++j) dsv[c][j] = __fmul_rn(__fmul_rn(pv[j], __fsub_rn(dsv[c][j], dt)), scale) * es_scale;
  }
  __syncthreads();                                           // every p~ read precedes the dS / q~ writes
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int key = 64 * ch + 32 * c + 8 * q;
      split8_smem_hu(dsv[c] + 8 * q, gS, (r >> 3) * 2048u + (key >> 3) * 128u + (r & 7) * 16u, 2 * kHB);
    }
  {                                                          // q~ over p~'s second half
    const uint2 ww[4] = {make_uint2(qreg[0].x, qreg[0].y), make_uint2(qreg[0].z, qreg[0].w),
                         make_uint2(qreg[1].x, qreg[1].y), make_uint2(qreg[1].z, qreg[1].w)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int d = 32 * hq + 8 * c;
      *reinterpret_cast<uint4*>(gQ + (t >> 3) * 1024u + (d >> 3) * 128u + (t & 7) * 16u) = codes8_f16(ww[c], inv);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    // dq = dS k~ (A K-major: key groups 128 B, row groups 2 KB; B = k~ MN-major), lo chain then hi
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        umma(tQ, desc_ns(sS + (pass == 0 ? 2 * kHB : 0u) + 256u * ks, 128, 2048), desc_ns(sK + 2048u * ks, 1024, 128),
             kIdQ, (pass | ks) != 0);
    // dk = dS^T q~ (A MN-major: row groups 2 KB, key groups 128 B; B = q~ MN-major)
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        umma(tK, desc_ns(sS + (pass == 0 ? 2 * kHB : 0u) + 4096u * ks, 2048, 128), desc_ns(sQ + 2048u * ks, 1024, 128),
             kIdK, (pass | ks) != 0);
    umma_commit(bar2);
  }
  __syncwarp();
  mbar_wait5(bar2, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- dq | dk | dv through shared memory (over the dS planes: the products are done)
  float* cs = reinterpret_cast<float*>(gS);                 // [128][kDH + 4]
  const float sinv = 1.0f / es_scale;
#pragma unroll 1
  for (int o = 0; o < 3; ++o) {
    const uint32_t t0 = o == 0 ? tQ : o == 1 ? tK : tV;
    const float f = o == 2 ? ginv : sinv;
    float a0[32];
    tmem_ld32x(t0 + la + 32 * ch, a0);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 32 * ch + j) =
          make_float4(a0[j] * f, a0[j + 1] * f, a0[j + 2] * f, a0[j + 3] * f);
    __syncthreads();
    for (int rr = 2 * warp + ((tid & 31) >> 4); rr < T; rr += 2 * (kTH / 32)) {
      const int d = 4 * (tid & 15);
      *reinterpret_cast<float4*>(gcat + (rbase + rr) * (3 * H) + o * H + hoff + d) =
          *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ------------------------------------------------------------------ tcgen05 forward, query-tiled, fp16 planes
// The query-tiled forward on two fp16 planes per operand.  q (the tile) and
// k (all keys) are scaled by one power of two each (their maxima in
// [2^14, 2^15)) and split as hi = RN_f16(x 2^e), lo = RN_f16(x 2^e - hi), so
// S = q k^T runs as ONE accumulator per key block: the lo chain (hi.lo +
// lo.hi over the 64 head dims) first, the hi.hi chain on top -- the
// accumulator's truncation acts on the hi additions only, as in the
// two-accumulator form, and TMEM holds the score tile with no combine pass.
// p and v use the f16x3 form of the dense products (lo scaled by 2^11, two
// accumulators).  fp16 planes halve the staging and shared memory: 89 KB at
// T = 197, 133 KB at T = 384.
__host__ __device__ constexpr size_t fwd5wh_smem(int t16) {
  return 1024 + 2 * size_t(kHPlane) + 2 * size_t(t16) * 128 + 8 * 128 * sizeof(float) + 64;
}

// q/k/v item: fp32 + bias (in place), its 16 codes for rows in range; returns max |x|
__device__ __forceinline__ float bias_codes16(float4 (&raw)[4], const float* __restrict__ bias, bool ok, bool code,
                                              uint32_t* __restrict__ codes, float qs, float lo, float hi) {
  float m = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 bb = __ldg(reinterpret_cast<const float4*>(bias) + c);
    raw[c] = ok ? make_float4(raw[c].x + bb.x, raw[c].y + bb.y, raw[c].z + bb.z, raw[c].w + bb.w)
                : make_float4(0.f, 0.f, 0.f, 0.f);
    m = fmaxf(m, max4abs(raw[c]));
  }
  if (ok && code)
    *reinterpret_cast<uint4*>(codes) = make_uint4(codes4(raw[0], qs, lo, hi), codes4(raw[1], qs, lo, hi),
                                                  codes4(raw[2], qs, lo, hi), codes4(raw[3], qs, lo, hi));
  return m;
}

__device__ __forceinline__ float block_max512(float m, float* red) {
#pragma unroll
  for (int k = 16; k; k >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, k));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < 16; ++w) r = fmaxf(r, red[w]);
  __syncthreads();
  return r;
}

// 16 values of one row (x 2^e): hi / unscaled-lo fp16 planes, K-major 64-wide layout
__device__ __forceinline__ void split16_kmajor_hu(const float4 (&v)[4], float sc, int row, int d0, unsigned char* base,
                                                  uint32_t plane) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float x[8] = {v[2 * c].x * sc, v[2 * c].y * sc, v[2 * c].z * sc, v[2 * c].w * sc,
                        v[2 * c + 1].x * sc, v[2 * c + 1].y * sc, v[2 * c + 1].z * sc, v[2 * c + 1].w * sc};
    const int d = d0 + 8 * c;
    split8_smem_hu(x, base, (row >> 3) * 1024u + (d >> 3) * 128u + (row & 7) * 16u, plane);
  }
}

__global__ void __launch_bounds__(kT5, 1) k_attn_fwd_tc5wh(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint8_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (sbase - raw);
  const int T16 = (T + 15) & ~15;
  const uint32_t KPL = static_cast<uint32_t>(T16) * 128u;            // one k (or v) fp16 plane
  const uint32_t sQ = sbase, sK = sbase + 2 * kHPlane;
  unsigned char* gQ = gbase;
  unsigned char* gK = gbase + 2 * kHPlane;
  float* redm = reinterpret_cast<float*>(gK + 2 * KPL);              // [4][128]
  float* reds = redm + 512;                                          // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reds + 512);          // S, P0, P1 (MMA done), F0, F1 (planes written)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  const uint32_t barS = static_cast<uint32_t>(__cvta_generic_to_shared(bars));

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int q0 = blockIdx.x * 128;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.y / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const int c1 = min(T, q0 + 128);                                   // code rows [q0, c1)

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barS + 8 * i));
#pragma unroll
    for (int i = 3; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(barS + 8 * i), "r"(kT5 / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int t7 = tid & 127, d0 = 16 * (tid >> 7);
  const int nkm = (T16 + 127) >> 7;
  float sinv;                                                        // 2^-(eq + ek)
  {
    float4 rq[4], rk[3][4];
    const int tq = q0 + t7;
    {
      const float* src = y3 + (rbase + tq) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rq[c] = tq < T ? __ldg(reinterpret_cast<const float4*>(src) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      const float* src = y3 + MH + (rbase + t) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rk[m][c] = (m < nkm && t < T) ? __ldg(reinterpret_cast<const float4*>(src) + c)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < nkm && t < T) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + MH));   // v, later
    }
    const float mq = bias_codes16(rq, bq + hoff + d0, tq < T, true, qc + (cbase + tq) * (kDH / 4) + d0 / 4, qs, lo, hi);
    float mk = 0.f;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm)
        mk = fmaxf(mk, bias_codes16(rk[m], bk + hoff + d0, t < T, t >= q0 && t < c1,
                                    kc + (cbase + (t < T ? t : 0)) * (kDH / 4) + d0 / 4, qs, lo, hi));
    }
    int eq, ek;
    const float sq = row_scale_exp(block_max512(mq, redm), eq);
    const float sk = row_scale_exp(block_max512(mk, redm), ek);
    sinv = pow2i(-eq) * pow2i(-ek);
    split16_kmajor_hu(rq, sq, t7, d0, gQ, kHPlane);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm && t < T16) split16_kmajor_hu(rk[m], sk, t, d0, gK, KPL);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t accC0 = tmem + 384, accC1 = tmem + 448;
  // kind::f16 with fp16 A and B
  constexpr uint32_t kIdC = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const int r = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;
  const uint32_t lane_addr = static_cast<uint32_t>(32 * (warp & 3)) << 16;

  // ---- S: one accumulator per key chunk of <= 256, lo chain then hi chain
  if (tid == 0) {
    for (int n0 = 0; n0 < T16; n0 += 256) {
      const int nn = min(256, T16 - n0);
      const uint32_t idS = (1u << 4) | ((static_cast<uint32_t>(nn) >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t sKn = sK + (n0 >> 3) * 1024u;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass)
#pragma unroll
        for (int ks = 0; ks < kDH / 16; ++ks) {
          const uint32_t off = ks * 256u;
          const uint64_t ah = desc_nosw(sQ + off, 128, 1024), bh_ = desc_nosw(sKn + off, 128, 1024);
          if (pass == 0) {
            umma(tmem + n0, ah, desc_nosw(sKn + KPL + off, 128, 1024), idS, ks != 0);
            umma(tmem + n0, desc_nosw(sQ + kHPlane + off, 128, 1024), bh_, idS, 1);
          } else {
            umma(tmem + n0, ah, bh_, idS, 1);
          }
        }
    }
    umma_commit(barS);
  }
  __syncwarp();
  mbar_wait5(barS, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // ---- row max, exp-sum over the four column quarters (scores rescaled from TMEM each pass)
  float mx = -INFINITY;
  for (int j = 0; j < nkm; ++j) {
    if (32 * qt < min(128, T16 - 128 * j)) {
      float a0[32];
      tmem_ld32x(tmem + lane_addr + 128 * j + 32 * qt, a0);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int key = 128 * j + 32 * qt + i;
        mx = fmaxf(mx, key < T ? __fmul_rn(a0[i] * sinv, scale) : -INFINITY);
      }
    }
  }
  redm[qt * 128 + r] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(redm[r], redm[128 + r]), fmaxf(redm[256 + r], redm[384 + r]));
  float sum = 0.f;
  for (int j = 0; j < nkm; ++j) {
    if (32 * qt < min(128, T16 - 128 * j)) {
      float a0[32];
      tmem_ld32x(tmem + lane_addr + 128 * j + 32 * qt, a0);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int key = 128 * j + 32 * qt + i;
        sum += key < T ? expf(__fmul_rn(a0[i] * sinv, scale) - mx) : 0.f;
      }
    }
  }
  reds[qt * 128 + r] = sum;
  // ---- v planes (f16x3 form, MN-major) over the k planes (S is complete)
  {
    const uint32_t vsbo = static_cast<uint32_t>(T16) * 16u;
    float4 rv[3][4];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      const float* src = y3 + 2 * MH + (rbase + t) * H + hoff + d0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        rv[m][c] = (m < nkm && t < T) ? __ldg(reinterpret_cast<const float4*>(src) + c)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm && t < T16) {
        bias_codes16(rv[m], bv + hoff + d0, t < T, t >= q0 && t < c1,
                     vc + (cbase + (t < T ? t : 0)) * (kDH / 4) + d0 / 4, qs, lo, hi);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float x[8] = {rv[m][2 * c].x, rv[m][2 * c].y, rv[m][2 * c].z, rv[m][2 * c].w,
                              rv[m][2 * c + 1].x, rv[m][2 * c + 1].y, rv[m][2 * c + 1].z, rv[m][2 * c + 1].w};
          const int d = d0 + 8 * c;
          split8_smem_h(x, gK, (d >> 3) * vsbo + (t >> 3) * 128u + (t & 7) * 16u, KPL);
        }
      }
    }
  }
  __syncthreads();
  sum = (reds[r] + reds[128 + r]) + (reds[256 + r] + reds[384 + r]);
  // ---- p: codes, planes for 32 keys at a time, ctx += p v on the tensor cores
  const int rg = q0 + r;
  uint8_t* prow = pc + (cbase + rg) * T;
  const int nch = (T16 + 31) >> 5;
  for (int c = 0; c < nch; ++c) {
    const int key0 = 32 * c + 8 * qt;
    float p[8];
    tmem_ld8(tmem + lane_addr + key0, p);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i)
      p[i] = key0 + i < T ? __fdiv_rn(expf(__fmul_rn(p[i] * sinv, scale) - mx), sum) : 0.f;
    if (rg < T) {
      if ((T & 7) == 0 && key0 + 8 <= T) {
        *reinterpret_cast<uint2*>(prow + key0) =
            make_uint2(prob_codes4(p[0], p[1], p[2], p[3], qs, hi), prob_codes4(p[4], p[5], p[6], p[7], qs, hi));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (key0 + i < T) prow[key0 + i] = static_cast<uint8_t>(prob_code(p[i], qs, hi));
      }
    }
    const int buf = c & 1;
    if (c >= 2) mbar_wait5(barS + 8 * (1 + buf), ((c - 2) >> 1) & 1);   // chunk c - 2's MMAs read this buffer
    split8_smem_h(p, gQ + buf * 2 * kW5PPlane, (r >> 3) * 512u + qt * 128u + (r & 7) * 16u, kW5PPlane);
    // no CTA barrier per chunk: each warp arrives on the buffer's mbarrier
    // and moves on; the issuing thread waits for all 16 warps
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(barS + 8 * (3 + buf)) : "memory");
    if (tid == 0) {
      mbar_wait5(barS + 8 * (3 + buf), (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int nks = min(2, (T16 - 32 * c) >> 4);
      for (int ks = 0; ks < nks; ++ks) {
        const uint32_t sa = sQ + buf * 2 * kW5PPlane + ks * 256u;
        const uint32_t sb = sK + c * 512u + ks * 256u;
        const uint64_t ah = desc_nosw(sa, 128, 512), al = desc_nosw(sa + kW5PPlane, 128, 512);
        const uint64_t bh_ = desc_nosw(sb, 128, static_cast<uint32_t>(T16) * 16u);
        const uint64_t bl = desc_nosw(sb + KPL, 128, static_cast<uint32_t>(T16) * 16u);
        const uint32_t acc = (c | ks) != 0;
        umma(accC0, ah, bh_, kIdC, acc);
        umma(accC1, ah, bl, kIdC, acc);
        umma(accC1, al, bh_, kIdC, 1);
      }
      umma_commit(barS + 8 * (1 + buf));
    }
    __syncwarp();
  }
  mbar_wait5(barS + 8 * (1 + ((nch - 1) & 1)), ((nch - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* cs = reinterpret_cast<float*>(gQ);                          // [128][kDH + 4] over q | p buffers
  {
    float u0[16], u1[16];
    tmem_ld16(accC0 + lane_addr + 16 * qt, u0);
    tmem_ld16(accC1 + lane_addr + 16 * qt, u1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 16 * qt + j) =
          make_float4(__fmaf_rn(0x1p-11f, u1[j], u0[j]), __fmaf_rn(0x1p-11f, u1[j + 1], u0[j + 1]),
                      __fmaf_rn(0x1p-11f, u1[j + 2], u0[j + 2]), __fmaf_rn(0x1p-11f, u1[j + 3], u0[j + 3]));
  }
  __syncthreads();
  for (int rr = 2 * warp + ((tid & 31) >> 4); rr < 128 && q0 + rr < T; rr += 2 * (kT5 / 32)) {
    const int d = 4 * (tid & 15);
    const float4 o = *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
    const int64_t go = (rbase + q0 + rr) * H + hoff + d;
    if (ctx) *reinterpret_cast<float4*>(ctx + go) = o;   // NULL: planes only
    if (xp) planes_store4f(o, xp, MH, go, pf);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------ tcgen05 backward, query-tiled (T <= 384)
// Two kernels, 512 threads each, exact code operands (q~, k~, v~, p~ as
// bf16), fp32 operands in three bf16 planes, every product three MMAs into
// two TMEM accumulators (the hi term alone, the two smaller terms together).
// (A) grid (ceil(T / 128) query tiles, B * h): dP = g v~^T in key blocks of
//     128 (hi term into the block's columns, small terms into a 128-column
//     scratch, combined in place as the forward does), the row sums
//     rs = sum_j dP p~ (written to ws for kernel B), then 32 keys at a time
//     dS = p~ (dP - rs) scale -> planes in one of two buffers while one
//     thread runs dq += dS k~ on the other.
// (B) grid (ceil(T / 128) key tiles, B * h): for each query tile in turn,
//     dP^T = v~ g^T (M = the tile's 128 keys) and dv += p~^T g, then every
//     thread (TMEM lane = key) forms dS^T = p~ (dP^T - rs) scale for 32 rows
//     into planes and dk += dS^T q~.  g serves as the K-major B operand of
//     dP^T and the MN-major B operand of dv (same bytes, strides swapped);
//     p~ (row-major codes) is the MN-major A operand of dv.
constexpr uint32_t kB5WG = 3 * 128 * kDH * 2;                 // g planes of 128 rows (48 KB)
__host__ __device__ constexpr size_t bwdq5w_smem(int t16) {
  return 1024 + size_t(kB5WG) + 2 * size_t(t16) * 128 + 4 * 128 * sizeof(float) + 64;
}
constexpr size_t kBwdKv5wSmem = 1024 + 16384 + kB5WG + 16384 + 32768 + 3 * 32768 + 128 * sizeof(float) + 64;

// 8 probability codes of row `row` (< T), keys [key0, key0 + 8) (0 past T), as floats
__device__ __forceinline__ void p_codes8(const uint8_t* __restrict__ prow, int key0, int T, float inv, float (&p)[8]) {
  if ((T & 7) == 0 && key0 + 8 <= T) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(prow + key0));
    const float4 a = decode4(w.x, inv), b = decode4(w.y, inv);
    p[0] = a.x; p[1] = a.y; p[2] = a.z; p[3] = a.w; p[4] = b.x; p[5] = b.y; p[6] = b.z; p[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      p[i] = key0 + i < T ? static_cast<float>(static_cast<int8_t>(__ldg(prow + key0 + i))) * inv : 0.f;
  }
}

// one 16-code quarter row of q~ / k~ / v~ -> bf16 (exact) in the 64-wide
// K-major layout (row group 1 KB, dim group 128 B); zeros when !ok
__device__ __forceinline__ void stage_code_row(const uint32_t* __restrict__ src, bool ok, float inv, int row, int d0,
                                               unsigned char* dst) {
  const uint4 w = ok ? __ldg(reinterpret_cast<const uint4*>(src)) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int d = d0 + 8 * c;
    *reinterpret_cast<uint4*>(dst + (row >> 3) * 1024u + (d >> 3) * 128u + (row & 7) * 16u) =
        codes8_bf16(c == 0 ? make_uint2(w.x, w.y) : make_uint2(w.z, w.w), inv);
  }
}

// one 16-float quarter row of g -> three planes (64-wide K-major layout)
__device__ __forceinline__ void stage_g_row(const float* __restrict__ src, bool ok, int row, int d0,
                                            unsigned char* dst) {
  float x[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(src) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    x[4 * c] = v.x;
    x[4 * c + 1] = v.y;
    x[4 * c + 2] = v.z;
    x[4 * c + 3] = v.w;
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int d = d0 + 8 * c;
    split8_smem(x + 8 * c, dst, (row >> 3) * 1024u + (d >> 3) * 128u + (row & 7) * 16u, 128u * kDH * 2);
  }
}

// rows [0, 128) of a [128][kDH + 4] fp32 staging tile -> rows row0 + rr < lim of gcat's block o
__device__ __forceinline__ void store_tile_rows(const float* cs, float* __restrict__ gcat, int64_t rbase, int row0,
                                                int lim, int H, int o, int hoff) {
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int rr = 2 * warp + ((tid & 31) >> 4); rr < 128 && row0 + rr < lim; rr += 2 * (kT5 / 32)) {
    const int d = 4 * (tid & 15);
    *reinterpret_cast<float4*>(gcat + (rbase + row0 + rr) * (3 * H) + o * H + hoff + d) =
        *reinterpret_cast<const float4*>(cs + rr * (kDH + 4) + d);
  }
}

// TMEM (hi, small) accumulator pair, 64 columns -> staging tile rows (lane = row)
__device__ __forceinline__ void acc_pair_to_smem(uint32_t t0, uint32_t t1, uint32_t la, int r, int qt, float* cs) {
  float a0[16], a1[16];
  tmem_ld16(t0 + la + 16 * qt, a0);
  tmem_ld16(t1 + la + 16 * qt, a1);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; j += 4)
    *reinterpret_cast<float4*>(cs + r * (kDH + 4) + 16 * qt + j) =
        make_float4(a0[j] + a1[j], a0[j + 1] + a1[j + 1], a0[j + 2] + a1[j + 2], a0[j + 3] + a1[j + 3]);
}

__global__ void __launch_bounds__(kT5, 1) k_attn_bwdq_tc5w(
    const float* __restrict__ g, const uint32_t* __restrict__ kc, const uint32_t* __restrict__ vc,
    const uint8_t* __restrict__ pc, int T, int h, float scale, float inv, float* __restrict__ gcat,
    float* __restrict__ rs_out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gb = smem_raw + (sbase - raw);
  const int T16 = (T + 15) & ~15;
  const uint32_t KPL = static_cast<uint32_t>(T16) * 128u;
  // [ g planes (later: two dS buffers, then the output staging) | v~ | k~ | row sums | barriers ]
  const uint32_t sG = sbase, sV = sbase + kB5WG, sK = sV + KPL;
  unsigned char* gG = gb;
  unsigned char* gV = gb + kB5WG;
  unsigned char* gK = gV + KPL;
  float* redt = reinterpret_cast<float*>(gK + KPL);                  // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(redt + 512);          // S, D0, D1 (MMA done), F0, F1 (dS written)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  const uint32_t barS = static_cast<uint32_t>(__cvta_generic_to_shared(bars));

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int q0 = blockIdx.x * 128;
  const int H = h * kDH;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barS + 8 * i));
#pragma unroll
    for (int i = 3; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(barS + 8 * i), "r"(kT5 / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int t7 = tid & 127, d0 = 16 * (tid >> 7);
  const int nkm = (T16 + 127) >> 7;
  {
    const int tq = q0 + t7;
    stage_g_row(g + (rbase + tq) * H + hoff + d0, tq < T, t7, d0, gG);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int t = 128 * m + t7;
      if (m < nkm && t < T16) {
        stage_code_row(vc + (cbase + t) * (kDH / 4) + d0 / 4, t < T, inv, t, d0, gV);
        stage_code_row(kc + (cbase + t) * (kDH / 4) + d0 / 4, t < T, inv, t, d0, gK);
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_sync();
  const uint32_t tmem = *tmem_slot;
  const uint32_t accX = tmem + 384, tQ0 = tmem + 384, tQ1 = tmem + 448;
  constexpr uint32_t kBase = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 4) << 24);
  constexpr uint32_t kIdQ = kBase | (1u << 16) | ((64u >> 3) << 17);             // dS k~ (B MN-major)
  constexpr uint32_t GPL = 128u * kDH * 2;
  const int r = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;
  const uint32_t la = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  const int rg = q0 + r;
  const uint8_t* prow = pc + (cbase + (rg < T ? rg : 0)) * T;

  // ---- dP in key blocks, combined in place; partial row sums of dP p~
  float part = 0.f;
  for (int j = 0; j < nkm; ++j) {
    const int nj = min(128, T16 - 128 * j);
    if (tid == 0) {
      const uint32_t idP = kBase | ((static_cast<uint32_t>(nj) >> 3) << 17);
#pragma unroll
      for (int ks = 0; ks < kDH / 16; ++ks) {
        const uint64_t bv = desc_ns(sV + j * 16384u + 256u * ks, 128, 1024);
        umma(tmem + 128 * j, desc_ns(sG + 256u * ks, 128, 1024), bv, idP, ks != 0);
        umma(accX, desc_ns(sG + 2 * GPL + 256u * ks, 128, 1024), bv, idP, ks != 0);
        umma(accX, desc_ns(sG + GPL + 256u * ks, 128, 1024), bv, idP, 1);
      }
      umma_commit(barS);
    }
    __syncwarp();
    mbar_wait5(barS, j & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (32 * qt < nj) {
      float a0[32], a1[32];
      tmem_ld32x(tmem + la + 128 * j + 32 * qt, a0);
      tmem_ld32x(accX + la + 32 * qt, a1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) a0[i] += a1[i];
      tmem_st32x(tmem + la + 128 * j + 32 * qt, a0);
      if (rg < T) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float p[8];
          p_codes8(prow, 128 * j + 32 * qt + 8 * c, T, inv, p);
#pragma unroll
          for (int i = 0; i < 8; ++i)                               // columns past T16 hold stale TMEM
            part += 128 * j + 32 * qt + 8 * c + i < T ? __fmul_rn(a0[8 * c + i], p[i]) : 0.f;
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_sync();
  }
  redt[qt * 128 + r] = part;
  __syncthreads();
  const float rs = (redt[r] + redt[128 + r]) + (redt[256 + r] + redt[384 + r]);
  if (qt == 0 && rg < T) rs_out[cbase + rg] = rs;
  // ---- dS for 32 keys at a time -> planes (two buffers over g), dq += dS k~
  const int nch = (T16 + 31) >> 5;
  for (int c = 0; c < nch; ++c) {
    const int key0 = 32 * c + 8 * qt;
    float dp[8], p[8];
    tmem_ld8(tmem + la + key0, dp);
    if (rg < T) p_codes8(prow, key0, T, inv, p);
    else {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = 0.f;
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i)
      dp[i] = key0 + i < T ? __fmul_rn(__fmul_rn(p[i], __fsub_rn(dp[i], rs)), scale) : 0.f;
    const int buf = c & 1;
    if (c >= 2) mbar_wait5(barS + 8 * (1 + buf), ((c - 2) >> 1) & 1);
    split8_smem(dp, gG + buf * 3 * kW5PPlane, (r >> 3) * 512u + qt * 128u + (r & 7) * 16u, kW5PPlane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(barS + 8 * (3 + buf)) : "memory");
    if (tid == 0) {
      mbar_wait5(barS + 8 * (3 + buf), (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int nks = min(2, (T16 - 32 * c) >> 4);
      for (int ks = 0; ks < nks; ++ks) {
        const uint32_t sa = sG + buf * 3 * kW5PPlane + ks * 256u;
        const uint64_t bk = desc_ns(sK + (4 * c + 2 * ks) * 1024u, 1024, 128);   // MN-major: key groups 1 KB
        const uint32_t acc = (c | ks) != 0;
        umma(tQ0, desc_ns(sa, 128, 512), bk, kIdQ, acc);
        umma(tQ1, desc_ns(sa + 2 * kW5PPlane, 128, 512), bk, kIdQ, acc);
        umma(tQ1, desc_ns(sa + kW5PPlane, 128, 512), bk, kIdQ, 1);
      }
      umma_commit(barS + 8 * (1 + buf));
    }
    __syncwarp();
  }
  mbar_wait5(barS + 8 * (1 + ((nch - 1) & 1)), ((nch - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* cs = reinterpret_cast<float*>(gG);
  acc_pair_to_smem(tQ0, tQ1, la, r, qt, cs);
  __syncthreads();
  store_tile_rows(cs, gcat, rbase, q0, T, H, 0, hoff);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

__global__ void __launch_bounds__(kT5, 1) k_attn_bwdkv_tc5w(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ vc,
    const uint8_t* __restrict__ pc, const float* __restrict__ rs_in, int T, int h, float scale, float inv,
    float* __restrict__ gcat) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  unsigned char* gb = smem_raw + (sbase - raw);
  // [ v~ tile 16 KB | g planes 48 KB | q~ 16 KB | p~ 32 KB | dS^T planes 96 KB (later: output staging) | rs | bars ]
  const uint32_t sVt = sbase, sG = sVt + 16384, sQ = sG + kB5WG, sP = sQ + 16384, sS = sP + 32768;
  unsigned char* gVt = gb;
  unsigned char* gG = gVt + 16384;
  unsigned char* gQ = gG + kB5WG;
  unsigned char* gP = gQ + 16384;
  unsigned char* gS = gP + 32768;
  float* rs_s = reinterpret_cast<float*>(gS + 3 * 32768);            // [128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rs_s + 128);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const uint32_t bar1 = static_cast<uint32_t>(__cvta_generic_to_shared(bars)), bar2 = bar1 + 8;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int k0 = blockIdx.x * 128;
  const int H = h * kDH;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar2));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot))), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int t7 = tid & 127, qtr = tid >> 7, d0 = 16 * qtr;
  {
    const int kk = k0 + t7;
    stage_code_row(vc + (cbase + kk) * (kDH / 4) + d0 / 4, kk < T, inv, t7, d0, gVt);
  }
  constexpr uint32_t kBase = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 4) << 24);
  constexpr uint32_t kIdPt = kBase | ((128u >> 3) << 17);                           // v~ g^T
  constexpr uint32_t kIdV = kBase | (1u << 15) | (1u << 16) | ((64u >> 3) << 17);  // p~^T g
  constexpr uint32_t kIdK = kBase | (1u << 16) | ((64u >> 3) << 17);               // dS^T q~
  constexpr uint32_t GPL = 128u * kDH * 2;
  const int kr = 32 * (warp & 3) + (tid & 31), qt = warp >> 2;     // TMEM lane = key of the tile
  const uint32_t la = static_cast<uint32_t>(32 * (warp & 3)) << 16;
  const int kg = k0 + kr;
  const int nq = (T + 127) >> 7;
  uint32_t tmem = 0;
  for (int i = 0; i < nq; ++i) {
    const int i0 = 128 * i;
    if (i > 0) mbar_wait5(bar2, (i - 1) & 1);                       // tile i - 1's products are done
    {
      const int t = i0 + t7;
      const bool ok = t < T;
      stage_g_row(g + (rbase + t) * H + hoff + d0, ok, t7, d0, gG);
      stage_code_row(qc + (cbase + t) * (kDH / 4) + d0 / 4, ok, inv, t7, d0, gQ);
      // p~ row t, keys [k0 + 32 qtr, +32) -> bf16 (row group 2 KB, key group 128 B)
      const uint8_t* prow = pc + (cbase + (ok ? t : 0)) * T;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int kk = 32 * qtr + 8 * c;
        float p[8];
        if (ok) p_codes8(prow, k0 + kk, T, inv, p);
        else {
#pragma unroll
          for (int e = 0; e < 8; ++e) p[e] = 0.f;
        }
        *reinterpret_cast<uint4*>(gP + (t7 >> 3) * 2048u + (kk >> 3) * 128u + (t7 & 7) * 16u) =
            make_uint4(bf2(p[0], p[1]), bf2(p[2], p[3]), bf2(p[4], p[5]), bf2(p[6], p[7]));
      }
      if (qtr == 0) rs_s[t7] = ok ? __ldg(rs_in + cbase + t) : 0.f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_sync();
    if (i == 0) tmem = *tmem_slot;
    const uint32_t tPt0 = tmem, tPt1 = tmem + 128, tV0 = tmem + 256, tV1 = tmem + 320;
    const uint32_t tK0 = tmem + 384, tK1 = tmem + 448;
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < kDH / 16; ++ks) {                       // dP^T: K = head dims
        const uint64_t av = desc_ns(sVt + 256u * ks, 128, 1024);
        umma(tPt0, av, desc_ns(sG + 256u * ks, 128, 1024), kIdPt, ks != 0);
        umma(tPt1, av, desc_ns(sG + 2 * GPL + 256u * ks, 128, 1024), kIdPt, ks != 0);
        umma(tPt1, av, desc_ns(sG + GPL + 256u * ks, 128, 1024), kIdPt, 1);
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {                              // dv: K = rows, 16 per step
        const uint64_t ap = desc_ns(sP + 4096u * ks, 2048, 128);    // MN-major: row groups 2 KB, key groups 128 B
        const uint32_t acc = (i | ks) != 0;
        umma(tV0, ap, desc_ns(sG + 2048u * ks, 1024, 128), kIdV, acc);
        umma(tV1, ap, desc_ns(sG + 2 * GPL + 2048u * ks, 1024, 128), kIdV, acc);
        umma(tV1, ap, desc_ns(sG + GPL + 2048u * ks, 1024, 128), kIdV, 1);
      }
      umma_commit(bar1);
    }
    __syncwarp();
    mbar_wait5(bar1, i & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- dS^T: thread = key kr, rows [32 qt, +32) of the tile
    {
      float dp[32];
      {
        float a0[16], a1[16];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          tmem_ld16(tPt0 + la + 32 * qt + 16 * c, a0);
          tmem_ld16(tPt1 + la + 32 * qt + 16 * c, a1);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) dp[16 * c + j] = a0[j] + a1[j];
        }
      }
      const bool kok = kg < T;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int row = 32 * qt + j;
        const uint16_t pb = *reinterpret_cast<const uint16_t*>(
            gP + (row >> 3) * 2048u + (kr >> 3) * 128u + (row & 7) * 16u + (kr & 7) * 2u);
        const float p = __uint_as_float(static_cast<uint32_t>(pb) << 16);
        dp[j] = (kok && i0 + row < T) ? __fmul_rn(__fmul_rn(p, __fsub_rn(dp[j], rs_s[row])), scale) : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
        split8_smem(dp + 8 * c, gS, (kr >> 3) * 2048u + ((32 * qt + 8 * c) >> 3) * 128u + (kr & 7) * 16u, 32768u);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_sync();
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {                              // dk: K = rows, 16 per step
        const uint64_t bq = desc_ns(sQ + 2048u * ks, 1024, 128);    // MN-major: row groups 1 KB, dim groups 128 B
        const uint32_t acc = (i | ks) != 0;
        umma(tK0, desc_ns(sS + 256u * ks, 128, 2048), bq, kIdK, acc);
        umma(tK1, desc_ns(sS + 2 * 32768u + 256u * ks, 128, 2048), bq, kIdK, acc);
        umma(tK1, desc_ns(sS + 32768u + 256u * ks, 128, 2048), bq, kIdK, 1);
      }
      umma_commit(bar2);
    }
    __syncwarp();
  }
  mbar_wait5(bar2, (nq - 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* cs = reinterpret_cast<float*>(gS);
#pragma unroll 1
  for (int o = 1; o < 3; ++o) {
    acc_pair_to_smem(o == 1 ? tmem + 384 : tmem + 256, o == 1 ? tmem + 448 : tmem + 320, la, kr, qt, cs);
    __syncthreads();
    store_tile_rows(cs, gcat, rbase, k0, T, H, o, hoff);
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------ wide forward (T <= 384)
// grid (ceil(T / 64), B * h); one CTA = 64 query rows of one head, all
// keys; 512 threads = 16 warps: warp w = (row group w / 4: rows
// [16 (w / 4), +16)) x (key group w % 4: keys [KW (w % 4), +KW), KW = 8 NT).
// Shared memory holds the tile's q planes and ALL keys' k planes; after the
// scores the k planes are replaced by the v planes (same space).  Scores,
// softmax, the 8-bit probability codes and the context follow the
// one-head kernel above (same operations, same order per element); the
// four key groups' partial contexts are summed in key order.  q codes are
// written for the tile's rows, k and v codes for the same row range (each
// head's rows are covered once by its tiles).
constexpr int kQT = 64;                  // query rows per CTA
constexpr int kKG = 4;                   // key groups
constexpr int kTW = 512;                 // threads
constexpr int kTMW = 384;                // max sequence length of the wide kernels

template <int NT>
constexpr size_t fwd_wide_smem() {
  return (3 * size_t(kQT) * kVB + 3 * size_t(kKG * 8 * NT) * kVB) * 2 + 2 * size_t(kKG) * kQT * sizeof(float);
}

// (row, d4) items of rows [row0, row0 + rows) of projection m: fp32 + bias
// -> three bf16 planes (row-major [row][kVB]); codes for rows in [c0, c1)
__device__ __forceinline__ void stage_planes(const float* __restrict__ src, float4 bias, int64_t rbase, int H,
                                             int hoff, int T, int row0, int rows, __nv_bfloat16* planes,
                                             size_t plane, uint32_t* __restrict__ codes, int64_t cbase, int c0,
                                             int c1, float qs, float lo, float hi) {
  const int d4 = threadIdx.x & 15;
  constexpr int kPer = 4;                // rows per thread in flight (32 rows per pass of 512 threads)
  for (int t0 = threadIdx.x >> 4; t0 < rows; t0 += kPer * (kTW / 16)) {
    float4 x[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int t = t0 + q * (kTW / 16), r = row0 + t;
      x[q] = (t < rows && r < T) ? add4(__ldg(reinterpret_cast<const float4*>(src + (rbase + r) * H + hoff) + d4), bias)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int t = t0 + q * (kTW / 16), r = row0 + t;
      if (t >= rows) continue;
      if (r < T && r >= c0 && r < c1) codes[(cbase + r) * (kDH / 4) + d4] = codes4(x[q], qs, lo, hi);
      uint32_t h0, m0, l0, h1, m1, l1;
      split_pair(x[q].x, x[q].y, h0, m0, l0);
      split_pair(x[q].z, x[q].w, h1, m1, l1);
      const size_t o = (static_cast<size_t>(t) * kVB + 4 * d4) / 2;
      uint32_t* P = reinterpret_cast<uint32_t*>(planes);
      P[o] = h0;
      P[o + 1] = h1;
      P[plane / 2 + o] = m0;
      P[plane / 2 + o + 1] = m1;
      P[plane + o] = l0;
      P[plane + o + 1] = l1;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(kTW, 1) k_attn_fwd_wide(
    const float* __restrict__ y3, const float* __restrict__ bq, const float* __restrict__ bk,
    const float* __restrict__ bv, int T, int h, float scale, float qs, float lo, float hi,
    float* __restrict__ ctx, uint32_t* __restrict__ qc, uint32_t* __restrict__ kc,
    uint32_t* __restrict__ vc, uint8_t* __restrict__ pc, __nv_bfloat16* __restrict__ xp, int pf) {
  static_assert(NT % 2 == 0 && NT % 4 == 0, "16-key MMA steps; n-tiles staged four at a time");
  constexpr int TK = kKG * 8 * NT;                               // padded keys
  constexpr size_t QPL = size_t(kQT) * kVB, KPL = size_t(TK) * kVB;
  extern __shared__ __align__(16) unsigned char smb[];
  __nv_bfloat16* Qp = reinterpret_cast<__nv_bfloat16*>(smb);      // [3][kQT][kVB]
  __nv_bfloat16* KVp = Qp + 3 * QPL;                              // [3][TK][kVB]: k, then v
  float* redm = reinterpret_cast<float*>(KVp + 3 * KPL);           // [kKG][kQT]
  float* reds = redm + kKG * kQT;                                 // [kKG][kQT]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int qt = blockIdx.x, bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t MH = static_cast<int64_t>(gridDim.y / h) * T * H;
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const int q0 = qt * kQT;
  {
    const int d4 = tid & 15;
    stage_planes(y3, __ldg(reinterpret_cast<const float4*>(bq + hoff) + d4), rbase, H, hoff, T, q0, kQT, Qp, QPL,
                 qc, cbase, q0, q0 + kQT, qs, lo, hi);
    stage_planes(y3 + MH, __ldg(reinterpret_cast<const float4*>(bk + hoff) + d4), rbase, H, hoff, T, 0, TK, KVp,
                 KPL, kc, cbase, q0, q0 + kQT, qs, lo, hi);
  }
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int rg = w / kKG, kg = w % kKG;
  const int R0 = 16 * rg, J0 = 8 * NT * kg;
  const uint32_t* Q32 = reinterpret_cast<const uint32_t*>(Qp);
  const uint32_t* K32 = reinterpret_cast<const uint32_t*>(KVp);
  constexpr int QW = int(QPL / 2), KW = int(KPL / 2), RW = kVB / 2;
  constexpr int PA[6] = {2, 0, 1, 1, 0, 0}, PB[6] = {0, 2, 1, 0, 1, 0};   // lh hl mm mh hm hh

  // ---- S = q k^T over this warp's keys (n-tiles four at a time)
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < kDH / 16; ++kb) {
    uint32_t a[3][4];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      a[p][0] = Q32[p * QW + (R0 + gq) * RW + 8 * kb + tq];
      a[p][1] = Q32[p * QW + (R0 + gq + 8) * RW + 8 * kb + tq];
      a[p][2] = Q32[p * QW + (R0 + gq) * RW + 8 * kb + 4 + tq];
      a[p][3] = Q32[p * QW + (R0 + gq + 8) * RW + 8 * kb + 4 + tq];
    }
#pragma unroll
    for (int n0 = 0; n0 < NT; n0 += 4) {
      uint32_t b0[3][4], b1[3][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          b0[p][u] = K32[p * KW + (J0 + 8 * (n0 + u) + gq) * RW + 8 * kb + tq];
          b1[p][u] = K32[p * KW + (J0 + 8 * (n0 + u) + gq) * RW + 8 * kb + 4 + tq];
        }
#pragma unroll
      for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) mma16816(acc[n0 + u], a[PA[q]], b0[PB[q]][u], b1[PB[q]][u]);
    }
  }

  // ---- softmax over all keys: rows R0 + gq (c0, c1) and R0 + gq + 8 (c2, c3)
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    const bool v0 = j < T, v1 = j + 1 < T;
    acc[nt][0] = v0 ? __fmul_rn(acc[nt][0], scale) : -INFINITY;
    acc[nt][1] = v1 ? __fmul_rn(acc[nt][1], scale) : -INFINITY;
    acc[nt][2] = v0 ? __fmul_rn(acc[nt][2], scale) : -INFINITY;
    acc[nt][3] = v1 ? __fmul_rn(acc[nt][3], scale) : -INFINITY;
    m0 = fmaxf(m0, fmaxf(acc[nt][0], acc[nt][1]));
    m1 = fmaxf(m1, fmaxf(acc[nt][2], acc[nt][3]));
  }
  m0 = fmaxf(m0, __shfl_xor_sync(0xFFFFFFFFu, m0, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xFFFFFFFFu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xFFFFFFFFu, m1, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xFFFFFFFFu, m1, 2));
  if (tq == 0) {
    redm[kg * kQT + R0 + gq] = m0;
    redm[kg * kQT + R0 + gq + 8] = m1;
  }
  __syncthreads();
  m0 = redm[R0 + gq];
  m1 = redm[R0 + gq + 8];
#pragma unroll
  for (int g2 = 1; g2 < kKG; ++g2) {
    m0 = fmaxf(m0, redm[g2 * kQT + R0 + gq]);
    m1 = fmaxf(m1, redm[g2 * kQT + R0 + gq + 8]);
  }
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    acc[nt][0] = j < T ? expf(acc[nt][0] - m0) : 0.f;
    acc[nt][1] = j + 1 < T ? expf(acc[nt][1] - m0) : 0.f;
    acc[nt][2] = j < T ? expf(acc[nt][2] - m1) : 0.f;
    acc[nt][3] = j + 1 < T ? expf(acc[nt][3] - m1) : 0.f;
    s0 += acc[nt][0] + acc[nt][1];
    s1 += acc[nt][2] + acc[nt][3];
  }
  s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, 1);
  s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, 2);
  s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, 1);
  s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, 2);
  if (tq == 0) {
    reds[kg * kQT + R0 + gq] = s0;
    reds[kg * kQT + R0 + gq + 8] = s1;
  }
  __syncthreads();                       // also: every warp is done reading the k planes
  s0 = reds[R0 + gq];
  s1 = reds[R0 + gq + 8];
#pragma unroll
  for (int g2 = 1; g2 < kKG; ++g2) {
    s0 += reds[g2 * kQT + R0 + gq];
    s1 += reds[g2 * kQT + R0 + gq + 8];
  }
  const int r0 = q0 + R0 + gq, r1 = r0 + 8;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    acc[nt][0] = __fdiv_rn(acc[nt][0], s0);
    acc[nt][1] = __fdiv_rn(acc[nt][1], s0);
    acc[nt][2] = __fdiv_rn(acc[nt][2], s1);
    acc[nt][3] = __fdiv_rn(acc[nt][3], s1);
    if (j < T) {
      if (r0 < T) pc[(cbase + r0) * T + j] = static_cast<uint8_t>(fixed_code(acc[nt][0], qs, lo, hi));
      if (r1 < T) pc[(cbase + r1) * T + j] = static_cast<uint8_t>(fixed_code(acc[nt][2], qs, lo, hi));
    }
    if (j + 1 < T) {
      if (r0 < T) pc[(cbase + r0) * T + j + 1] = static_cast<uint8_t>(fixed_code(acc[nt][1], qs, lo, hi));
      if (r1 < T) pc[(cbase + r1) * T + j + 1] = static_cast<uint8_t>(fixed_code(acc[nt][3], qs, lo, hi));
    }
  }
  // ---- v planes over the k planes
  stage_planes(y3 + 2 * MH, __ldg(reinterpret_cast<const float4*>(bv + hoff) + (tid & 15)), rbase, H, hoff, T, 0,
               TK, KVp, KPL, vc, cbase, q0, q0 + kQT, qs, lo, hi);
  __syncthreads();

  // ---- ctx partial = p v over this warp's keys, head dims in two halves
  //      of 32 (A = p from registers, split; B = v planes via ldmatrix.trans)
  float* part = reinterpret_cast<float*>(smb);             // [kKG - 1][4][16][kDH + 4], over q planes | v
  float o[2][4][4];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) o[hf][nt][0] = o[hf][nt][1] = o[hf][nt][2] = o[hf][nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < NT / 2; ++kb) {
    uint32_t a[3][4];
    split_pair(acc[2 * kb][0], acc[2 * kb][1], a[0][0], a[1][0], a[2][0]);
    split_pair(acc[2 * kb][2], acc[2 * kb][3], a[0][1], a[1][1], a[2][1]);
    split_pair(acc[2 * kb + 1][0], acc[2 * kb + 1][1], a[0][2], a[1][2], a[2][2]);
    split_pair(acc[2 * kb + 1][2], acc[2 * kb + 1][3], a[0][3], a[1][3], a[2][3]);
    const int jrow = J0 + 16 * kb + (lane & 15);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      uint32_t b0[3][4], b1[3][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int p = 0; p < 3; ++p)
          ldsm_x2_trans(b0[p][u], b1[p][u], KVp + p * KPL + jrow * kVB + 32 * hf + 8 * u);
#pragma unroll
      for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) mma16816(o[hf][u], a[PA[q]], b0[PB[q]][u], b1[PB[q]][u]);
    }
  }
  __syncthreads();                                          // v planes no longer read: partials go over them
  if (kg > 0) {
    float* my = part + ((kg - 1) * 4 + rg) * 16 * (kDH + 4);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 32 * hf + 8 * u + 2 * tq;
        *reinterpret_cast<float2*>(my + gq * (kDH + 4) + d) = make_float2(o[hf][u][0], o[hf][u][1]);
        *reinterpret_cast<float2*>(my + (gq + 8) * (kDH + 4) + d) = make_float2(o[hf][u][2], o[hf][u][3]);
      }
  }
  __syncthreads();
  if (kg == 0) {
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 32 * hf + 8 * u + 2 * tq;
        float2 c0 = make_float2(o[hf][u][0], o[hf][u][1]), c1 = make_float2(o[hf][u][2], o[hf][u][3]);
#pragma unroll
        for (int g2 = 1; g2 < kKG; ++g2) {                 // key order
          const float* pp = part + ((g2 - 1) * 4 + rg) * 16 * (kDH + 4);
          const float2 x0 = *reinterpret_cast<const float2*>(pp + gq * (kDH + 4) + d);
          const float2 x1 = *reinterpret_cast<const float2*>(pp + (gq + 8) * (kDH + 4) + d);
          c0.x += x0.x;
          c0.y += x0.y;
          c1.x += x1.x;
          c1.y += x1.y;
        }
        if (r0 < T) {
          *reinterpret_cast<float2*>(ctx + (rbase + r0) * H + hoff + d) = c0;
          if (xp) planes_store2f(c0.x, c0.y, xp, MH, (rbase + r0) * H + hoff + d, pf);
        }
        if (r1 < T) {
          *reinterpret_cast<float2*>(ctx + (rbase + r1) * H + hoff + d) = c1;
          if (xp) planes_store2f(c1.x, c1.y, xp, MH, (rbase + r1) * H + hoff + d, pf);
        }
      }
  }
}

// ------------------------------------------------------------------ wide backward (T <= 384)
// Two kernels.  (A) grid (ceil(T / 64), B * h), 16 warps as in the wide
// forward: for the tile's 64 query rows over all keys dP = g v~^T, the row
// sums rs = sum_j dP p~ (written out), dS = p~ (dP - rs) scale in
// registers, dq = dS k~ (the four key groups' partials summed in key order).
// (B) grid (ceil(T / 64), B * h), 8 warps: for the tile's 64 keys, over all
// query tiles, dP of the (query tile, key tile) block again, dS with the
// rows' rs, written transposed into shared memory as three bf16 planes,
// then dk += dS^T q~ (warps 0-3) and dv += p~^T g (warps 4-7) in registers.
// Code operands are exact in bf16; fp32 operands take the exact 3-term
// split, so every product is three MMAs (as in the one-head kernels).
template <int NT>
constexpr size_t bwdq_wide_smem() {
  return (3 * size_t(kQT) * kVB + 2 * size_t(kKG * 8 * NT) * kVB) * 2 + size_t(kKG) * kQT * sizeof(float);
}
constexpr size_t kBwdKvSmem = (size_t(kQT) * kVB * (1 + 3 + 1 + 1 + 3)) * 2 + kQT * sizeof(float);

// rows [row0, row0 + rows) of int8 codes (B, h, T, 64) -> bf16 [row][kVB] (exact)
__device__ __forceinline__ void stage_codes(const uint32_t* __restrict__ codes, int64_t cbase, int T, int row0,
                                            int rows, float inv, __nv_bfloat16* dst, int nthreads) {
  for (int idx = threadIdx.x; idx < rows * (kDH / 4); idx += nthreads) {
    const int t = idx / (kDH / 4), c4 = idx - t * (kDH / 4), r = row0 + t;
    const float4 v = r < T ? decode4(__ldg(codes + (cbase + r) * (kDH / 4) + c4), inv) : make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + t * kVB + 4 * c4);
    d[0] = bf2(v.x, v.y);
    d[1] = bf2(v.z, v.w);
  }
}

template <int NT>
__global__ void __launch_bounds__(kTW, 1) k_attn_bwdq_wide(
    const float* __restrict__ g, const uint32_t* __restrict__ kc, const uint32_t* __restrict__ vc,
    const uint8_t* __restrict__ pc, int T, int h, float scale, float inv, float* __restrict__ gcat,
    float* __restrict__ rs_out, __nv_bfloat16* __restrict__ xp) {
  constexpr int TK = kKG * 8 * NT;
  constexpr size_t QPL = size_t(kQT) * kVB;
  extern __shared__ __align__(16) unsigned char smb[];
  __nv_bfloat16* Gp = reinterpret_cast<__nv_bfloat16*>(smb);      // [3][kQT][kVB]
  __nv_bfloat16* Vb = Gp + 3 * QPL;                               // [TK][kVB]  v~
  __nv_bfloat16* Kb = Vb + size_t(TK) * kVB;                      // [TK][kVB]  k~
  float* redr = reinterpret_cast<float*>(Kb + size_t(TK) * kVB);  // [kKG][kQT]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int qt = blockIdx.x, bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t P3 = static_cast<int64_t>(gridDim.y / h) * T * 3 * H;   // gcat planes' stride
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const int q0 = qt * kQT;
  stage_planes(g, make_float4(0.f, 0.f, 0.f, 0.f), rbase, H, hoff, T, q0, kQT, Gp, QPL, nullptr, 0, 0, 0, 1.f, 0.f,
               0.f);
  stage_codes(vc, cbase, T, 0, TK, inv, Vb, kTW);
  stage_codes(kc, cbase, T, 0, TK, inv, Kb, kTW);
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int rg = w / kKG, kg = w % kKG;
  const int R0 = 16 * rg, J0 = 8 * NT * kg;
  const int r0 = q0 + R0 + gq, r1 = r0 + 8;
  const uint32_t* G32 = reinterpret_cast<const uint32_t*>(Gp);
  const uint32_t* V32 = reinterpret_cast<const uint32_t*>(Vb);
  constexpr int GW = int(QPL / 2), RW = kVB / 2;
  // p codes of this thread's entries: bytes (r0, j), (r0, j+1), (r1, j), (r1, j+1)
  uint32_t pw[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int j = J0 + 8 * nt + 2 * tq;
    uint32_t v = 0;
    if (r0 < T && j < T) v |= __ldg(pc + (cbase + r0) * T + j);
    if (r0 < T && j + 1 < T) v |= static_cast<uint32_t>(__ldg(pc + (cbase + r0) * T + j + 1)) << 8;
    if (r1 < T && j < T) v |= static_cast<uint32_t>(__ldg(pc + (cbase + r1) * T + j)) << 16;
    if (r1 < T && j + 1 < T) v |= static_cast<uint32_t>(__ldg(pc + (cbase + r1) * T + j + 1)) << 24;
    pw[nt] = v;
  }
  // ---- dP = g v~^T (A: g planes, B: v~ rows)
  float acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < kDH / 16; ++kb) {
    uint32_t a[3][4];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      a[p][0] = G32[p * GW + (R0 + gq) * RW + 8 * kb + tq];
      a[p][1] = G32[p * GW + (R0 + gq + 8) * RW + 8 * kb + tq];
      a[p][2] = G32[p * GW + (R0 + gq) * RW + 8 * kb + 4 + tq];
      a[p][3] = G32[p * GW + (R0 + gq + 8) * RW + 8 * kb + 4 + tq];
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint32_t b0 = V32[(J0 + 8 * nt + gq) * RW + 8 * kb + tq];
      const uint32_t b1 = V32[(J0 + 8 * nt + gq) * RW + 8 * kb + 4 + tq];
      mma16816(acc[nt], a[2], b0, b1);                     // lo, mid, hi: smallest first
      mma16816(acc[nt], a[1], b0, b1);
      mma16816(acc[nt], a[0], b0, b1);
    }
  }
  // ---- row sums of dP p~, over the four key groups
  float t0s = 0.f, t1s = 0.f;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float p00 = code_f(static_cast<int8_t>(pw[nt] & 0xFFu), inv);
    const float p01 = code_f(static_cast<int8_t>((pw[nt] >> 8) & 0xFFu), inv);
    const float p10 = code_f(static_cast<int8_t>((pw[nt] >> 16) & 0xFFu), inv);
    const float p11 = code_f(static_cast<int8_t>(pw[nt] >> 24), inv);
    t0s += __fmul_rn(acc[nt][0], p00) + __fmul_rn(acc[nt][1], p01);
    t1s += __fmul_rn(acc[nt][2], p10) + __fmul_rn(acc[nt][3], p11);
  }
  t0s += __shfl_xor_sync(0xFFFFFFFFu, t0s, 1);
  t0s += __shfl_xor_sync(0xFFFFFFFFu, t0s, 2);
  t1s += __shfl_xor_sync(0xFFFFFFFFu, t1s, 1);
  t1s += __shfl_xor_sync(0xFFFFFFFFu, t1s, 2);
  if (tq == 0) {
    redr[kg * kQT + R0 + gq] = t0s;
    redr[kg * kQT + R0 + gq + 8] = t1s;
  }
  __syncthreads();
  float dt0 = redr[R0 + gq], dt1 = redr[R0 + gq + 8];
#pragma unroll
  for (int g2 = 1; g2 < kKG; ++g2) {
    dt0 += redr[g2 * kQT + R0 + gq];
    dt1 += redr[g2 * kQT + R0 + gq + 8];
  }
  if (kg == 0 && tq == 0) {
    if (r0 < T) rs_out[cbase + r0] = dt0;
    if (r1 < T) rs_out[cbase + r1] = dt1;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float p00 = code_f(static_cast<int8_t>(pw[nt] & 0xFFu), inv);
    const float p01 = code_f(static_cast<int8_t>((pw[nt] >> 8) & 0xFFu), inv);
    const float p10 = code_f(static_cast<int8_t>((pw[nt] >> 16) & 0xFFu), inv);
    const float p11 = code_f(static_cast<int8_t>(pw[nt] >> 24), inv);
    acc[nt][0] = __fmul_rn(__fmul_rn(p00, __fsub_rn(acc[nt][0], dt0)), scale);
    acc[nt][1] = __fmul_rn(__fmul_rn(p01, __fsub_rn(acc[nt][1], dt0)), scale);
    acc[nt][2] = __fmul_rn(__fmul_rn(p10, __fsub_rn(acc[nt][2], dt1)), scale);
    acc[nt][3] = __fmul_rn(__fmul_rn(p11, __fsub_rn(acc[nt][3], dt1)), scale);
  }
  // ---- dq partial = dS k~ over this warp's keys (A: dS split from registers,
  //      B: k~ via ldmatrix.trans), head dims in two halves
  float o[2][4][4];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) o[hf][nt][0] = o[hf][nt][1] = o[hf][nt][2] = o[hf][nt][3] = 0.f;
#pragma unroll
  for (int kb = 0; kb < NT / 2; ++kb) {
    uint32_t a[3][4];
    split_pair(acc[2 * kb][0], acc[2 * kb][1], a[0][0], a[1][0], a[2][0]);
    split_pair(acc[2 * kb][2], acc[2 * kb][3], a[0][1], a[1][1], a[2][1]);
    split_pair(acc[2 * kb + 1][0], acc[2 * kb + 1][1], a[0][2], a[1][2], a[2][2]);
    split_pair(acc[2 * kb + 1][2], acc[2 * kb + 1][3], a[0][3], a[1][3], a[2][3]);
    const int jrow = J0 + 16 * kb + (lane & 15);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      uint32_t b0[4], b1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) ldsm_x2_trans(b0[u], b1[u], Kb + jrow * kVB + 32 * hf + 8 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mma16816(o[hf][u], a[2], b0[u], b1[u]);
        mma16816(o[hf][u], a[1], b0[u], b1[u]);
        mma16816(o[hf][u], a[0], b0[u], b1[u]);
      }
    }
  }
  __syncthreads();                                          // planes no longer read: partials over them
  float* part = reinterpret_cast<float*>(smb);
  if (kg > 0) {
    float* my = part + ((kg - 1) * 4 + rg) * 16 * (kDH + 4);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 32 * hf + 8 * u + 2 * tq;
        *reinterpret_cast<float2*>(my + gq * (kDH + 4) + d) = make_float2(o[hf][u][0], o[hf][u][1]);
        *reinterpret_cast<float2*>(my + (gq + 8) * (kDH + 4) + d) = make_float2(o[hf][u][2], o[hf][u][3]);
      }
  }
  __syncthreads();
  if (kg == 0) {
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = 32 * hf + 8 * u + 2 * tq;
        float2 c0 = make_float2(o[hf][u][0], o[hf][u][1]), c1 = make_float2(o[hf][u][2], o[hf][u][3]);
#pragma unroll
        for (int g2 = 1; g2 < kKG; ++g2) {
          const float* pp = part + ((g2 - 1) * 4 + rg) * 16 * (kDH + 4);
          const float2 x0 = *reinterpret_cast<const float2*>(pp + gq * (kDH + 4) + d);
          const float2 x1 = *reinterpret_cast<const float2*>(pp + (gq + 8) * (kDH + 4) + d);
          c0.x += x0.x;
          c0.y += x0.y;
          c1.x += x1.x;
          c1.y += x1.y;
        }
        if (r0 < T) {
          *reinterpret_cast<float2*>(gcat + (rbase + r0) * (3 * H) + hoff + d) = c0;
          if (xp) planes_store2(c0.x, c0.y, xp, P3, (rbase + r0) * (3 * H) + hoff + d);
        }
        if (r1 < T) {
          *reinterpret_cast<float2*>(gcat + (rbase + r1) * (3 * H) + hoff + d) = c1;
          if (xp) planes_store2(c1.x, c1.y, xp, P3, (rbase + r1) * (3 * H) + hoff + d);
        }
      }
  }
}

constexpr int kTKV = 256;                 // kernel B threads

__global__ void __launch_bounds__(kTKV, 2) k_attn_bwdkv_wide(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ vc,
    const uint8_t* __restrict__ pc, const float* __restrict__ rs, int T, int h, float scale, float inv,
    float* __restrict__ gcat, __nv_bfloat16* __restrict__ xp) {
  constexpr size_t PL = size_t(kQT) * kVB;
  extern __shared__ __align__(16) unsigned char smb[];
  __nv_bfloat16* Vt = reinterpret_cast<__nv_bfloat16*>(smb);      // [key][kVB]    v~ of the key tile
  __nv_bfloat16* Gp = Vt + PL;                                    // [3][row][kVB] g planes
  __nv_bfloat16* Qb = Gp + 3 * PL;                                // [row][kVB]    q~
  __nv_bfloat16* Pt = Qb + PL;                                    // [key][kVB]    p~^T (rows along)
  __nv_bfloat16* St = Pt + PL;                                    // [3][key][kVB] dS^T planes
  float* rsr = reinterpret_cast<float*>(St + 3 * PL);              // [row]

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kt = blockIdx.x, bh = blockIdx.y, b = bh / h, hh = bh - b * h;
  const int H = h * kDH;
  const int64_t P3 = static_cast<int64_t>(gridDim.y / h) * T * 3 * H;   // gcat planes' stride
  const int64_t rbase = static_cast<int64_t>(b) * T;
  const int hoff = hh * kDH;
  const int64_t cbase = static_cast<int64_t>(bh) * T;
  const int k0 = kt * kQT;
  const int gq = lane >> 2, tq = lane & 3;
  constexpr int RW = kVB / 2, PW = int(PL / 2);
  stage_codes(vc, cbase, T, k0, kQT, inv, Vt, kTKV);
  // dP phase: warp = rows [16 (w & 3), +16) x keys [32 (w >> 2), +32)
  const int R0 = 16 * (w & 3), J0 = 32 * (w >> 2);
  // dK / dV phase: warps 0-3 dk, 4-7 dv, keys [16 (w & 3), +16)
  const int KR = 16 * (w & 3);
  const bool is_dv = w >= 4;
  float accO[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) accO[nt][0] = accO[nt][1] = accO[nt][2] = accO[nt][3] = 0.f;
  const uint32_t* G32 = reinterpret_cast<const uint32_t*>(Gp);
  const uint32_t* V32 = reinterpret_cast<const uint32_t*>(Vt);
  const uint32_t* S32 = reinterpret_cast<const uint32_t*>(St);
  const uint32_t* P32 = reinterpret_cast<const uint32_t*>(Pt);
  const int nqt = (T + kQT - 1) / kQT;
  for (int qt = 0; qt < nqt; ++qt) {
    const int q0 = qt * kQT;
    __syncthreads();                                        // previous tile's planes fully consumed
    // ---- stage: g planes, q~, p~^T (transposed), rs of the query tile
    {
      const int d4 = tid & 15;
      for (int t = tid >> 4; t < kQT; t += kTKV / 16) {
        const int r = q0 + t;
        const float4 x = r < T ? __ldg(reinterpret_cast<const float4*>(g + (rbase + r) * H + hoff) + d4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t h0, m0, l0, h1, m1, l1;
        split_pair(x.x, x.y, h0, m0, l0);
        split_pair(x.z, x.w, h1, m1, l1);
        uint32_t* P = reinterpret_cast<uint32_t*>(Gp) + (t * kVB + 4 * d4) / 2;
        P[0] = h0;
        P[1] = h1;
        P[PW] = m0;
        P[PW + 1] = m1;
        P[2 * PW] = l0;
        P[2 * PW + 1] = l1;
      }
      stage_codes(qc, cbase, T, q0, kQT, inv, Qb, kTKV);
      for (int idx = tid; idx < kQT * kQT; idx += kTKV) {
        const int t = idx / kQT, jj = idx - t * kQT, r = q0 + t, j = k0 + jj;
        const float pv = (r < T && j < T) ? code_f(static_cast<int8_t>(__ldg(pc + (cbase + r) * T + j)), inv) : 0.f;
        Pt[jj * kVB + t] = __float2bfloat16_rn(pv);
      }
      for (int t = tid; t < kQT; t += kTKV) rsr[t] = q0 + t < T ? __ldg(rs + cbase + q0 + t) : 0.f;
    }
    __syncthreads();
    // ---- dP block = g v~^T, then dS^T planes
    {
      float acc[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
      for (int kb = 0; kb < kDH / 16; ++kb) {
        uint32_t a[3][4];
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          a[p][0] = G32[p * PW + (R0 + gq) * RW + 8 * kb + tq];
          a[p][1] = G32[p * PW + (R0 + gq + 8) * RW + 8 * kb + tq];
          a[p][2] = G32[p * PW + (R0 + gq) * RW + 8 * kb + 4 + tq];
          a[p][3] = G32[p * PW + (R0 + gq + 8) * RW + 8 * kb + 4 + tq];
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const uint32_t b0 = V32[(J0 + 8 * nt + gq) * RW + 8 * kb + tq];
          const uint32_t b1 = V32[(J0 + 8 * nt + gq) * RW + 8 * kb + 4 + tq];
          mma16816(acc[nt], a[2], b0, b1);
          mma16816(acc[nt], a[1], b0, b1);
          mma16816(acc[nt], a[0], b0, b1);
        }
      }
      const float dt0 = rsr[R0 + gq], dt1 = rsr[R0 + gq + 8];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int jj = J0 + 8 * nt + 2 * tq;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = R0 + gq + (e >= 2 ? 8 : 0), key = jj + (e & 1);
          const float pv = __bfloat162float(Pt[key * kVB + row]);
          const float ds = __fmul_rn(__fmul_rn(pv, __fsub_rn(acc[nt][e], e >= 2 ? dt1 : dt0)), scale);
          float hv, mv, lv;
          split3(ds, hv, mv, lv);
          St[key * kVB + row] = __float2bfloat16_rn(hv);
          St[PL + key * kVB + row] = __float2bfloat16_rn(mv);
          St[2 * PL + key * kVB + row] = __float2bfloat16_rn(lv);
        }
      }
    }
    __syncthreads();
    // ---- dk += dS^T q~ (A: dS^T planes, B: q~ rows via ldmatrix.trans);
    //      dv += p~^T g (A: p~^T, B: g planes via ldmatrix.trans)
#pragma unroll
    for (int kb = 0; kb < kQT / 16; ++kb) {
      const int rrow = 16 * kb + (lane & 15);
      if (!is_dv) {
        uint32_t a[3][4];
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          a[p][0] = S32[p * PW + (KR + gq) * RW + 8 * kb + tq];
          a[p][1] = S32[p * PW + (KR + gq + 8) * RW + 8 * kb + tq];
          a[p][2] = S32[p * PW + (KR + gq) * RW + 8 * kb + 4 + tq];
          a[p][3] = S32[p * PW + (KR + gq + 8) * RW + 8 * kb + 4 + tq];
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          uint32_t b0, b1;
          ldsm_x2_trans(b0, b1, Qb + rrow * kVB + 8 * nt);
          mma16816(accO[nt], a[2], b0, b1);
          mma16816(accO[nt], a[1], b0, b1);
          mma16816(accO[nt], a[0], b0, b1);
        }
      } else {
        uint32_t a[4];
        a[0] = P32[(KR + gq) * RW + 8 * kb + tq];
        a[1] = P32[(KR + gq + 8) * RW + 8 * kb + tq];
        a[2] = P32[(KR + gq) * RW + 8 * kb + 4 + tq];
        a[3] = P32[(KR + gq + 8) * RW + 8 * kb + 4 + tq];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          uint32_t b0[3], b1[3];
#pragma unroll
          for (int p = 0; p < 3; ++p) ldsm_x2_trans(b0[p], b1[p], Gp + p * PL + rrow * kVB + 8 * nt);
          mma16816(accO[nt], a, b0[2], b1[2]);
          mma16816(accO[nt], a, b0[1], b1[1]);
          mma16816(accO[nt], a, b0[0], b1[0]);
        }
      }
    }
  }
  // ---- write dk | dv for the tile's keys
  const int j0 = k0 + KR + gq, j1 = j0 + 8;
  const int64_t coff = (is_dv ? 2 * H : H) + hoff;
  float* base = gcat + coff;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int d = 8 * nt + 2 * tq;
    if (j0 < T) {
      *reinterpret_cast<float2*>(base + (rbase + j0) * (3 * H) + d) = make_float2(accO[nt][0], accO[nt][1]);
      if (xp) planes_store2(accO[nt][0], accO[nt][1], xp, P3, (rbase + j0) * (3 * H) + coff + d);
    }
    if (j1 < T) {
      *reinterpret_cast<float2*>(base + (rbase + j1) * (3 * H) + d) = make_float2(accO[nt][2], accO[nt][3]);
      if (xp) planes_store2(accO[nt][2], accO[nt][3], xp, P3, (rbase + j1) * (3 * H) + coff + d);
    }
  }
}

constexpr size_t kFwdSmem = ((64 + 2 * kTM) * kVS + 256) * sizeof(float);
constexpr size_t kBwdSmem = 2 * kTM * kVS * sizeof(float) + (kTM * kTM + 2 * kTM * kDH) +
                            2 * kTM * sizeof(float);
static_assert(kTM * kVS <= (64 + kTM) * kVS, "Pt fits over Q|K");
static_assert(kTM * kSS <= 2 * kTM * kVS, "dS fits over G|V");

// SLIMFIT_ATTN_TC=0 selects the FP32-FMA kernels (kept as the reference
// implementation the tensor-core path is tested against); =2 the mma.sync
// forward instead of the tcgen05 one (T <= 128); =3 tcgen05 with the one-head
// forward on three bf16 planes instead of two fp16 planes
int g_attn_impl = -1;     // -1: from the environment on first use; 0 FMA; 1 tcgen05; 2 mma.sync only; 3 tcgen05 bf16
inline int attn_impl_raw() {
  if (g_attn_impl < 0) {
    const char* e = getenv("SLIMFIT_ATTN_TC");
    g_attn_impl = (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : (e && e[0] == '3') ? 3 : 1;
  }
  return g_attn_impl;
}
inline int attn_impl() { return attn_impl_raw() == 3 ? 1 : attn_impl_raw(); }
inline bool attn_tc() { return attn_impl() != 0; }
inline bool attn_fp16() { return attn_impl_raw() != 3; }

inline bool attn_ok(int64_t B, int64_t T, int64_t heads, int64_t dh) {
  return B > 0 && T > 0 && T <= kTMW && heads > 0 && dh == kDH && B * heads <= 65535;
}
// one-head kernels up to T = 128 (T % 4 == 0); the query-tiled ones above
inline bool attn_narrow(int64_t T) { return T <= kTM && T % 4 == 0; }

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" {

int sf_attention_fwd_p(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                       int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                       void* v_codes, void* p_codes, void* ctx_planes, void* stream) {
  return sf_attention_fwd_pf(y3, bq, bk, bv, B, T, heads, dh, scale, fb, ctx, q_codes, k_codes, v_codes, p_codes,
                             ctx_planes, 0, stream);
}

int sf_attention_fwd_pf(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                        int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                        void* v_codes, void* p_codes, void* ctx_planes, int planes_format, void* stream) {
  if (planes_format < 0 || planes_format > 1) return SF_EINVAL;
  __nv_bfloat16* xp = static_cast<__nv_bfloat16*>(ctx_planes);
  if (reinterpret_cast<uintptr_t>(ctx_planes) & 7u) return SF_EINVAL;
  // ctx may be NULL when ctx_planes is given and an fp16-plane tcgen05 kernel
  // runs (impl 1): the output projection is frozen and reads only the planes
  const bool planes_only = ctx == nullptr;
  if (planes_only && (!xp || attn_impl() != 1 || !attn_fp16())) return SF_EINVAL;
  if (!y3 || !bq || !bk || !bv || !q_codes || !k_codes || !v_codes || !p_codes || fb < 0 || fb > 8 ||
      !attn_ok(B, T, heads, dh) || !aligned16(y3) || (ctx && !aligned16(ctx)) || !aligned16(bq) ||
      !aligned16(bk) || !aligned16(bv))
    return SF_EINVAL;
  for (const void* p : {q_codes, k_codes, v_codes, p_codes})
    if (reinterpret_cast<uintptr_t>(p) & 3u) return SF_EINVAL;
  static unsigned long long done_fma = 0, done_tc = 0, done_w8 = 0, done_w12 = 0;
  smem_optin(k_attn_fwd, kFwdSmem, done_fma);
  smem_optin(k_attn_fwd_tc, kFwdTcSmem, done_tc);
  if (!attn_narrow(T) && attn_impl() == 1 && attn_fp16()) {
    static unsigned long long done5wh = 0;
    const int t16 = static_cast<int>((T + 15) & ~int64_t(15));
    const size_t sm = std::max(fwd5wh_smem(t16), size_t(120) << 10);  // one CTA per SM: it takes all of TMEM
    smem_optin(k_attn_fwd_tc5wh, std::max(fwd5wh_smem(kT5W), size_t(120) << 10), done5wh);
    const dim3 grid(static_cast<unsigned>((T + 127) / 128), static_cast<unsigned>(B * heads));
    k_attn_fwd_tc5wh<<<grid, kT5, sm, as_stream(stream)>>>(
        y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb), -128.f,
        127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes), static_cast<uint32_t*>(v_codes),
        static_cast<uint8_t*>(p_codes), xp, planes_format);
    return check_launch();
  }
  if (!attn_narrow(T) && attn_impl() == 1) {
    static unsigned long long done5w = 0;
    const int t16 = static_cast<int>((T + 15) & ~int64_t(15));
    const size_t sm = std::max(fwd5w_smem(t16), size_t(120) << 10);   // one CTA per SM: it takes all of TMEM
    smem_optin(k_attn_fwd_tc5w, fwd5w_smem(kT5W) > (size_t(120) << 10) ? fwd5w_smem(kT5W) : size_t(120) << 10,
               done5w);
    const dim3 grid(static_cast<unsigned>((T + 127) / 128), static_cast<unsigned>(B * heads));
    k_attn_fwd_tc5w<<<grid, kT5, sm, as_stream(stream)>>>(
        y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb), -128.f,
        127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes), static_cast<uint32_t*>(v_codes),
        static_cast<uint8_t*>(p_codes), xp, planes_format);
    return check_launch();
  }
  if (!attn_narrow(T)) {
    const dim3 grid(static_cast<unsigned>((T + kQT - 1) / kQT), static_cast<unsigned>(B * heads));
    const float qsc = static_cast<float>(1 << fb);
    if (T <= 256) {
      smem_optin(k_attn_fwd_wide<8>, fwd_wide_smem<8>(), done_w8);
      k_attn_fwd_wide<8><<<grid, kTW, fwd_wide_smem<8>(), as_stream(stream)>>>(
          y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, qsc, -128.f, 127.f, ctx,
          static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes), static_cast<uint32_t*>(v_codes),
          static_cast<uint8_t*>(p_codes), xp, planes_format);
    } else {
      smem_optin(k_attn_fwd_wide<12>, fwd_wide_smem<12>(), done_w12);
      k_attn_fwd_wide<12><<<grid, kTW, fwd_wide_smem<12>(), as_stream(stream)>>>(
          y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, qsc, -128.f, 127.f, ctx,
          static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes), static_cast<uint32_t*>(v_codes),
          static_cast<uint8_t*>(p_codes), xp, planes_format);
    }
    return check_launch();
  }
  if (attn_impl() == 1 && attn_fp16()) {
    static unsigned long long done5h = 0;
    smem_optin(k_attn_fwd_tc5h, kFwdHSmem, done5h);
    k_attn_fwd_tc5h<<<static_cast<unsigned>(B * heads), kTH, kFwdHSmem, as_stream(stream)>>>(
        y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb),
        -128.f, 127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes),
        static_cast<uint32_t*>(v_codes), static_cast<uint8_t*>(p_codes), xp, planes_format);
    return check_launch();
  }
  if (attn_impl() == 1) {
    static unsigned long long done5 = 0;
    smem_optin(k_attn_fwd_tc5, kFwd5Smem, done5);
    k_attn_fwd_tc5<<<static_cast<unsigned>(B * heads), kT5, kFwd5Smem, as_stream(stream)>>>(
        y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb),
        -128.f, 127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes),
        static_cast<uint32_t*>(v_codes), static_cast<uint8_t*>(p_codes), xp, planes_format);
    return check_launch();
  }
  if (attn_tc()) {
    k_attn_fwd_tc<<<static_cast<unsigned>(B * heads), kTF, kFwdTcSmem, as_stream(stream)>>>(
        y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb),
        -128.f, 127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes),
        static_cast<uint32_t*>(v_codes), static_cast<uint16_t*>(p_codes), xp, planes_format);
    return check_launch();
  }
  const dim3 grid(static_cast<unsigned>((T + 63) / 64), static_cast<unsigned>(B * heads));
  k_attn_fwd<<<grid, kFT, kFwdSmem, as_stream(stream)>>>(
      y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb), -128.f,
      127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes),
      static_cast<uint32_t*>(v_codes), static_cast<uint32_t*>(p_codes), xp, planes_format);
  return check_launch();
}

int sf_attention_fwd(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                     int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                     void* v_codes, void* p_codes, void* stream) {
  return sf_attention_fwd_p(y3, bq, bk, bv, B, T, heads, dh, scale, fb, ctx, q_codes, k_codes, v_codes, p_codes,
                            nullptr, stream);
}

int sf_attention_set_impl(int tensor_cores) {
  if (tensor_cores < 0 || tensor_cores > 3) return SF_EINVAL;
  g_attn_impl = tensor_cores;
  return SF_OK;
}

size_t sf_attention_bwd_workspace_bytes(int64_t B, int64_t T, int64_t heads) {
  if (B <= 0 || T <= 0 || heads <= 0 || attn_narrow(T)) return 0;
  return static_cast<size_t>(B * heads * T) * sizeof(float);      // row sums of dP p~
}

int sf_attention_bwd_p(const float* g, const void* q_codes, const void* k_codes, const void* v_codes,
                       const void* p_codes, int64_t B, int64_t T, int64_t heads, int64_t dh, float scale, int fb,
                       float* gcat, void* ws, void* gcat_planes, void* stream) {
  __nv_bfloat16* xp = static_cast<__nv_bfloat16*>(gcat_planes);
  if (reinterpret_cast<uintptr_t>(gcat_planes) & 7u) return SF_EINVAL;
  if (!g || !gcat || !q_codes || !k_codes || !v_codes || !p_codes || fb < 0 || fb > 8 ||
      !attn_ok(B, T, heads, dh) || !aligned16(g) || !aligned16(gcat))
    return SF_EINVAL;
  for (const void* p : {q_codes, k_codes, v_codes, p_codes})
    if (reinterpret_cast<uintptr_t>(p) & 3u) return SF_EINVAL;
  if (!attn_narrow(T)) {
    if (!ws) return SF_EINVAL;
    static unsigned long long done_q8 = 0, done_q12 = 0, done_kv = 0;
    const dim3 grid(static_cast<unsigned>((T + kQT - 1) / kQT), static_cast<unsigned>(B * heads));
    const float iv = 1.0f / static_cast<float>(1 << fb);
    float* rsw = static_cast<float*>(ws);
    if (attn_impl() == 1 && !xp) {
      static unsigned long long done5q = 0, done5kv = 0;
      const int t16 = static_cast<int>((T + 15) & ~int64_t(15));
      const size_t smq = std::max(bwdq5w_smem(t16), size_t(120) << 10);   // one CTA per SM: all of TMEM
      smem_optin(k_attn_bwdq_tc5w, bwdq5w_smem(kT5W), done5q);
      smem_optin(k_attn_bwdkv_tc5w, kBwdKv5wSmem, done5kv);
      const dim3 grid5(static_cast<unsigned>((T + 127) / 128), static_cast<unsigned>(B * heads));
      k_attn_bwdq_tc5w<<<grid5, kT5, smq, as_stream(stream)>>>(
          g, static_cast<const uint32_t*>(k_codes), static_cast<const uint32_t*>(v_codes),
          static_cast<const uint8_t*>(p_codes), static_cast<int>(T), static_cast<int>(heads), scale, iv, gcat, rsw);
      k_attn_bwdkv_tc5w<<<grid5, kT5, kBwdKv5wSmem, as_stream(stream)>>>(
          g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(v_codes),
          static_cast<const uint8_t*>(p_codes), rsw, static_cast<int>(T), static_cast<int>(heads), scale, iv, gcat);
      return check_launch();
    }
    if (T <= 256) {
      smem_optin(k_attn_bwdq_wide<8>, bwdq_wide_smem<8>(), done_q8);
      k_attn_bwdq_wide<8><<<grid, kTW, bwdq_wide_smem<8>(), as_stream(stream)>>>(
          g, static_cast<const uint32_t*>(k_codes), static_cast<const uint32_t*>(v_codes),
          static_cast<const uint8_t*>(p_codes), static_cast<int>(T), static_cast<int>(heads), scale, iv, gcat, rsw, xp);
    } else {
      smem_optin(k_attn_bwdq_wide<12>, bwdq_wide_smem<12>(), done_q12);
      k_attn_bwdq_wide<12><<<grid, kTW, bwdq_wide_smem<12>(), as_stream(stream)>>>(
          g, static_cast<const uint32_t*>(k_codes), static_cast<const uint32_t*>(v_codes),
          static_cast<const uint8_t*>(p_codes), static_cast<int>(T), static_cast<int>(heads), scale, iv, gcat, rsw, xp);
    }
    smem_optin(k_attn_bwdkv_wide, kBwdKvSmem, done_kv);
    k_attn_bwdkv_wide<<<grid, kTKV, kBwdKvSmem, as_stream(stream)>>>(
        g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(v_codes),
        static_cast<const uint8_t*>(p_codes), rsw, static_cast<int>(T), static_cast<int>(heads), scale, iv, gcat, xp);
    return check_launch();
  }
  if (attn_impl() == 1 && !xp && attn_fp16()) {
    static unsigned long long done5h = 0;
    smem_optin(k_attn_bwd_tc5h, kBwdHSmem, done5h);
    k_attn_bwd_tc5h<<<static_cast<unsigned>(B * heads), kTH, kBwdHSmem, as_stream(stream)>>>(
        g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(k_codes),
        static_cast<const uint32_t*>(v_codes), static_cast<const uint8_t*>(p_codes), static_cast<int>(T),
        static_cast<int>(heads), scale, 1.0f / static_cast<float>(1 << fb), gcat);
    return check_launch();
  }
  if (attn_impl() == 1 && !xp) {
    static unsigned long long done5 = 0;
    smem_optin(k_attn_bwd_tc5, kBwd5SmemP, done5);
    const int64_t nbh = B * heads;
    k_attn_bwd_tc5<<<static_cast<unsigned>(nbh < num_sms() ? nbh : num_sms()), kT5, kBwd5SmemP, as_stream(stream)>>>(
        g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(k_codes),
        static_cast<const uint32_t*>(v_codes), static_cast<const uint8_t*>(p_codes), static_cast<int>(T),
        static_cast<int>(heads), scale, 1.0f / static_cast<float>(1 << fb), gcat, static_cast<int>(nbh));
    return check_launch();
  }
  static unsigned long long done_fma = 0, done_tc = 0;
  smem_optin(k_attn_bwd, kBwdSmem, done_fma);
  smem_optin(k_attn_bwd_tc, kBwdTcSmem, done_tc);
  if (attn_tc()) {
    k_attn_bwd_tc<<<static_cast<unsigned>(B * heads), kTB, kBwdTcSmem, as_stream(stream)>>>(
        g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(k_codes),
        static_cast<const uint32_t*>(v_codes), static_cast<const uint32_t*>(p_codes), static_cast<int>(T),
        static_cast<int>(heads), scale, 1.0f / static_cast<float>(1 << fb), gcat, xp);
    return check_launch();
  }
  k_attn_bwd<<<static_cast<unsigned>(B * heads), kBT, kBwdSmem, as_stream(stream)>>>(
      g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(k_codes),
      static_cast<const uint32_t*>(v_codes), static_cast<const uint32_t*>(p_codes), static_cast<int>(T),
      static_cast<int>(heads), scale, 1.0f / static_cast<float>(1 << fb), gcat, xp);
  return check_launch();
}

int sf_attention_bwd(const float* g, const void* q_codes, const void* k_codes, const void* v_codes,
                     const void* p_codes, int64_t B, int64_t T, int64_t heads, int64_t dh, float scale, int fb,
                     float* gcat, void* ws, void* stream) {
  return sf_attention_bwd_p(g, q_codes, k_codes, v_codes, p_codes, B, T, heads, dh, scale, fb, gcat, ws, nullptr,
                            stream);
}

}  // extern "C"
