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
// Limits: head dim 64, T <= 128, T % 4 == 0 (BERT/ViT shapes); the host
// keeps the unfused path for anything else.
#include "common.cuh"

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
    uint32_t* __restrict__ vc, uint32_t* __restrict__ pc) {
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
  }
}

// ------------------------------------------------------------------ backward
// grid (B * h); CTA = one head, 512 threads.
// smem: region A = [G 128 x kVS | V~ 128 x kVS]  (reused as dS 128 x kSS)
//       Pc 128 x 128 bytes, Qc / Kc 128 x 64 bytes, row dots.
__global__ void __launch_bounds__(kBT, 1) k_attn_bwd(
    const float* __restrict__ g, const uint32_t* __restrict__ qc, const uint32_t* __restrict__ kc,
    const uint32_t* __restrict__ vc, const uint32_t* __restrict__ pc, int T, int h, float scale,
    float inv, float* __restrict__ gcat) {
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
      if (j < T)
        st4s(gcat + (rbase + j) * (3 * H) + 2 * H + hoff + dc,
             make_float4(o[i][0], o[i][1], o[i][2], o[i][3]));
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
    }
  }
}

constexpr size_t kFwdSmem = ((64 + 2 * kTM) * kVS + 256) * sizeof(float);
constexpr size_t kBwdSmem = 2 * kTM * kVS * sizeof(float) + (kTM * kTM + 2 * kTM * kDH) +
                            2 * kTM * sizeof(float);
static_assert(kTM * kVS <= (64 + kTM) * kVS, "Pt fits over Q|K");
static_assert(kTM * kSS <= 2 * kTM * kVS, "dS fits over G|V");

inline bool attn_ok(int64_t B, int64_t T, int64_t heads, int64_t dh) {
  return B > 0 && T > 0 && T <= kTM && T % 4 == 0 && heads > 0 && dh == kDH && B * heads <= 65535;
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" {

int sf_attention_fwd(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                     int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                     void* v_codes, void* p_codes, void* stream) {
  if (!y3 || !bq || !bk || !bv || !ctx || !q_codes || !k_codes || !v_codes || !p_codes || fb < 0 || fb > 8 ||
      !attn_ok(B, T, heads, dh) || !aligned16(y3) || !aligned16(ctx) || !aligned16(bq) || !aligned16(bk) ||
      !aligned16(bv))
    return SF_EINVAL;
  for (const void* p : {q_codes, k_codes, v_codes, p_codes})
    if (reinterpret_cast<uintptr_t>(p) & 3u) return SF_EINVAL;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFwdSmem));
    attr = true;
  }
  const dim3 grid(static_cast<unsigned>((T + 63) / 64), static_cast<unsigned>(B * heads));
  k_attn_fwd<<<grid, kFT, kFwdSmem, as_stream(stream)>>>(
      y3, bq, bk, bv, static_cast<int>(T), static_cast<int>(heads), scale, static_cast<float>(1 << fb), -128.f,
      127.f, ctx, static_cast<uint32_t*>(q_codes), static_cast<uint32_t*>(k_codes),
      static_cast<uint32_t*>(v_codes), static_cast<uint32_t*>(p_codes));
  return check_launch();
}

int sf_attention_bwd(const float* g, const void* q_codes, const void* k_codes, const void* v_codes,
                     const void* p_codes, int64_t B, int64_t T, int64_t heads, int64_t dh, float scale, int fb,
                     float* gcat, void* stream) {
  if (!g || !gcat || !q_codes || !k_codes || !v_codes || !p_codes || fb < 0 || fb > 8 ||
      !attn_ok(B, T, heads, dh) || !aligned16(g) || !aligned16(gcat))
    return SF_EINVAL;
  for (const void* p : {q_codes, k_codes, v_codes, p_codes})
    if (reinterpret_cast<uintptr_t>(p) & 3u) return SF_EINVAL;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kBwdSmem));
    attr = true;
  }
  k_attn_bwd<<<static_cast<unsigned>(B * heads), kBT, kBwdSmem, as_stream(stream)>>>(
      g, static_cast<const uint32_t*>(q_codes), static_cast<const uint32_t*>(k_codes),
      static_cast<const uint32_t*>(v_codes), static_cast<const uint32_t*>(p_codes), static_cast<int>(T),
      static_cast<int>(heads), scale, 1.0f / static_cast<float>(1 << fb), gcat);
  return check_launch();
}

}  // extern "C"
