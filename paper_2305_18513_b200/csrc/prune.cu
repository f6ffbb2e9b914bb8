// K6 prune_topk / K7 restore: global top-k by magnitude with stable ties.
//
// Reference: prune_topk / restore (compression.py:137-169), used by the
// frozen-LayerNorm x~ cache (tensor.py:471-477, :482).
//
// Keys are order-preserving uint32 images of the ranking value with NaN
// mapped strictly below everything (numpy's argsort of -key puts NaN last)
// and -0.0 folded onto +0.0 (they compare equal, so they tie):
//   magnitude: u = (bits & 0x7FFFFFFF) + 1, NaN -> 0
//   signed:    u = bits ^ (sign ? 0xFFFFFFFF : 0x80000000), NaN -> 0
//
// Two passes over x (the second normally served from L2) plus small
// candidate work, no host round trip:
//  P1  15-bit digit histogram (u >> 17) in 128 KB of shared memory, one CTA
//      per SM; the last CTA picks the digit D that holds rank k from the top.
//  P2  per 4096-element tile: count keys above D (-> tile_gt) and compact the
//      keys of digit D ("candidates", (key, index)) with one global atomic
//      per CTA; a 9-bit histogram of the candidates' next digit; its last CTA
//      picks that digit D9.
//  P3  over the candidates: those above D9 bump their tile's count; those in
//      D9 go to a small list; the last CTA selects the exact threshold T
//      from the small list, adds the (> T, == T) counts of the small list to
//      their tiles and scans the tile counts into output offsets.
//  P4  write pass: warp ballots over coalesced loads emit every u > T and
//      the first k - #(u > T) elements with u == T, in index order.
// Fallbacks keep it exact for any input: if digit D holds more candidates
// than the buffer takes (heavy ties), the last CTA of P1 finishes the
// selection itself by scanning x and P2 counts tiles against the final T; if
// D9 holds more than the small list takes, P3's last CTA scans the
// candidate buffer instead.
#include "common.cuh"

namespace sf {

constexpr int kPT = 256;                 // threads per CTA (tile passes)
constexpr int kRows = 16;                // elements per lane per tile
constexpr int kTile = kPT * kRows;       // 4096 elements per tile (512 per warp)
constexpr int kD15 = 1 << 15;            // P1 digit bins
constexpr int kH1T = 1024;               // P1 threads per CTA
constexpr int kSmallCap = 4096;          // exact-select list capacity

struct PruneState {
  unsigned int ticket[4];
  unsigned int d15, d9, T;
  int mode;                       // 0 fast, 1 = T known after P1 (tie fallback)
  unsigned int cand_count, small_count;
  unsigned long long above15;     // keys with digit15 > d15
  unsigned long long need15;      // rank (from the top) inside digit d15
  unsigned long long need9;       // rank inside (d15, d9)
  unsigned long long need_eq;     // keys == T to keep, in index order
  unsigned int hist9[512];
  unsigned int hist15[kD15];
};

__device__ __forceinline__ uint32_t rank_key(float x, bool mag) {
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7FFFFFFFu) > 0x7F800000u) return 0u;   // NaN ranks lowest
  if (mag) return (b & 0x7FFFFFFFu) + 1u;
  if (b == 0x80000000u) b = 0u;                     // -0.0 ties with +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ bool last_cta(unsigned int* ticket) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Among `nb` bins (bin index = digit, larger digit = larger keys) find the
// digit holding rank `need` (1-based from the top).  All threads of the CTA
// call it; returns the digit and the count strictly above it.
__device__ void select_digit(const volatile unsigned int* hist, int nb, unsigned long long need,
                             unsigned int& digit, unsigned long long& above) {
  __shared__ unsigned long long tsum[1024];
  __shared__ unsigned int s_digit;
  __shared__ unsigned long long s_above;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  unsigned long long s = 0;
  for (int j = 0; j < per && b0 + j < nb; ++j) s += hist[b0 + j];
  tsum[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long ab = 0;
    int t = blockDim.x - 1;
    while (t > 0 && ab + tsum[t] < need) ab += tsum[t--];
    int d = min(nb, (t + 1) * per) - 1;
    while (d > t * per && ab + hist[d] < need) ab += hist[d--];
    s_digit = static_cast<unsigned int>(d);
    s_above = ab;
  }
  __syncthreads();
  digit = s_digit;
  above = s_above;
}

// Exact k-th largest key among keys matching (prefix, mask), by 8-bit MSD
// radix over the remaining bits, scanning `src` with one CTA.  Used only by
// the fallbacks.  `need` is the rank (1-based from the top) among matches.
template <typename Getter>
__device__ void cta_select(Getter get, int64_t count, uint32_t prefix, uint32_t mask,
                           unsigned long long need, uint32_t& T, unsigned long long& need_eq) {
  __shared__ unsigned int h[256];
  for (int shift = 24; shift >= 0; shift -= 8) {
    if (((mask >> shift) & 0xFFu) == 0xFFu) continue;   // byte already fixed
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
      const uint32_t u = get(i);
      if ((u & mask) == prefix) atomicAdd(h + ((u >> shift) & 0xFFu), 1u);
    }
    __syncthreads();
    unsigned int d;
    unsigned long long above;
    select_digit(h, 256, need, d, above);
    prefix |= d << shift;
    mask |= 0xFFu << shift;
    need -= above;
    __syncthreads();
  }
  T = prefix;
  need_eq = need;
}

// ------------------------------------------------------------------ P1

__global__ void __launch_bounds__(kH1T) k_p1(const float* __restrict__ x, int64_t n, bool mag,
                                             unsigned long long k, unsigned long long cap,
                                             PruneState* st) {
  extern __shared__ unsigned int sh[];     // kD15 bins
  for (int i = threadIdx.x; i < kD15; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t S = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = aligned16(x) ? n / 4 : 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + S < n4; i += 2 * S) {
    const float4 a = ld_stream(x4 + i), b = ld_stream(x4 + i + S);
    atomicAdd(sh + (rank_key(a.x, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.y, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.z, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.w, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(b.x, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(b.y, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(b.z, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(b.w, mag) >> 17), 1u);
  }
  for (; i < n4; i += S) {
    const float4 a = ld_stream(x4 + i);
    atomicAdd(sh + (rank_key(a.x, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.y, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.z, mag) >> 17), 1u);
    atomicAdd(sh + (rank_key(a.w, mag) >> 17), 1u);
  }
  for (int64_t j = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += S)
    atomicAdd(sh + (rank_key(x[j], mag) >> 17), 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kD15; b += blockDim.x)
    if (sh[b]) atomicAdd(st->hist15 + b, sh[b]);
  if (!last_cta(&st->ticket[0])) return;
  unsigned int d;
  unsigned long long above;
  select_digit(st->hist15, kD15, k, d, above);
  if (threadIdx.x == 0) {
    st->d15 = d;
    st->above15 = above;
    st->need15 = k - above;
  }
  const unsigned long long ncand = *(volatile unsigned int*)(st->hist15 + d);
  if (ncand <= cap) return;
  // Tie fallback: digit d holds more keys than the candidate buffer; finish
  // the exact selection here by scanning x (slow, only for tie-heavy input).
  uint32_t T;
  unsigned long long need_eq;
  cta_select([&](int64_t j) { return rank_key(x[j], mag); }, n, d << 17, 0xFFFE0000u, k - above, T,
             need_eq);
  if (threadIdx.x == 0) {
    st->T = T;
    st->need_eq = need_eq;
    st->mode = 1;
  }
}

// ------------------------------------------------------------------ P2

__device__ __forceinline__ unsigned int block_sum(unsigned int v, unsigned int* sh_w) {
  v = __reduce_add_sync(0xFFFFFFFFu, v);
  if ((threadIdx.x & 31) == 0) sh_w[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned int t = 0;
  for (int w = 0; w < kPT / 32; ++w) t += sh_w[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kPT) k_p2(const float* __restrict__ x, int64_t n, bool mag,
                                            PruneState* st, unsigned int* __restrict__ tile_gt,
                                            unsigned int* __restrict__ tile_eq,
                                            uint2* __restrict__ cands) {
  const int mode = st->mode;
  const uint32_t d15 = st->d15, T = st->T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = static_cast<int64_t>(blockIdx.x) * kTile + warp * (32 * kRows);
  const unsigned lt = (1u << lane) - 1u;
  __shared__ unsigned int sh_w[kPT / 32];
  __shared__ unsigned int h9[512];
  __shared__ unsigned int s_base;
  for (int i = threadIdx.x; i < 512; i += kPT) h9[i] = 0;
  uint32_t u[kRows];
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    u[j] = i < n ? rank_key(__ldg(x + i), mag) : 0u;
  }
  unsigned int gt = 0, eq = 0, mine = 0;
  if (mode == 1) {              // T already known: count against it directly
#pragma unroll
    for (int j = 0; j < kRows; ++j) {
      const bool in = wbase + 32 * j + lane < n;
      gt += in && u[j] > T;
      eq += in && u[j] == T;
    }
    gt = block_sum(gt, sh_w);
    eq = block_sum(eq, sh_w);
    if (threadIdx.x == 0) {
      tile_gt[blockIdx.x] = gt;
      tile_eq[blockIdx.x] = eq;
    }
    return;
  }
  // fast mode: count above digit d15, compact digit-d15 candidates
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const bool in = wbase + 32 * j + lane < n;
    gt += in && (u[j] >> 17) > d15;
    mine += in && (u[j] >> 17) == d15;
  }
  __syncthreads();
  // per-warp candidate counts -> block offsets -> one global reservation
  const unsigned int wc = __reduce_add_sync(0xFFFFFFFFu, mine);
  if (lane == 0) sh_w[warp] = wc;
  __syncthreads();
  unsigned int wofs = 0, tot = 0;
  for (int w = 0; w < kPT / 32; ++w) {
    if (w < warp) wofs += sh_w[w];
    tot += sh_w[w];
  }
  if (threadIdx.x == 0) s_base = tot ? atomicAdd(&st->cand_count, tot) : 0u;
  __syncthreads();
  unsigned int pos = s_base + wofs;
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    const bool c = i < n && (u[j] >> 17) == d15;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, c);
    if (c) {
      cands[pos + __popc(m & lt)] = make_uint2(u[j], static_cast<unsigned int>(i));
      atomicAdd(h9 + ((u[j] >> 8) & 0x1FFu), 1u);
    }
    pos += __popc(m);
  }
  gt = block_sum(gt, sh_w);
  if (threadIdx.x == 0) {
    tile_gt[blockIdx.x] = gt;
    tile_eq[blockIdx.x] = 0;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 512; b += kPT)
    if (h9[b]) atomicAdd(st->hist9 + b, h9[b]);
  if (!last_cta(&st->ticket[1])) return;
  unsigned int d;
  unsigned long long above;
  select_digit(st->hist9, 512, st->need15, d, above);
  if (threadIdx.x == 0) {
    st->d9 = d;
    st->need9 = st->need15 - above;
  }
}

// ------------------------------------------------------------------ P3

__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long* sh_warp,
                                                                   unsigned long long& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh_warp[warp] = inc;
  __syncthreads();
  unsigned long long base = 0, tot = 0;
  for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) {
    if (w < warp) base += sh_warp[w];
    tot += sh_warp[w];
  }
  __syncthreads();
  total = tot;
  return base + inc - v;
}

__global__ void __launch_bounds__(kPT) k_p3(PruneState* st, const uint2* __restrict__ cands,
                                            uint2* __restrict__ small,
                                            unsigned int* __restrict__ tile_gt,
                                            unsigned int* __restrict__ tile_eq, int64_t ntiles,
                                            unsigned long long* __restrict__ out_off,
                                            unsigned long long* __restrict__ eq_before) {
  const int mode = st->mode;
  if (mode == 0) {
    const uint32_t d9 = st->d9;
    const unsigned int nc = st->cand_count;
    for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
      const uint2 c = cands[i];
      const uint32_t dig = (c.x >> 8) & 0x1FFu;
      if (dig > d9) {
        atomicAdd(tile_gt + c.y / kTile, 1u);
      } else if (dig == d9) {
        const unsigned int p = atomicAdd(&st->small_count, 1u);
        if (p < kSmallCap) small[p] = c;
      }
    }
  }
  if (!last_cta(&st->ticket[2])) return;
  if (mode == 0) {
    // exact threshold among the (d15, d9) candidates: final 8 bits
    const unsigned int ns = *(volatile unsigned int*)&st->small_count;
    const uint32_t prefix = (st->d15 << 17) | (st->d9 << 8);
    uint32_t T;
    unsigned long long need_eq;
    if (ns <= kSmallCap) {
      cta_select([&](int64_t j) { return small[j].x; }, ns, prefix, 0xFFFFFF00u, st->need9, T,
                 need_eq);
      for (unsigned int j = threadIdx.x; j < ns; j += blockDim.x) {
        const uint2 c = small[j];
        if (c.x > T) atomicAdd(tile_gt + c.y / kTile, 1u);
        if (c.x == T) atomicAdd(tile_eq + c.y / kTile, 1u);
      }
    } else {   // small list overflowed (ties): work from the full candidate list
      const unsigned int nc = *(volatile unsigned int*)&st->cand_count;
      cta_select([&](int64_t j) { return cands[j].x; }, nc, prefix, 0xFFFFFF00u, st->need9, T,
                 need_eq);
      for (unsigned int j = threadIdx.x; j < nc; j += blockDim.x) {
        const uint2 c = cands[j];
        if ((c.x & 0xFFFFFF00u) != prefix) continue;
        if (c.x > T) atomicAdd(tile_gt + c.y / kTile, 1u);
        if (c.x == T) atomicAdd(tile_eq + c.y / kTile, 1u);
      }
    }
    if (threadIdx.x == 0) {
      st->T = T;
      st->need_eq = need_eq;
    }
    __threadfence();
    __syncthreads();
  }
  // scan the tile counts: each thread owns a contiguous run of tiles
  const unsigned long long need_eq = *(volatile unsigned long long*)&st->need_eq;
  const int64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
  const volatile unsigned int* vg = tile_gt;
  const volatile unsigned int* ve = tile_eq;
  unsigned long long my_gt = 0, my_eq = 0;
  for (int64_t t = t0; t < t1; ++t) {
    my_gt += vg[t];
    my_eq += ve[t];
  }
  __shared__ unsigned long long sw[kPT / 32];
  unsigned long long tot;
  unsigned long long gb = block_exclusive_scan(my_gt, sw, tot);
  unsigned long long eb = block_exclusive_scan(my_eq, sw, tot);
  for (int64_t t = t0; t < t1; ++t) {
    eq_before[t] = eb;
    out_off[t] = gb + (eb < need_eq ? eb : need_eq);
    gb += vg[t];
    eb += ve[t];
  }
}

// ------------------------------------------------------------------ P4

// Warp w of the tile owns elements [base + 512 w, +512); lane l holds
// base + 512 w + 32 j + l (j = 0..15): each load is one coalesced 128 B line
// and (j, l) order is index order, so warp ballots give every kept element
// its output slot directly.
__global__ void __launch_bounds__(kPT) k_p4(const float* __restrict__ x, int64_t n, bool mag,
                                            const PruneState* __restrict__ st,
                                            const unsigned long long* __restrict__ out_off,
                                            const unsigned long long* __restrict__ eq_before,
                                            float* __restrict__ values,
                                            int32_t* __restrict__ indices) {
  const uint32_t T = st->T;
  const unsigned long long need_eq = st->need_eq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = static_cast<int64_t>(blockIdx.x) * kTile + warp * (32 * kRows);
  const unsigned lt = (1u << lane) - 1u;
  float v[kRows];
  uint32_t u[kRows];
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    v[j] = i < n ? __ldg(x + i) : 0.f;
    u[j] = i < n ? rank_key(v[j], mag) : 0u;
  }
  unsigned int wgt = 0, weq = 0;
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    wgt += __popc(__ballot_sync(0xFFFFFFFFu, i < n && u[j] > T));
    weq += __popc(__ballot_sync(0xFFFFFFFFu, i < n && u[j] == T));
  }
  __shared__ unsigned int s_gt[kPT / 32], s_eq[kPT / 32];
  if (lane == 0) {
    s_gt[warp] = wgt;
    s_eq[warp] = weq;
  }
  __syncthreads();
  const unsigned long long eq_tile0 = eq_before[blockIdx.x];
  unsigned long long eq_run = eq_tile0, gt_run = 0;
  for (int w = 0; w < warp; ++w) {
    gt_run += s_gt[w];
    eq_run += s_eq[w];
  }
  const unsigned long long kept_eq_tile0 = eq_tile0 < need_eq ? eq_tile0 : need_eq;
  unsigned long long pos = out_off[blockIdx.x] + gt_run +
                           ((eq_run < need_eq ? eq_run : need_eq) - kept_eq_tile0);
#pragma unroll
  for (int j = 0; j < kRows; ++j) {
    const int64_t i = wbase + 32 * j + lane;
    const bool valid = i < n;
    const bool is_eq = valid && u[j] == T;
    const unsigned eqm = __ballot_sync(0xFFFFFFFFu, is_eq);
    const unsigned long long my_eq_rank = eq_run + __popc(eqm & lt);
    const bool keep = valid && (u[j] > T || (is_eq && my_eq_rank < need_eq));
    const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
    if (keep) {
      const unsigned long long o = pos + __popc(km & lt);
      values[o] = v[j];
      indices[o] = static_cast<int32_t>(i);
    }
    pos += __popc(km);
    eq_run += __popc(eqm);
  }
}

// ------------------------------------------------------------------ K7

// first position j in [0, k) with indices[j] >= target, 32-way warp search
__device__ int64_t warp_lower_bound(const int32_t* __restrict__ idx, int64_t k, int64_t target) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = k;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t pos = lo + lane * step;
    const bool below = pos < hi && static_cast<int64_t>(__ldg(idx + pos)) < target;
    const int nb = __popc(__ballot_sync(0xFFFFFFFFu, below));   // probes below: a prefix
    const int64_t nlo = nb == 0 ? lo : lo + (nb - 1) * step + 1;
    const int64_t nhi = nb == 32 ? hi : min(hi, lo + nb * step);
    lo = nlo;
    hi = max(nlo, nhi);
  }
  const int64_t pos = lo + lane;
  const bool below = pos < hi && static_cast<int64_t>(__ldg(idx + pos)) < target;
  return lo + __popc(__ballot_sync(0xFFFFFFFFu, below));
}

// dense = 0 with survivors scattered in.  Each CTA owns a tile of the dense
// output; warp 0 finds the tile's slice of the ascending index list (32-way
// search), all threads write zeros with float4 stores, then scatter.
__global__ void __launch_bounds__(kPT) k_restore(const float* __restrict__ values,
                                                 const int32_t* __restrict__ indices, int64_t k,
                                                 float* __restrict__ dense, int64_t n) {
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t t1 = min(n, t0 + kTile);
  __shared__ int64_t range[2];
  if (threadIdx.x < 32) {
    const int64_t a = warp_lower_bound(indices, k, t0);
    const int64_t b = warp_lower_bound(indices, k, t1);
    if (threadIdx.x == 0) {
      range[0] = a;
      range[1] = b;
    }
  }
  if (aligned16(dense) && t1 - t0 == kTile) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = threadIdx.x; i < kTile / 4; i += blockDim.x)
      reinterpret_cast<float4*>(dense + t0)[i] = z;
  } else {
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) dense[i] = 0.f;
  }
  __syncthreads();
  for (int64_t j = range[0] + threadIdx.x; j < range[1]; j += blockDim.x)
    dense[__ldg(indices + j)] = __ldg(values + j);
}

inline int64_t ntiles_of(int64_t n) { return (n + kTile - 1) / kTile; }
inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
inline int64_t cand_cap(int64_t n) { return n / 8 + 4096; }

}  // namespace sf

using namespace sf;

extern "C" {

size_t sf_prune_workspace_bytes(int64_t n) {
  const int64_t nn = n > 0 ? n : 1;
  const int64_t nt = ntiles_of(nn);
  return align256(sizeof(PruneState)) + 2 * align256(nt * sizeof(unsigned int)) +
         2 * align256(nt * sizeof(unsigned long long)) +
         align256(static_cast<size_t>(cand_cap(nn)) * sizeof(uint2)) +
         align256(kSmallCap * sizeof(uint2));
}

int sf_prune_topk(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                  int32_t* indices, void* ws, void* stream) {
  if (n <= 0 || k < 1 || k > n || n > 0x7FFFFFFFLL || !x || !values || !indices || !ws)
    return SF_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int64_t nt = ntiles_of(n);
  char* w = static_cast<char*>(ws);
  PruneState* st = reinterpret_cast<PruneState*>(w);
  w += align256(sizeof(PruneState));
  unsigned int* tile_gt = reinterpret_cast<unsigned int*>(w);
  w += align256(nt * sizeof(unsigned int));
  unsigned int* tile_eq = reinterpret_cast<unsigned int*>(w);
  w += align256(nt * sizeof(unsigned int));
  unsigned long long* out_off = reinterpret_cast<unsigned long long*>(w);
  w += align256(nt * sizeof(unsigned long long));
  unsigned long long* eq_before = reinterpret_cast<unsigned long long*>(w);
  w += align256(nt * sizeof(unsigned long long));
  uint2* cands = reinterpret_cast<uint2*>(w);
  w += align256(static_cast<size_t>(cand_cap(n)) * sizeof(uint2));
  uint2* small = reinterpret_cast<uint2*>(w);

  if (cudaMemsetAsync(st, 0, sizeof(PruneState), s) != cudaSuccess) return check_launch();
  const bool mag = by_magnitude != 0;
  const size_t smem1 = kD15 * sizeof(unsigned int);
  cudaFuncSetAttribute(k_p1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem1));
  const unsigned g1 = static_cast<unsigned>(num_sms());
  k_p1<<<g1, kH1T, smem1, s>>>(x, n, mag, static_cast<unsigned long long>(k),
                               static_cast<unsigned long long>(cand_cap(n)), st);
  k_p2<<<static_cast<unsigned>(nt), kPT, 0, s>>>(x, n, mag, st, tile_gt, tile_eq, cands);
  const unsigned g3 = grid_for(cand_cap(n), kPT, 2);
  k_p3<<<g3, kPT, 0, s>>>(st, cands, small, tile_gt, tile_eq, nt, out_off, eq_before);
  k_p4<<<static_cast<unsigned>(nt), kPT, 0, s>>>(x, n, mag, st, out_off, eq_before, values, indices);
  return check_launch();
}

int sf_restore(const float* values, const int32_t* indices, int64_t k, float* dense, int64_t n,
               void* stream) {
  if (n <= 0 || k < 0 || k > n || !dense || (k > 0 && (!values || !indices))) return SF_EINVAL;
  k_restore<<<static_cast<unsigned>(ntiles_of(n)), kPT, 0, as_stream(stream)>>>(values, indices, k,
                                                                               dense, n);
  return check_launch();
}

}  // extern "C"
