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
// The k-th largest key T comes from an 11/11/10-bit MSD radix select: three
// histogram passes, each finished by the last CTA to arrive (no host round
// trip).  Histogram increments are aggregated per warp (match.any: one
// shared-memory atomic per distinct digit per warp), which matters because
// the digits of a standardized activation concentrate in a few bins.  A
// tile pass then counts (#u > T, #u == T) per 4096-element tile and its last
// CTA scans the tile counts; the write pass emits every u > T plus the
// first k - #(u > T) elements with u == T in index order (stable ties),
// using warp ballots over coalesced loads so output order is index order.
#include "common.cuh"

namespace sf {

constexpr int kPT = 256;                 // threads per CTA
constexpr int kRows = 16;                // elements per lane per tile
constexpr int kTile = kPT * kRows;       // 4096 elements per tile (512 per warp)
constexpr int kDigits = 2048;

struct PruneState {
  // -- zeroed by the host-side memset before pass 0 --
  unsigned int hist0[kDigits];
  unsigned int ticket[4];
  // -- zeroed by CTA 0 of pass 0 --
  unsigned int hist1[kDigits];
  unsigned int hist2[kDigits];
  // -- written by the last CTA of each pass --
  unsigned int prefix;        // key bits fixed so far
  unsigned int mask;          // which bits of prefix are fixed
  unsigned long long k_rem;   // rank (1-based, from the top) still to find below prefix
  unsigned long long n_gt;    // keys strictly greater than the final threshold
  unsigned long long need_eq; // keys equal to the threshold to keep (index order)
};
constexpr size_t kMemsetBytes = offsetof(PruneState, hist1);

__device__ __forceinline__ uint32_t rank_key(float x, bool mag) {
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7FFFFFFFu) > 0x7F800000u) return 0u;   // NaN ranks lowest
  if (mag) return (b & 0x7FFFFFFFu) + 1u;
  if (b == 0x80000000u) b = 0u;                     // -0.0 ties with +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ int pass_shift(int p) { return p == 0 ? 21 : (p == 1 ? 10 : 0); }
__device__ __forceinline__ uint32_t pass_dmask(int p) { return p == 2 ? 0x3FFu : 0x7FFu; }

// warp-aggregated histogram increment: lanes with equal digits elect one
// leader that adds the group's population
__device__ __forceinline__ void hist_add(unsigned int* sh, bool take, uint32_t digit) {
  const unsigned act = __ballot_sync(0xFFFFFFFFu, take);
  if (!take) return;
  const unsigned peers = __match_any_sync(act, digit);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(sh + digit, __popc(peers));
}

// One radix pass: histogram of digit p among keys matching the prefix; the
// last CTA picks the digit holding rank k_rem and narrows the prefix.
__global__ void __launch_bounds__(kPT) k_radix_pass(const float* __restrict__ x, int64_t n,
                                                    bool mag, int p, unsigned long long k0,
                                                    PruneState* st) {
  __shared__ unsigned int sh[kDigits];
  for (int i = threadIdx.x; i < kDigits; i += blockDim.x) sh[i] = 0;
  if (p == 0 && blockIdx.x == 0) {
    for (int i = threadIdx.x; i < kDigits; i += blockDim.x) st->hist1[i] = st->hist2[i] = 0;
  }
  __syncthreads();
  const uint32_t prefix = p == 0 ? 0u : st->prefix, mask = p == 0 ? 0u : st->mask;
  const int shift = pass_shift(p);
  const uint32_t dm = pass_dmask(p);
  const int64_t S = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = aligned16(x) ? n / 4 : 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  // every lane runs the same trip count (warp-synchronous ballots inside)
  const int64_t trips = (n4 + S - 1) / S;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t t = 0; t < trips; ++t) {
    const int64_t i = i0 + t * S;
    const bool in = i < n4;
    const float4 v = in ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t u0 = rank_key(v.x, mag), u1 = rank_key(v.y, mag), u2 = rank_key(v.z, mag),
                   u3 = rank_key(v.w, mag);
    hist_add(sh, in && (u0 & mask) == prefix, (u0 >> shift) & dm);
    hist_add(sh, in && (u1 & mask) == prefix, (u1 >> shift) & dm);
    hist_add(sh, in && (u2 & mask) == prefix, (u2 >> shift) & dm);
    hist_add(sh, in && (u3 & mask) == prefix, (u3 >> shift) & dm);
  }
  for (int64_t i = n4 * 4 + i0; i < n; i += S) {
    const uint32_t u = rank_key(x[i], mag);
    if ((u & mask) == prefix) atomicAdd(sh + ((u >> shift) & dm), 1u);
  }
  __syncthreads();
  unsigned int* gh = p == 0 ? st->hist0 : (p == 1 ? st->hist1 : st->hist2);
  for (int i = threadIdx.x; i < kDigits; i += blockDim.x)
    if (sh[i]) atomicAdd(gh + i, sh[i]);

  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&st->ticket[p], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Last CTA: suffix-scan the digit histogram from the top digit down.
  // Each thread owns kDigits / kPT = 8 consecutive digits.
  constexpr int kPer = kDigits / kPT;
  __shared__ unsigned long long tsum[kPT];
  __shared__ unsigned long long sel_above;
  __shared__ int sel_t;
  const volatile unsigned int* vh = gh;
  unsigned int loc[kPer];
  unsigned long long s = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    loc[j] = vh[threadIdx.x * kPer + j];
    s += loc[j];
  }
  tsum[threadIdx.x] = s;
  __syncthreads();
  const unsigned long long need = p == 0 ? k0 : st->k_rem;
  if (threadIdx.x == 0) {
    unsigned long long above = 0;
    int t = kPT - 1;
    while (t > 0 && above + tsum[t] < need) above += tsum[t--];
    sel_above = above;
    sel_t = t;
  }
  __syncthreads();
  if (threadIdx.x == sel_t) {
    unsigned long long above = sel_above;
    int d = kPer - 1;
    while (d > 0 && above + loc[d] < need) above += loc[d--];
    const uint32_t digit = static_cast<uint32_t>(threadIdx.x * kPer + d);
    st->prefix = prefix | (digit << shift);
    st->mask = mask | (dm << shift);
    st->k_rem = need - above;          // rank within the chosen digit
    st->n_gt = (p == 0 ? 0ull : st->n_gt) + above;
    if (p == 2) st->need_eq = need - above;
  }
}

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
  for (int w = 0; w < kPT / 32; ++w) {
    if (w < warp) base += sh_warp[w];
    tot += sh_warp[w];
  }
  __syncthreads();
  total = tot;
  return base + inc - v;
}

// Per tile: (#u > T, #u == T); the last CTA turns them into exclusive
// prefix sums (output offset, equal keys before) for the write pass.
__global__ void __launch_bounds__(kPT) k_tile_count(const float* __restrict__ x, int64_t n,
                                                    bool mag, PruneState* st,
                                                    unsigned int* __restrict__ tile_gt,
                                                    unsigned int* __restrict__ tile_eq,
                                                    unsigned long long* __restrict__ out_off,
                                                    unsigned long long* __restrict__ eq_before) {
  const uint32_t T = st->prefix;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  const bool vec = aligned16(x) && base + kTile <= n;
  unsigned int gt = 0, eq = 0;
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(x + base);
#pragma unroll
    for (int j = 0; j < kTile / 4 / kPT; ++j) {
      const float4 v = __ldg(x4 + j * kPT + threadIdx.x);
      const uint32_t u[4] = {rank_key(v.x, mag), rank_key(v.y, mag), rank_key(v.z, mag),
                             rank_key(v.w, mag)};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        gt += u[q] > T;
        eq += u[q] == T;
      }
    }
  } else {
    for (int j = 0; j < kRows; ++j) {
      const int64_t i = base + j * kPT + threadIdx.x;
      if (i < n) {
        const uint32_t u = rank_key(x[i], mag);
        gt += u > T;
        eq += u == T;
      }
    }
  }
  gt = __reduce_add_sync(0xFFFFFFFFu, gt);
  eq = __reduce_add_sync(0xFFFFFFFFu, eq);
  __shared__ unsigned int sg[kPT / 32], se[kPT / 32];
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    se[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int a = 0, b = 0;
    for (int w = 0; w < kPT / 32; ++w) {
      a += sg[w];
      b += se[w];
    }
    tile_gt[blockIdx.x] = a;
    tile_eq[blockIdx.x] = b;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&st->ticket[3], 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // scan the tile counts: each thread owns a contiguous run of tiles
  const int64_t nt = gridDim.x;
  const int64_t per = (nt + kPT - 1) / kPT;
  const int64_t t0 = threadIdx.x * per, t1 = min(nt, t0 + per);
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
  const unsigned long long need_eq = st->need_eq;
  for (int64_t t = t0; t < t1; ++t) {
    eq_before[t] = eb;
    out_off[t] = gb + (eb < need_eq ? eb : need_eq);
    gb += vg[t];
    eb += ve[t];
  }
}

// Write pass.  Warp w of the tile owns elements [base + 512 w, +512); lane l
// holds elements base + 512 w + 32 j + l (j = 0..15): each load is one
// coalesced 128 B line and (j, l) order is index order, so warp ballots give
// every kept element its output slot directly.
__global__ void __launch_bounds__(kPT) k_tile_write(const float* __restrict__ x, int64_t n,
                                                    bool mag, const PruneState* __restrict__ st,
                                                    const unsigned long long* __restrict__ out_off,
                                                    const unsigned long long* __restrict__ eq_before,
                                                    float* __restrict__ values,
                                                    int32_t* __restrict__ indices) {
  const uint32_t T = st->prefix;
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
  // per-warp (gt, eq) totals -> warp offsets inside the tile
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
  unsigned long long eq_run = eq_before[blockIdx.x], gt_run = 0;
  for (int w = 0; w < warp; ++w) {
    gt_run += s_gt[w];
    eq_run += s_eq[w];
  }
  // position of the next kept element = tile offset + kept-before-in-tile
  const unsigned long long eq_tile0 = eq_before[blockIdx.x];
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

// K7: dense = 0 with survivors scattered in.  Each CTA owns a tile of the
// dense output; warp 0 finds the tile's slice of the ascending index list
// (32-way search), all threads write zeros with float4 stores, then scatter.
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

}  // namespace sf

using namespace sf;

extern "C" {

size_t sf_prune_workspace_bytes(int64_t n) {
  const int64_t nt = ntiles_of(n > 0 ? n : 1);
  return align256(sizeof(PruneState)) + 2 * align256(nt * sizeof(unsigned int)) +
         2 * align256(nt * sizeof(unsigned long long));
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

  if (cudaMemsetAsync(st, 0, kMemsetBytes, s) != cudaSuccess) return check_launch();
  const bool mag = by_magnitude != 0;
  const unsigned grid = grid_for((n + 3) / 4, kPT, 4);
  const unsigned long long kk = static_cast<unsigned long long>(k);
  for (int p = 0; p < 3; ++p) k_radix_pass<<<grid, kPT, 0, s>>>(x, n, mag, p, kk, st);
  k_tile_count<<<static_cast<unsigned>(nt), kPT, 0, s>>>(x, n, mag, st, tile_gt, tile_eq, out_off,
                                                         eq_before);
  k_tile_write<<<static_cast<unsigned>(nt), kPT, 0, s>>>(x, n, mag, st, out_off, eq_before, values,
                                                         indices);
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
