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
// One persistent kernel (one 1024-thread CTA per SM, grid barriers between
// phases) after a memset of the small state; x is read once.  Every warp
// owns a contiguous range of x (n / #warps elements, in 16-element quanta)
// and keeps what it learns about that range in registers across phases:
//  bracket  every CTA takes the same 4096-key pseudo-random sample and
//           brackets rank k between two of its order statistics (+-4.5
//           sigma, a min/max-scaled 4096-bin histogram in shared memory),
//           while its warps' first loads of x are in flight.
//  stream   each warp streams its range: keys >= the bracket's low end
//           (~k plus the bracket, ~12% of n) are compacted in index order
//           into the warp's slots of a staging list (L2-resident), keys
//           inside the bracket are counted into 2048 fine bins.
//  gather   [barrier] every CTA locates the fine bin F holding rank k;
//           each warp counts its staged keys above F and gathers its keys
//           inside F (a few hundred in all).
//  rank     [barrier] every CTA ranks F's keys for the exact threshold T
//           (and how many keys == T to keep); each warp's kept count
//           follows from its count above F and F's keys in its range.
//  emit     [barrier: per-CTA totals] each warp filters its staged keys
//           (> T, or == T within the tie quota) into (values, indices) at
//           its global offset, plus the CSR row pointers.
// Exact for any input: a warp whose range stages more keys than its slots
// (keep_frac above ~0.14, skewed or tie-heavy data) reads its range of x
// again instead; if the bracket misses rank k or F holds more keys than
// the gather buffer (heavy ties), T comes from a grid-wide radix select
// over x (four more passes; never taken on activation data).
#include "common.cuh"
#include "prune_state.cuh"

#include <algorithm>

namespace sf {

constexpr int kFT = 1024;                // threads per CTA
constexpr int kFW = kFT / 32;            // warps per CTA
constexpr int kChunkW = 512;             // elements per warp per step of the x paths (16 per lane)
constexpr int kCW = 256;                 // elements per warp per streaming step (8 per lane)
constexpr int kStages = 4;               // streaming ring depth per warp (3 steps in flight)
constexpr int kQ = 16;                   // range quantum (elements)
constexpr int kSlack = 64;               // staging slots per warp beyond 5/32 of its range
constexpr int kSample = 4 * kFT;         // sample keys (4 per thread)
constexpr int kBins = 4096;              // bracket histogram bins
constexpr int kCandCap = 65536;          // gathered keys of the threshold bin F (key, index)
constexpr int kCandSmem = 4096;          // F keys ranked in shared memory
constexpr int kBList = 2048;             // hinted path: bracket keys per CTA (in the bracket-histogram area)
constexpr int kBListCap = 65536;         // hinted path: bracket keys over all CTAs (global list)
constexpr uint32_t kHintHalf = 1u << 14; // hinted bracket: T -+ 2^14 key units (|x| -+ 0.1-0.2%) at first
constexpr int kLocal = 2048;             // F keys >= T in one CTA's range, listed in shared memory
constexpr int kPT = 256;                 // restore threads per CTA
constexpr int kRTile = 4096;             // restore tile (floats, staged in shared memory)
constexpr size_t kRingBytes = size_t(kFW) * kStages * kCW * sizeof(float);    // 128 KB
constexpr size_t kFusedSmem = kRingBytes + kBins * sizeof(unsigned int) + (kFine + 1) * sizeof(unsigned int);
static_assert((2 * kCandSmem + 2 * kLocal) * 4 <= kRingBytes, "F's keys and lists fit the ring after streaming");
static_assert(kBList * 8 <= kBins * 4, "the per-CTA bracket list fits the bracket-histogram area");

// Block-wide exclusive scan: warp scans by shuffles, then every warp scans
// the (<= 32) warp totals across its lanes -- no serial loop over warps.
template <typename V>
__device__ __forceinline__ V block_scan_impl(V v, V* sh_warp, V& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = static_cast<int>(blockDim.x >> 5);
  V inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sh_warp[warp] = inc;
  __syncthreads();
  V t = lane < nw ? sh_warp[lane] : V(0);
  V tinc = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V y = __shfl_up_sync(0xFFFFFFFFu, tinc, o);
    if (lane >= o) tinc += y;
  }
  const V base = __shfl_sync(0xFFFFFFFFu, tinc - t, warp);   // exclusive prefix of my warp
  total = __shfl_sync(0xFFFFFFFFu, tinc, 31);
  __syncthreads();
  return base + inc - v;
}

__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long v,
                                                                   unsigned long long* sh_warp,
                                                                   unsigned long long& total) {
  return block_scan_impl<unsigned long long>(v, sh_warp, total);
}

__device__ __forceinline__ unsigned int block_exclusive_scan32(unsigned int v, unsigned int* sh_warp,
                                                              unsigned int& total) {
  return block_scan_impl<unsigned int>(v, sh_warp, total);
}

// Among `nb` bins (larger bin = larger keys) find the bin holding rank
// `need` (1-based from the top).  Whole CTA calls; each thread owns a
// contiguous run of bins, a block scan locates the owning thread and only
// that thread walks its run.  Returns the bin and the count strictly above
// it.  Loops stay rolled: single-CTA callers are bound by instruction
// fetch along their path, not by issue.
__device__ __noinline__ void select_digit(const unsigned int* hist, int nb, unsigned long long need,
                             unsigned int& digit, unsigned long long& above) {
  __shared__ unsigned long long sw[32];
  __shared__ unsigned int s_digit;
  __shared__ unsigned long long s_above;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  const int cnt = max(0, min(per, nb - b0));
  unsigned long long s = 0;
#pragma unroll 1
  for (int j = 0; j < cnt; ++j) s += hist[b0 + j];
  unsigned long long total;
  const unsigned long long before = block_exclusive_scan(s, sw, total);
  const unsigned long long ab = total - before - s;       // counts in higher threads' bins
  if (s > 0 && ab < need && need <= ab + s) {
    unsigned long long a = ab;
    int d = cnt - 1;
#pragma unroll 1
    for (; d > 0; --d) {
      const unsigned int c = hist[b0 + d];
      if (a + c >= need) break;
      a += c;
    }
    s_digit = static_cast<unsigned int>(b0 + d);
    s_above = a;
  }
  __syncthreads();
  digit = s_digit;
  above = s_above;
  __syncthreads();
}

// Exact key of rank `need` (from the top) among keys in [lo, hi], by 8-bit
// MSD radix with one CTA scanning `count` keys from `get`.  Returns T and
// the number of keys equal to T to keep.
template <typename Getter>
__device__ void cta_select(Getter get, int64_t count, uint32_t lo, uint32_t hi,
                           unsigned long long need, uint32_t& T, unsigned long long& need_eq) {
  __shared__ unsigned int h[256];
  uint32_t prefix = 0, mask = 0;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
      const uint32_t u = get(i);
      if (u >= lo && u <= hi && (u & mask) == prefix) atomicAdd(h + ((u >> shift) & 0xFFu), 1u);
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

// ------------------------------------------------------------------ warp / grid helpers

__device__ __forceinline__ unsigned int lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned int lanemask_lt() {
  unsigned int m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned int warp_incl_scan(unsigned int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane_id() >= static_cast<unsigned>(o)) v += y;
  }
  return v;
}

// All CTAs of the grid (co-resident: one per SM) arrive before any leaves.
// `target` = gridDim.x times the number of barriers passed so far.
__device__ __forceinline__ void grid_sync(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// 16 consecutive floats at x[base, base + 16) (zero at or past `end`)
__device__ __forceinline__ void load16(const float* __restrict__ x, int64_t end, int64_t base, float (&v)[16]) {
  if (base + 16 <= end && aligned16(x)) {
    const float4* p = reinterpret_cast<const float4*>(x + base);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float4 q = __ldg(p + w);
      v[4 * w] = q.x;
      v[4 * w + 1] = q.y;
      v[4 * w + 2] = q.z;
      v[4 * w + 3] = q.w;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = base + j < end ? __ldg(x + base + j) : 0.f;
}

// Asynchronous global -> shared copies (zero-filled past `bytes`).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// Bulk prefetch of [p, p + bytes) into L2 (TMA; bytes a multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ------------------------------------------------------------------ bracket

// Bins holding ranks R0 and R1 (1-based from the top; 0 = not wanted) of a
// kBins histogram: one block scan over per-thread runs of four bins.
__device__ void dual_select(const unsigned int* hist, unsigned int R0, unsigned int R1, unsigned int& d0,
                            unsigned int& d1) {
  static_assert(kBins == 4 * kFT, "four bins per thread");
  __shared__ unsigned int sw[kFW];
  __shared__ unsigned int s_d[2];
  const uint4 c = reinterpret_cast<const uint4*>(hist)[threadIdx.x];
  const unsigned int cc[4] = {c.x, c.y, c.z, c.w};
  const unsigned int sum = c.x + c.y + c.z + c.w;
  unsigned int total;
  const unsigned int before = block_exclusive_scan32(sum, sw, total);
  const unsigned int ab = total - before - sum;          // keys in higher threads' bins
  const unsigned int R[2] = {R0, R1};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (R[q] && ab < R[q] && R[q] <= ab + sum) {
      unsigned int acc = ab;
      int d = 3;
      for (; d > 0; --d) {
        if (acc + cc[d] >= R[q]) break;
        acc += cc[d];
      }
      s_d[q] = 4 * threadIdx.x + d;
    }
  }
  __syncthreads();
  d0 = s_d[0];
  d1 = s_d[1];
}

__device__ __forceinline__ void phase_time(PruneState* st, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    st->t[i] = t;
  }
}


// Keys of rank about k from the top lie in [lo, hi] with overwhelming
// probability: order statistics k/n * m -+ (4.5 sigma + 16) of an m-key
// sample, rounded outwards to the bins of a histogram scaled to the
// sample's [min, max].  Whole CTA calls; every CTA gets the same bracket.
__device__ __forceinline__ void load_sample(const float* __restrict__ x, int64_t n, float (&sv)[kSample / kFT]) {
  const int m = static_cast<int>(n < kSample ? n : kSample);
  const uint32_t span = static_cast<uint32_t>(n / m);
#pragma unroll
  for (int r = 0; r < kSample / kFT; ++r) {
    const int j = threadIdx.x + r * kFT;
    uint32_t h = static_cast<uint32_t>(j) * 2654435761u;
    h ^= h >> 16;
    sv[r] = j < m ? __ldg(x + static_cast<int64_t>(j) * span + __umulhi(h, span)) : 0.f;
  }
}

template <bool MAG>
__device__ void find_bracket(const float (&sv)[kSample / kFT], int64_t n, unsigned long long k, unsigned int* bins,
                             uint32_t& lo, uint32_t& hi, PruneState* st_dbg) {
  __shared__ uint32_t s_min[kFW], s_max[kFW];
  const int m = static_cast<int>(n < kSample ? n : kSample);
  uint32_t u[kSample / kFT];
  for (int i = threadIdx.x; i < kBins; i += kFT) bins[i] = 0;
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
#pragma unroll
  for (int r = 0; r < kSample / kFT; ++r) {
    u[r] = rank_key<MAG>(sv[r]);
    if (static_cast<int>(threadIdx.x) + r * kFT < m) {
      mn = min(mn, u[r]);
      mx = max(mx, u[r]);
    }
  }
  mn = __reduce_min_sync(0xFFFFFFFFu, mn);
  mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  if (lane_id() == 0) {
    s_min[threadIdx.x >> 5] = mn;
    s_max[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  mn = __reduce_min_sync(0xFFFFFFFFu, s_min[lane_id()]);
  mx = __reduce_max_sync(0xFFFFFFFFu, s_max[lane_id()]);
  phase_time(st_dbg, 2);
  const int rbits = 32 - __clz(mx - mn);                // (mx - mn) >> s1 < kBins = 2^12
  const uint32_t s1 = rbits > 12 ? rbits - 12 : 0;
#pragma unroll
  for (int r = 0; r < kSample / kFT; ++r)
    if (static_cast<int>(threadIdx.x) + r * kFT < m) atomicAdd(bins + ((u[r] - mn) >> s1), 1u);
  __syncthreads();
  const double p = static_cast<double>(k) / static_cast<double>(n);
  const double rr = p * m;
  const double dlt = 4.5 * sqrt(m * p * (1.0 - p)) + 16.0;
  const int64_t r_hi = static_cast<int64_t>(floor(rr - dlt));   // 0-based top-rank of the upper key
  const int64_t r_lo = static_cast<int64_t>(ceil(rr + dlt));    // 0-based top-rank of the lower key
  unsigned int d0, d1;
  phase_time(st_dbg, 1);
  dual_select(bins, r_hi > 0 ? static_cast<unsigned int>(r_hi) + 1 : 0u, r_lo < m ? static_cast<unsigned int>(r_lo) + 1 : 0u,
              d0, d1);
  const unsigned long long top = static_cast<unsigned long long>(mn) + ((d0 + 1ull) << s1) - 1ull;
  hi = r_hi > 0 ? static_cast<uint32_t>(top > 0xFFFFFFFFull ? 0xFFFFFFFFull : top) : 0xFFFFFFFFu;
  lo = r_lo < m ? mn + (d1 << s1) : 0u;
}

// ------------------------------------------------------------------ rank inside F

// Exact key of rank `need` (1-based from the top) among keys[0, nc), all in
// [flo, flo + 2^shf): MSD radix over the offsets key - flo in rounds of up
// to 11 bits (one round when F spans at most 2048 key values), histograms
// in `bins` (2048 words).  Returns T and how many keys == T to keep.
__device__ void select_in_f(const uint32_t* keys, unsigned int nc, uint32_t flo, uint32_t shf,
                            unsigned long long need, unsigned int* bins, uint32_t& T,
                            unsigned long long& need_eq) {
  uint32_t prefix = 0;
#pragma unroll 1
  for (int top = static_cast<int>(shf); top > 0; top -= 11) {
    const int sh = top > 11 ? top - 11 : 0;
    const int nb = 1 << (top - sh);
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    for (unsigned int j = threadIdx.x; j < nc; j += blockDim.x) {
      const uint32_t o = keys[j] - flo;
      if ((static_cast<uint64_t>(o) >> top) == (static_cast<uint64_t>(prefix) >> top))
        atomicAdd(bins + ((o >> sh) & static_cast<uint32_t>(nb - 1)), 1u);
    }
    __syncthreads();
    unsigned int d;
    unsigned long long ab;
    select_digit(bins, nb, need, d, ab);
    prefix |= d << sh;
    need -= ab;
  }
  T = flo + prefix;
  need_eq = need;
}

// ------------------------------------------------------------------ emit

// One warp's output from its staged keys: key > T, or == T while the tie
// quota lasts, in index order, at `off` onward.  Row pointers: the next row
// start p is tracked warp-uniformly; the first staged key at or past p
// (a ballot) tells how many kept keys lie before it.
// The staged pairs pass through the warp's idle ring slice (`wsm`, 512
// pairs): eight rounds' loads in flight, then a rolled loop over the rounds
// -- a small loop body, so the emit stays inside the instruction cache.
template <bool MAG>
__device__ void emit_staged(const uint2* __restrict__ sp, unsigned int cnt,
                            int64_t a, int64_t end, uint32_t T, bool ties, unsigned long long need_eq,
                            unsigned long long off, unsigned long long eqb, float* __restrict__ values,
                            int32_t* __restrict__ indices, uint32_t row_len, int32_t* __restrict__ row_ptr,
                            uint2* wsm) {
  const unsigned int lane = lane_id(), lt = lanemask_lt();
  // rows starting in [a, end): r_next .. r_last
  uint32_t r_next = a == 0 ? 0u : static_cast<uint32_t>(a - 1) / row_len + 1u;
  const uint32_t r_last = static_cast<uint32_t>(end - 1) / row_len;
  uint32_t p_next = r_next * row_len;
#pragma unroll 1
  for (unsigned int r00 = 0; r00 < cnt; r00 += 256) {
    {
      uint2 pr[8];                                            // eight rounds' loads in flight
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const unsigned int j = r00 + 32 * q + lane;
        pr[q] = j < cnt ? __ldcg(sp + j) : make_uint2(0u, 0u);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) wsm[32 * q + lane] = pr[q];
      __syncwarp();
    }
#pragma unroll 1
    for (int q = 0; q < 8; ++q) {
      const unsigned int r0 = r00 + 32 * q;
      if (r0 >= cnt) break;                                   // warp-uniform
      const bool in = r0 + lane < cnt;
      const uint2 prq = wsm[32 * q + lane];
      const float v = __uint_as_float(prq.x);
      const uint32_t ix = prq.y;
      const uint32_t u = rank_key<MAG>(v);
      bool keep = in && u > T;
      if (ties) {                                             // warp-uniform
        const unsigned int eqm = __ballot_sync(0xFFFFFFFFu, in && u == T);
        if (in && u == T && eqb + __popc(eqm & lt) < need_eq) keep = true;
        eqb += __popc(eqm);
      }
      const unsigned int km = __ballot_sync(0xFFFFFFFFu, keep);
      const unsigned long long pos = off + __popc(km & lt);
      if (keep) {
        values[pos] = v;
        indices[pos] = static_cast<int32_t>(ix);
      }
      if (row_ptr) {                                          // warp-uniform
        const unsigned int nin = min(32u, cnt - r0);
        const uint32_t last_ix = __shfl_sync(0xFFFFFFFFu, ix, nin - 1);
        while (r_next <= r_last && p_next <= last_ix) {
          const unsigned int f = __ballot_sync(0xFFFFFFFFu, in && ix >= p_next);
          const unsigned int fl = __ffs(f) - 1;
          if (lane == 0) row_ptr[r_next] = static_cast<int32_t>(off + __popc(km & ((1u << fl) - 1u)));
          ++r_next;
          p_next += row_len;
        }
      }
      off += __popc(km);
    }
    __syncwarp();                                             // the slice is refilled next chunk
  }
  if (row_ptr)                                                // rows after the last staged key
    for (uint32_t r = r_next + lane; r <= r_last && r_next <= r_last; r += 32) row_ptr[r] = static_cast<int32_t>(off);
}

// The same from x itself (rounds of 128 elements, four consecutive per lane).
template <bool MAG>
__device__ void emit_from_x(const float* __restrict__ x, int64_t a, int64_t end, uint32_t T, bool ties,
                            unsigned long long need_eq, unsigned long long off, unsigned long long eqb,
                            float* __restrict__ values, int32_t* __restrict__ indices, uint32_t row_len,
                            int32_t* __restrict__ row_ptr) {
  const unsigned int lane = lane_id();
#pragma unroll 1
  for (int64_t r0 = a; r0 < end; r0 += 128) {
    const int64_t e0 = r0 + 4 * lane;
    float v[4];
    if (e0 + 4 <= end && aligned16(x)) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(x + e0));
      v[0] = q.x;
      v[1] = q.y;
      v[2] = q.z;
      v[3] = q.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = e0 + q < end ? __ldg(x + e0 + q) : 0.f;
    }
    unsigned int km = 0, em = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t u = rank_key<MAG>(v[q]);
      const bool in = e0 + q < end;
      km |= (in && u > T) ? (1u << q) : 0u;
      em |= (in && u == T) ? (1u << q) : 0u;
    }
    if (ties) {
      const unsigned int ei = warp_incl_scan(__popc(em));
      unsigned long long r = eqb + ei - __popc(em);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (em & (1u << q)) {
          if (r < need_eq) km |= 1u << q;
          ++r;
        }
      }
      eqb += __shfl_sync(0xFFFFFFFFu, ei, 31);
    }
    const unsigned int ki = warp_incl_scan(__popc(km));
    unsigned long long pos = off + ki - __popc(km);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t e = e0 + q;
      if (row_ptr && e < end && static_cast<uint32_t>(e) % row_len == 0)
        row_ptr[static_cast<uint32_t>(e) / row_len] = static_cast<int32_t>(pos);
      if (km & (1u << q)) {
        values[pos] = v[q];
        indices[pos] = static_cast<int32_t>(e);
        ++pos;
      }
    }
    off += __shfl_sync(0xFFFFFFFFu, ki, 31);
  }
}

// ------------------------------------------------------------------ stream step

// One streaming step of a warp (kCW elements from its ring slot; lane l
// takes elements l + 32 t, so a ballot per t orders the kept keys): keys >=
// lo staged as (value, index) pairs at `run` onward, keys inside [lo, hi]
// counted into the fine bins (out-of-bracket keys into the dummy bin
// kFine, so the shared reduction needs no branch).  FAST: magnitude keys
// with 1 <= lo and hi <= key(inf): u - lo == |bits| - (lo - 1) for numbers,
// and a NaN's difference exceeds both limits.
template <bool MAG, bool FAST, bool FULL, bool LIST>
__device__ __forceinline__ void stream_step(const float* slot, uint32_t base, uint32_t end32, uint32_t lo,
                                            uint32_t lom1, uint32_t klim, uint32_t wid, uint32_t shf,
                                            uint32_t fine_addr, unsigned int lt, unsigned int cap, uint2* sp,
                                            unsigned int& run, bool& ovf, uint2* blist_s, unsigned int* s_bl,
                                            unsigned int& inbc, float lo_f = 0.f, float hi_f = 0.f) {
  // FAST && LIST (hinted): keep / in-bracket by two float compares on |x|
  // (|x| >= lo_f <=> key >= lo for every number; NaN fails both), the key
  // itself only for the rare bracket keys -- fewer integer-pipe instructions
  const unsigned int lane = lane_id();
  float val[kCW / 32];
  unsigned int kb[kCW / 32], pre[kCW / 32];
  unsigned int step = 0;
#pragma unroll
  for (int t = 0; t < kCW / 32; ++t) {
    val[t] = slot[lane + 32 * t];
    uint32_t d = 0;
    bool keep, inb;
    if (FAST && LIST) {
      const float av = fabsf(val[t]);
      keep = av >= lo_f;
      inb = keep && av <= hi_f;
    } else if (FAST) {
      d = (__float_as_uint(val[t]) & 0x7FFFFFFFu) - lom1;
      keep = d <= klim;
      inb = d <= wid;
    } else {
      const uint32_t u = rank_key<MAG>(val[t]);
      d = u - lo;
      keep = u >= lo;
      inb = d <= wid;
    }
    if (!FULL) {
      const bool ok = base + 32 * t < end32;
      keep = keep && ok;
      inb = inb && ok;
    }
    if (!LIST) {                                         // (the hinted path histograms its list instead)
      const uint32_t bin = inb ? (d >> shf) : static_cast<uint32_t>(kFine);
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(fine_addr + (bin << 2)) : "memory");
    }
    if (LIST) {                                          // hinted path: list the bracket's keys
      const unsigned int bm = __ballot_sync(0xFFFFFFFFu, inb);
      if (bm) {                                          // warp-uniform, rare (a narrow bracket)
        unsigned int p0 = 0;
        if (lane == 0) p0 = atomicAdd(s_bl, static_cast<unsigned int>(__popc(bm)));
        p0 = __shfl_sync(0xFFFFFFFFu, p0, 0);
        const unsigned int p = p0 + __popc(bm & lt);
        if (inb && p < static_cast<unsigned int>(kBList))
          blist_s[p] = make_uint2((__float_as_uint(val[t]) & 0x7FFFFFFFu) + 1u, base + 32 * t);
        inbc += __popc(bm);
      }
    }
    kb[t] = __ballot_sync(0xFFFFFFFFu, keep);
    pre[t] = step;
    step += __popc(kb[t]);
  }
  if (!ovf && run + step <= cap) {                       // warp-uniform
#pragma unroll
    for (int t = 0; t < kCW / 32; ++t) {
      const unsigned int pos = run + pre[t] + __popc(kb[t] & lt);
      const uint32_t mine = (kb[t] >> lane) & 1u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.v2.u32 [%1], {%2, %3};\n\t}"
                   :: "r"(mine), "l"(sp + pos), "r"(__float_as_uint(val[t])), "r"(base + 32 * t) : "memory");
    }
  } else {
    ovf = true;
  }
  run += step;
}

// ------------------------------------------------------------------ the kernel

// HINT: the caller passes a per-site hint {valid, T, half width} that this
// kernel rewrites with the call's threshold.  With a valid hint the bracket
// is T_prev -+ half (no sample), the stream also lists the bracket's keys
// (a few thousand) per CTA into a global list, and after the ONE grid
// barrier every CTA reads that list itself: F's keys, the exact T, the
// counts above T / equal to T before each of its warps and the CTAs before
// it (from the per-CTA above-bracket totals) -- no gather / rank barriers.
// A hint whose bracket misses rank k (or whose lists overflow) falls into
// the general path below, exactly as without a hint, and the next call's
// half width doubles.
template <bool MAG, bool HINT>
__global__ void __launch_bounds__(kFT, 1) k_prune(const float* __restrict__ x, int64_t n, unsigned long long k,
                                                  PruneState* st, unsigned long long* __restrict__ cta_tot,
                                                  uint2* __restrict__ cands, uint2* __restrict__ staged,
                                                  float* __restrict__ values,
                                                  int32_t* __restrict__ indices, int row_len_i,
                                                  int32_t* __restrict__ row_ptr, uint32_t* __restrict__ hint,
                                                  uint2* __restrict__ blist,
                                                  unsigned long long* __restrict__ cta_abv) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float* ring = reinterpret_cast<float*>(dsm);                              // per-warp streaming rings
  unsigned int* bins = reinterpret_cast<unsigned int*>(dsm + kRingBytes);   // bracket histogram
  unsigned int* fine_s = bins + kBins;                                      // fine bins
  __shared__ unsigned int s_above;
  __shared__ unsigned int w_gt[kFW], w_eq[kFW];
  __shared__ unsigned long long s_before[2];
  const unsigned int lane = lane_id(), warp = threadIdx.x >> 5, lt = lanemask_lt();
  const unsigned int G = gridDim.x;
  const uint32_t row_len = static_cast<uint32_t>(row_len_i);
  // ---- this warp's range [a, end) and staging slots [sbase, sbase + cap)
  const int64_t W = static_cast<int64_t>(G) * kFW, gw = static_cast<int64_t>(blockIdx.x) * kFW + warp;
  const int64_t nq = (n + kQ - 1) / kQ;
  const int64_t q0 = gw * nq / W, q1 = (gw + 1) * nq / W;
  const int64_t a = q0 * kQ, end = min(n, q1 * kQ);
  const int64_t sbase = q0 * 5 / 2 + kSlack * gw;
  const unsigned int cap = static_cast<unsigned int>(q1 * 5 / 2 + kSlack * (gw + 1) - sbase);
  uint2* sp = staged + sbase;                            // (value bits, index) pairs
  float v[16];
  phase_time(st, 0);
  // ---- the streaming ring: step c of this warp lands in slot c % kStages
  float* wring = ring + static_cast<size_t>(warp) * kStages * kCW;
  const uint32_t wring_s = static_cast<uint32_t>(__cvta_generic_to_shared(wring));
  const bool al16 = aligned16(x);
  const int64_t nsteps = end > a ? (end - a + kCW - 1) / kCW : 0;
  auto issue = [&](int64_t c) {
    if (c < nsteps) {
      const int64_t base = a + c * kCW;
      const uint32_t ds = wring_s + static_cast<uint32_t>((c % kStages) * kCW * 4);
      if (al16 && base + kCW <= end) {
#pragma unroll
        for (int q = 0; q < kCW / 128; ++q) {
          const int p = lane + 32 * q;
          cp_async16(ds + 16u * p, x + base + 4 * p, 16u);
        }
      } else if (al16) {
#pragma unroll
        for (int q = 0; q < kCW / 128; ++q) {
          const int p = lane + 32 * q;
          const int64_t e = base + 4 * p;
          const uint32_t bytes = e >= end ? 0u : static_cast<uint32_t>((end - e) >= 4 ? 16 : (end - e) * 4);
          cp_async16(ds + 16u * p, bytes ? static_cast<const void*>(x + e) : static_cast<const void*>(x), bytes);
        }
      } else {
#pragma unroll
        for (int q = 0; q < kCW / 32; ++q) {
          const int64_t e = base + lane + 32 * q;
          const uint32_t bytes = e < end ? 4u : 0u;
          cp_async4(ds + 4u * (lane + 32 * q), bytes ? static_cast<const void*>(x + e) : static_cast<const void*>(x),
                    bytes);
        }
      }
    }
    cp_async_commit();
  };
  // hinted bracket: T_prev -+ half (keys of finite magnitudes, lo >= 1)
  bool hv = false;
  uint32_t lo = 0, hi = 0, hhalf = kHintHalf;
  if (HINT) {
    const uint4 hw = __ldcg(reinterpret_cast<const uint4*>(hint));
    hhalf = hw.z ? hw.z : kHintHalf;
    if (MAG && hw.x == 1u && hw.y >= 2u && hw.y <= 0x7F800000u) {
      hv = true;
      lo = hw.y > hhalf ? hw.y - hhalf : 1u;
      hi = hw.y + hhalf < 0x7F800001u ? hw.y + hhalf : 0x7F800001u;
    }
  }
  __shared__ unsigned int s_bl;
  uint2* blist_s = reinterpret_cast<uint2*>(bins);      // hinted: this CTA's bracket keys
  unsigned int inbc = 0;                                 // hinted: this warp's bracket keys
  if (hv) {                                              // block-uniform
#pragma unroll
    for (int c = 0; c < kStages - 1; ++c) issue(c);
    if (threadIdx.x == 0) {
      s_above = 0;
      s_bl = 0;
    }
  } else {
    float smp[kSample / kFT];
    load_sample(x, n, smp);                              // first in the memory queues
#pragma unroll
    for (int c = 0; c < kStages - 1; ++c) issue(c);     // in flight while the bracket is found
    if (threadIdx.x == 0) s_above = 0;
    // ---- bracket
    find_bracket<MAG>(smp, n, k, bins, lo, hi, st);
  }
  // fine bins of width 2^shf: ((hi - lo) >> shf) < kFine = 2^11
  const uint32_t wid = hi - lo;
  const int wbits = 32 - __clz(wid);
  const uint32_t shf = wbits > 11 ? wbits - 11 : 0;
  const bool fast = MAG && lo >= 1u && hi <= 0x7F800001u;
  for (int i = threadIdx.x; i <= kFine; i += kFT) fine_s[i] = 0;   // + the dummy bin
  __syncthreads();
  // ---- stream: stage keys >= lo in index order, histogram the bracket.
  // Lane l takes elements l + 32 t of a step, so a ballot per t orders the
  // kept keys and their stores are coalesced.
  const uint32_t fine_addr = static_cast<uint32_t>(__cvta_generic_to_shared(fine_s));
  const uint32_t lom1 = lo - 1u, klim = 0x7F800000u - lom1;
  const float lo_f = __uint_as_float(lom1), hi_f = __uint_as_float(hi - 1u);   // keys lo / hi as |x|
  const uint32_t end32 = static_cast<uint32_t>(end);
  unsigned int run = 0;
  bool ovf = false;
#pragma unroll 1
  for (int64_t c = 0; c < nsteps; ++c) {
    issue(c + kStages - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
    __syncwarp();
    const float* slot = wring + (c % kStages) * kCW;
    const uint32_t base = static_cast<uint32_t>(a + c * kCW) + lane;
    if (HINT && hv) {                                    // block-uniform; hv implies MAG and fast
      if (a + (c + 1) * kCW <= end)
        stream_step<MAG, true, true, true>(slot, base, end32, lo, lom1, klim, wid, shf, fine_addr, lt, cap, sp, run,
                                           ovf, blist_s, &s_bl, inbc, lo_f, hi_f);
      else
        stream_step<MAG, true, false, true>(slot, base, end32, lo, lom1, klim, wid, shf, fine_addr, lt, cap, sp,
                                            run, ovf, blist_s, &s_bl, inbc, lo_f, hi_f);
    } else if (MAG && fast) {                            // block-uniform
      if (a + (c + 1) * kCW <= end)
        stream_step<MAG, true, true, false>(slot, base, end32, lo, lom1, klim, wid, shf, fine_addr, lt, cap, sp, run,
                                            ovf, nullptr, nullptr, inbc);
      else
        stream_step<MAG, true, false, false>(slot, base, end32, lo, lom1, klim, wid, shf, fine_addr, lt, cap, sp,
                                             run, ovf, nullptr, nullptr, inbc);
    } else {
      stream_step<MAG, false, false, false>(slot, base, end32, lo, lom1, klim, wid, shf, fine_addr, lt, cap, sp, run,
                                            ovf, nullptr, nullptr, inbc);
    }
    __syncwarp();                                        // the slot is refilled next step
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (lane == 0 && run) atomicAdd(&s_above, run);      // keys >= lo in this CTA
  __shared__ unsigned int s_abv, s_blbase;
  if (HINT && hv) {
    if (threadIdx.x == 0) s_abv = 0;
    __syncthreads();
    if (lane == 0 && run - inbc) atomicAdd(&s_abv, run - inbc);   // keys above the bracket
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_above) atomicAdd(&st->staged, static_cast<unsigned long long>(s_above));
  if (HINT && hv) {                                      // this CTA's bracket keys -> the global list
    const unsigned int nb = s_bl;
    if (threadIdx.x == 0) {
      cta_abv[blockIdx.x] = s_abv;
      unsigned int b = 0xFFFFFFFFu;
      if (nb > static_cast<unsigned int>(kBList)) {
        atomicExch(&st->blist_ovf, 1u);
      } else if (nb) {
        b = atomicAdd(&st->blist_n, nb);
        if (b + nb > static_cast<unsigned int>(kBListCap)) atomicExch(&st->blist_ovf, 1u);
      }
      s_blbase = b;
    }
    __syncthreads();
    const unsigned int b = s_blbase;
    if (b != 0xFFFFFFFFu && b + nb <= static_cast<unsigned int>(kBListCap))
      for (unsigned int j = threadIdx.x; j < nb; j += kFT) {
        const uint2 e = blist_s[j];
        blist[b + j] = e;
        atomicAdd(st->fine + ((e.x - lo) >> shf), 1u);  // the bracket's histogram, merged before the barrier
      }
  }
  if (!(HINT && hv))
    for (int i = threadIdx.x; i < kFine; i += kFT)
      if (fine_s[i]) atomicAdd(st->fine + i, fine_s[i]);
  phase_time(st, 3);
  unsigned int nbar = 1;
  grid_sync(&st->bar, G * nbar++);
  phase_time(st, 4);
  __shared__ unsigned int sw32[kFW];
  uint32_t T;
  unsigned long long need_eq;
  unsigned int gt_w = 0, eq_w = 0;
  bool ok = false, fastb = false;
  unsigned int fb = 0;
  unsigned long long above_tot = 0, above_f = 0;
  if (HINT && hv) {
    // ---- hinted single-barrier path: every CTA reads the whole bracket
    // list (a few thousand keys) itself -- its histogram, F, the exact T
    // and the counts before its warps -- no gather / rank barriers
    __shared__ unsigned long long sw64h[kFW];
    {
      const unsigned long long g = threadIdx.x < G ? __ldcg(cta_abv + threadIdx.x) : 0ull;
      block_exclusive_scan(g, sw64h, above_tot);         // keys above the bracket, all CTAs
    }
    const unsigned int nl = __ldcg(&st->blist_n);
    ok = __ldcg(&st->blist_ovf) == 0u && above_tot < k && k <= above_tot + nl;
    constexpr unsigned int kLS = static_cast<unsigned int>(kRingBytes / sizeof(uint2));   // list cached in the ring
    const bool cached = nl <= kLS;
    if (ok && cached) {                                  // the whole list in flight while F is found
      const uint32_t ls = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
      for (unsigned int j = 2 * threadIdx.x; j < nl; j += 2 * kFT)
        cp_async16(ls + 8u * j, blist + j, j + 1 < nl ? 16u : 8u);
      cp_async_commit();
    }
    if (ok) {
      for (int i = threadIdx.x; i < kFine; i += kFT) fine_s[i] = __ldcg(st->fine + i);
      __syncthreads();
      phase_time(st, 5);
      select_digit(fine_s, kFine, k - above_tot, fb, above_f);
      fastb = fine_s[fb] <= static_cast<unsigned int>(kBList);
      phase_time(st, 6);
    }
    if (ok && cached) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    if (fastb) {
      const uint32_t flo = lo + (fb << shf);
      const uint64_t fhi64 = static_cast<uint64_t>(flo) + (1ull << shf) - 1ull;
      const uint32_t fhi = fhi64 > hi ? hi : static_cast<uint32_t>(fhi64);
      const uint32_t fw = fhi - flo;
      const unsigned long long need_f = k - above_tot - above_f;
      const uint2* lst = reinterpret_cast<const uint2*>(ring);
      uint32_t* keys = reinterpret_cast<uint32_t*>(bins);   // F's keys (<= kBList)
      uint32_t* kidx = keys + kBList;
      __shared__ unsigned int s_lgt[kFW], s_leq[kFW], s_nf;
      __shared__ uint32_t s_wb[kFW + 1];                 // this CTA's warp boundaries (elements)
      const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kFW;
      if (threadIdx.x <= kFW) s_wb[threadIdx.x] = static_cast<uint32_t>(min(n, (w0 + threadIdx.x) * nq / W * kQ));
      if (threadIdx.x < kFW) {
        s_lgt[threadIdx.x] = 0;
        s_leq[threadIdx.x] = 0;
      }
      if (threadIdx.x == 0) s_nf = 0;
      __syncthreads();
      const uint32_t ca = s_wb[0], cend = s_wb[kFW];
      // the warp of this CTA whose range holds element ix (ca <= ix < cend)
      auto warp_of = [&](uint32_t ix) -> unsigned int {
        unsigned int w = 0;
#pragma unroll
        for (unsigned int st2 = kFW / 2; st2; st2 >>= 1)
          if (s_wb[w + st2] <= ix) w += st2;
        return w;
      };
      unsigned long long bgt = 0, beq = 0;               // before this CTA: keys > T, == T
#pragma unroll 1
      for (unsigned int j = threadIdx.x; j < nl; j += kFT) {
        const uint2 e = cached ? lst[j] : __ldcg(blist + j);
        if (e.x > fhi) {
          if (e.y < ca) ++bgt;
          else if (e.y < cend) atomicAdd(s_lgt + warp_of(e.y), 1u);
        } else if (e.x - flo <= fw) {
          const unsigned int p = atomicAdd(&s_nf, 1u);
          keys[p] = e.x;
          kidx[p] = e.y;
        }
      }
      __syncthreads();
      phase_time(st, 1);
      const unsigned int nf = s_nf;
      if (nf <= 32u) {                                   // F's few keys ranked by one warp
        __shared__ uint32_t s_T;
        __shared__ unsigned long long s_neq;
        if (warp == 0) {
          const bool have = lane < nf;
          const uint32_t u = have ? keys[lane] : 0u;
          unsigned int gt = 0, eq = 0;
          for (unsigned int j = 0; j < nf; ++j) {
            const uint32_t v = __shfl_sync(0xFFFFFFFFu, u, j);
            gt += v > u ? 1u : 0u;
            eq += v == u ? 1u : 0u;
          }
          // the key of rank need_f from the top: gt < need_f <= gt + eq
          const bool mine = have && gt < need_f && need_f <= static_cast<unsigned long long>(gt) + eq;
          const unsigned int mm = __ballot_sync(0xFFFFFFFFu, mine);
          if (mm && lane == static_cast<unsigned int>(__ffs(mm) - 1)) {
            s_T = u;
            s_neq = need_f - gt;
          }
        }
        __syncthreads();
        T = s_T;
        need_eq = s_neq;
      } else {
        select_in_f(keys, nf, flo, shf, need_f, fine_s, T, need_eq);
      }
      phase_time(st, 2);
      for (unsigned int j = threadIdx.x; j < nf; j += kFT) {
        const uint32_t u = keys[j], ix = kidx[j];
        if (u >= T) {
          if (ix < ca) {
            if (u > T) ++bgt; else ++beq;
          } else if (ix < cend) {
            atomicAdd((u > T ? s_lgt : s_leq) + warp_of(ix), 1u);
          }
        }
      }
      // CTAs before this one: their keys above the bracket
      const unsigned long long g = threadIdx.x < blockIdx.x ? __ldcg(cta_abv + threadIdx.x) : 0ull;
      unsigned long long tg, tge;                        // (list counts <= 2^16 each: packed)
      block_exclusive_scan(g, sw64h, tg);
      block_exclusive_scan((bgt << 32) | beq, sw64h, tge);
      if (threadIdx.x == 0) {
        s_before[0] = tg + (tge >> 32);
        s_before[1] = tge & 0xFFFFFFFFull;
      }
      __syncthreads();
      phase_time(st, 8);
      gt_w = (run - inbc) + s_lgt[warp];
      eq_w = s_leq[warp];
    } else {
      ok = false;                                        // the hint missed: the grid-wide select
    }
  } else {
    // ---- the fine bin F holding rank k (every CTA, from the merged bins)
    unsigned int part = 0;
    for (int i = threadIdx.x; i < kFine; i += kFT) {
      const unsigned int c = __ldcg(st->fine + i);
      fine_s[i] = c;
      part += c;
    }
    unsigned int in_bracket;
    block_exclusive_scan32(part, sw32, in_bracket);
    above_tot = __ldcg(&st->staged) - in_bracket;      // keys above the bracket
    ok = above_tot < k && k <= above_tot + in_bracket;
    if (ok) {
      select_digit(fine_s, kFine, k - above_tot, fb, above_f);
      ok = fine_s[fb] <= static_cast<unsigned int>(kCandCap);
    }
  }
  if (fastb) {
    // done above
  } else if (ok) {
    const uint32_t flo = lo + (fb << shf);
    const uint64_t fhi64 = static_cast<uint64_t>(flo) + (1ull << shf) - 1ull;
    const uint32_t fhi = fhi64 > hi ? hi : static_cast<uint32_t>(fhi64);
    const uint32_t fw = fhi - flo;
    // ---- gather: this warp's keys above F counted, its keys inside F listed
    // (into a per-warp scratch in the idle ring during the walk, copied out
    // once the CTA's slot in the global list is known)
    constexpr unsigned int kScr = kStages * kCW / 2;     // (key, index) pairs per warp
    uint2* scr = reinterpret_cast<uint2*>(wring);
    unsigned int gtf = 0, winf = 0;
    if (!ovf) {
#pragma unroll 1
      for (unsigned int i0 = 0; i0 < run; i0 += 256) {
        uint2 pr[8];                                     // eight loads in flight per lane
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const unsigned int i = i0 + lane + 32 * t;
          pr[t] = i < run ? __ldcg(sp + i) : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const uint32_t u = rank_key<MAG>(__uint_as_float(pr[t].x));
          const bool in = i0 + lane + 32 * t < run;
          gtf += (in && u > fhi) ? 1u : 0u;
          const bool f = in && u - flo <= fw;
          const unsigned int fb_ = __ballot_sync(0xFFFFFFFFu, f);
          if (f) {
            const unsigned int p = winf + __popc(fb_ & lt);
            if (p < kScr) scr[p] = make_uint2(u, pr[t].y);
          }
          winf += __popc(fb_);
        }
      }
    } else {
#pragma unroll 1
      for (int64_t c0 = a; c0 < end; c0 += kChunkW) {
        const int64_t base = c0 + 16 * lane;
        load16(x, end, base, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t u = rank_key<MAG>(v[j]);
          const bool okj = base + j < end;
          gtf += (okj && u > fhi) ? 1u : 0u;
          winf += __popc(__ballot_sync(0xFFFFFFFFu, okj && u - flo <= fw));
        }
      }
    }
    gtf = __reduce_add_sync(0xFFFFFFFFu, gtf);
    // one atomic per CTA: the warps' F counts scanned in shared memory
    if (lane == 0) w_eq[warp] = winf;
    __syncthreads();
    if (warp == 0) {
      const unsigned int c = w_eq[lane];
      const unsigned int ci = warp_incl_scan(c);
      unsigned int cb = 0;
      if (lane == 31 && ci) cb = atomicAdd(&st->inf_count, ci);
      cb = __shfl_sync(0xFFFFFFFFu, cb, 31);
      w_gt[lane] = cb + ci - c;                          // this warp's first slot
    }
    __syncthreads();
    const unsigned int gbase = w_gt[warp];
    __syncthreads();
    if (winf && !ovf && winf <= kScr) {
      for (unsigned int j = lane; j < winf; j += 32) cands[gbase + j] = scr[j];
    } else if (winf) {                                   // rare: walk again, listing F's keys
      unsigned int pos = gbase;
      if (!ovf) {
        for (unsigned int i0 = 0; i0 < run; i0 += 32) {
          const unsigned int i = i0 + lane;
          const uint2 pr = i < run ? __ldcg(sp + i) : make_uint2(0u, 0u);
          const uint32_t u = rank_key<MAG>(__uint_as_float(pr.x));
          const bool f = i < run && u - flo <= fw;
          const unsigned int fb_ = __ballot_sync(0xFFFFFFFFu, f);
          if (f) cands[pos + __popc(fb_ & lt)] = make_uint2(u, pr.y);
          pos += __popc(fb_);
        }
      } else {
#pragma unroll 1
        for (int64_t c0 = a; c0 < end; c0 += kChunkW) {
          const int64_t base = c0 + 16 * lane;
          load16(x, end, base, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t u = rank_key<MAG>(v[j]);
            const bool f = base + j < end && u - flo <= fw;
            const unsigned int fb_ = __ballot_sync(0xFFFFFFFFu, f);
            if (f) cands[pos + __popc(fb_ & lt)] = make_uint2(u, static_cast<unsigned int>(base + j));
            pos += __popc(fb_);
          }
        }
      }
    }
    phase_time(st, 5);
    grid_sync(&st->bar, G * nbar++);
    phase_time(st, 6);
    // ---- rank: T among F's keys (every CTA), then this warp's kept counts
    const unsigned int nc = __ldcg(&st->inf_count);
    const unsigned long long need_f = k - above_tot - above_f;
    uint32_t* keys = reinterpret_cast<uint32_t*>(ring);
    uint32_t* kidx = keys + kCandSmem;
    const bool in_smem = nc <= static_cast<unsigned int>(kCandSmem);
    if (in_smem) {
      for (unsigned int j = threadIdx.x; j < nc; j += kFT) {
        const uint2 c = __ldcg(cands + j);
        keys[j] = c.x;
        kidx[j] = c.y;
      }
      __syncthreads();
      select_in_f(keys, nc, flo, shf, need_f, fine_s, T, need_eq);
    } else {
      cta_select([&](int64_t j) { return __ldcg(&cands[j].x); }, nc, flo, fhi, need_f, T, need_eq);
    }
    // F's keys >= T inside this CTA's range, listed once per CTA (a few)
    __shared__ unsigned int s_nloc;
    uint32_t* lkey = kidx + kCandSmem;
    uint32_t* lidx = lkey + kLocal;
    const int64_t cq0 = static_cast<int64_t>(blockIdx.x) * kFW * nq / W, cq1 = (static_cast<int64_t>(blockIdx.x) + 1) * kFW * nq / W;
    const int64_t ca = cq0 * kQ, cend = min(n, cq1 * kQ);
    if (threadIdx.x == 0) s_nloc = 0;
    __syncthreads();
    for (unsigned int j = threadIdx.x; j < nc; j += kFT) {
      const uint32_t key = in_smem ? keys[j] : __ldcg(&cands[j].x);
      const int64_t ix = in_smem ? kidx[j] : __ldcg(&cands[j].y);
      if (ix >= ca && ix < cend && key >= T) {
        const unsigned int p = atomicAdd(&s_nloc, 1u);
        if (p < static_cast<unsigned int>(kLocal)) {
          lkey[p] = key;
          lidx[p] = static_cast<uint32_t>(ix);
        }
      }
    }
    __syncthreads();
    const unsigned int nloc = s_nloc;
    const bool local = nloc <= static_cast<unsigned int>(kLocal);
    const unsigned int nscan = local ? nloc : nc;
    unsigned int cg = 0, ce = 0;
    for (unsigned int j = lane; j < nscan; j += 32) {
      const uint32_t key = local ? lkey[j] : (in_smem ? keys[j] : __ldcg(&cands[j].x));
      const int64_t ix = local ? lidx[j] : (in_smem ? kidx[j] : __ldcg(&cands[j].y));
      if (ix >= a && ix < end) {
        cg += key > T ? 1u : 0u;
        ce += key == T ? 1u : 0u;
      }
    }
    gt_w = gtf + __reduce_add_sync(0xFFFFFFFFu, cg);
    eq_w = __reduce_add_sync(0xFFFFFFFFu, ce);
  } else {
    // ---- slow path: T by a grid-wide 8-bit radix select over x, four rounds
    uint32_t prefix = 0, mask = 0;
    unsigned long long need = k;
    unsigned int* h = fine_s;                            // 256 bins
#pragma unroll 1
    for (int r = 0; r < 4; ++r) {
      const int shift = 24 - 8 * r;
      __syncthreads();
      for (int i = threadIdx.x; i < 256; i += kFT) h[i] = 0;
      __syncthreads();
#pragma unroll 1
      for (int64_t c0 = a; c0 < end; c0 += kChunkW) {
        const int64_t base = c0 + 16 * lane;
        load16(x, end, base, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t u = rank_key<MAG>(v[j]);
          if (base + j < end && (u & mask) == prefix) atomicAdd(h + ((u >> shift) & 0xFFu), 1u);
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < 256; i += kFT)
        if (h[i]) atomicAdd(&st->rhist[r][i], h[i]);
      grid_sync(&st->bar, G * nbar++);
      for (int i = threadIdx.x; i < 256; i += kFT) h[i] = __ldcg(&st->rhist[r][i]);
      __syncthreads();
      unsigned int d;
      unsigned long long ab;
      select_digit(h, 256, need, d, ab);
      prefix |= d << shift;
      mask |= 0xFFu << shift;
      need -= ab;
    }
    T = prefix;
    need_eq = need;
    ovf = true;                                          // every warp emits from x
    unsigned int g = 0, e = 0;
#pragma unroll 1
    for (int64_t c0 = a; c0 < end; c0 += kChunkW) {
      const int64_t base = c0 + 16 * lane;
      load16(x, end, base, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t u = rank_key<MAG>(v[j]);
        const bool okj = base + j < end;
        g += (okj && u > T) ? 1u : 0u;
        e += (okj && u == T) ? 1u : 0u;
      }
    }
    gt_w = __reduce_add_sync(0xFFFFFFFFu, g);
    eq_w = __reduce_add_sync(0xFFFFFFFFu, e);
  }
  // ---- offsets: warps of this CTA, then the CTAs before it
  if (lane == 0) {
    w_gt[warp] = gt_w;
    w_eq[warp] = eq_w;
  }
  __syncthreads();
  unsigned long long wg_ex, we_ex;
  {
    const unsigned int g = w_gt[lane], e = w_eq[lane];
    wg_ex = __reduce_add_sync(0xFFFFFFFFu, lane < warp ? g : 0u);
    we_ex = __reduce_add_sync(0xFFFFFFFFu, lane < warp ? e : 0u);
    if (warp == 0 && !fastb) {
      const unsigned int tg = __reduce_add_sync(0xFFFFFFFFu, g), te = __reduce_add_sync(0xFFFFFFFFu, e);
      if (lane == 0) {
        cta_tot[2 * blockIdx.x] = tg;
        cta_tot[2 * blockIdx.x + 1] = te;
      }
    }
  }
  if (HINT && blockIdx.x == 0 && threadIdx.x == 0) {   // the next call's bracket (read before barrier 1)
    const uint32_t nh = hv && !fastb ? (hhalf < (1u << 22) ? 2u * hhalf : hhalf) : hhalf;
    __stcg(reinterpret_cast<uint4*>(hint), make_uint4(MAG ? 1u : 0u, T, nh, 0u));
  }
  phase_time(st, 7);
  if (!fastb) {
    grid_sync(&st->bar, G * nbar++);
    phase_time(st, 8);
    unsigned long long g = 0, e = 0;
    if (threadIdx.x < blockIdx.x) {
      g = __ldcg(cta_tot + 2 * threadIdx.x);
      e = __ldcg(cta_tot + 2 * threadIdx.x + 1);
    }
    __shared__ unsigned long long sw64[kFW];
    unsigned long long tg, te;
    block_exclusive_scan(g, sw64, tg);
    block_exclusive_scan(e, sw64, te);
    if (threadIdx.x == 0) {
      s_before[0] = tg;
      s_before[1] = te;
    }
    __syncthreads();
  }
  if (HINT) {                                            // the persistent state: last CTA out resets it
    __shared__ unsigned int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&st->done, 1u) == G - 1u;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      constexpr int nw = static_cast<int>(offsetof(PruneState, t) / 4);
      unsigned int* w = reinterpret_cast<unsigned int*>(st);
      for (int i = threadIdx.x; i < nw; i += kFT) w[i] = 0u;
    }
  }
  if (row_ptr && blockIdx.x == 0 && threadIdx.x == 0) row_ptr[n / row_len] = static_cast<int32_t>(k);
  if (a >= end) return;
  const unsigned long long gb = s_before[0] + wg_ex, eb = s_before[1] + we_ex;
  const unsigned long long off = gb + (eb < need_eq ? eb : need_eq);
  const bool ties = eq_w != 0;
  if (!ovf)
    emit_staged<MAG>(sp, run, a, end, T, ties, need_eq, off, eb, values, indices, row_len, row_ptr,
                     reinterpret_cast<uint2*>(wring));
  else
    emit_from_x<MAG>(x, a, end, T, ties, need_eq, off, eb, values, indices, row_len, row_ptr);
  phase_time(st, 9);
}

// ------------------------------------------------------------------ K7

// first position j in [lo, hi) with indices[j] >= target (hi if none),
// given that the answer lies in [lo, hi]; 32-way warp search
__device__ int64_t warp_lower_bound(const int32_t* __restrict__ idx, int64_t lo, int64_t hi,
                                    int64_t target) {
  const int lane = threadIdx.x & 31;
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

// dense = 0 with survivors scattered in.  Persistent CTAs, each owning a
// contiguous run of 4096-float output tiles: one 32-way search finds where
// the CTA's run starts in the ascending index list, after which the list is
// read sequentially -- per tile one round of 1024 (index, value) loads
// (four per thread, all in flight), the in-tile ones scattered into the
// tile in shared memory (a prefix of the round, the indices ascend), then
// the tile leaves in float4 stores and is re-zeroed by the same threads.
// DRAM sees one coalesced write per output byte and one read per survivor.
constexpr int kRRound = 4 * kPT;

__global__ void __launch_bounds__(kPT) k_restore(const float* __restrict__ values,
                                                 const int32_t* __restrict__ indices, int64_t k,
                                                 float* __restrict__ dense, int64_t n) {
  __shared__ float4 tile4[kRTile / 4];
  float* tile = reinterpret_cast<float*>(tile4);
  __shared__ int64_t s_j;
  const int64_t ntiles = (n + kRTile - 1) / kRTile;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * ntiles / gridDim.x;
  const int64_t t1 = (static_cast<int64_t>(blockIdx.x) + 1) * ntiles / gridDim.x;
  if (t0 >= t1) return;
  if (threadIdx.x < 32) {
    const int64_t r = warp_lower_bound(indices, 0, k, t0 * kRTile);
    if (threadIdx.x == 0) s_j = r;
  }
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = threadIdx.x; i < kRTile / 4; i += kPT) tile4[i] = z;
  __syncthreads();
  int64_t j = s_j;
  __shared__ int s_cnt[kPT / 32];
  const bool vec = aligned16(dense);
#pragma unroll 1
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t base = t * kRTile, lim = min(n, base + kRTile);
#pragma unroll 1
    while (true) {                                       // rounds until the tile's slice ends
      int32_t ix[4];
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t jj = j + threadIdx.x + q * kPT;
        ix[q] = jj < k ? __ldg(indices + jj) : 0x7FFFFFFF;
        v[q] = jj < k ? __ldg(values + jj) : 0.f;
      }
      int in = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (ix[q] < lim) {
          tile[ix[q] - base] = v[q];
          ++in;
        }
      }
      in = __reduce_add_sync(0xFFFFFFFFu, in);
      if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = in;
      __syncthreads();
      int taken = 0;
#pragma unroll
      for (int w = 0; w < kPT / 32; ++w) taken += s_cnt[w];
      __syncthreads();
      j += taken;
      if (taken < kRRound) break;
    }
    if (vec && lim - base == kRTile) {
      float4* d4 = reinterpret_cast<float4*>(dense + base);
#pragma unroll
      for (int i = threadIdx.x; i < kRTile / 4; i += kPT) {
        d4[i] = tile4[i];
        tile4[i] = z;
      }
    } else {
      for (int64_t i = threadIdx.x; i < kRTile; i += kPT) {
        if (base + i < lim) dense[base + i] = tile[i];
        tile[i] = 0.f;
      }
    }
    __syncthreads();
  }
}

// K7 with the CSR row pointers sf_prune_topk_rows writes: a CTA restores
// kRRows rows; its slice of (index, value) pairs is [row_ptr[r0],
// row_ptr[r0 + kRRows]) -- no search.  Pairs scatter into a zeroed shared
// tile (every load of the slice issued before any store), the tile leaves
// as float4 stores.
constexpr int kRRows = 8;
__global__ void __launch_bounds__(kPT) k_restore_rows(const float* __restrict__ values,
                                                      const int32_t* __restrict__ indices,
                                                      const int32_t* __restrict__ row_ptr, int64_t rows, int H,
                                                      float* __restrict__ dense) {
  extern __shared__ float4 rtile4[];
  float* tile = reinterpret_cast<float*>(rtile4);
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRRows;
  const int nr = static_cast<int>(rows - r0 < kRRows ? rows - r0 : kRRows);
  const int len = nr * H, len4 = len >> 2;
  const int64_t a = __ldg(row_ptr + r0), b = __ldg(row_ptr + r0 + nr);
  const int64_t base = r0 * H;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = threadIdx.x; i < len4; i += kPT) rtile4[i] = z;
  __syncthreads();
  for (int64_t j0 = a + threadIdx.x; j0 < b; j0 += 4 * kPT) {
    int32_t ix[4];
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + q * kPT;
      ix[q] = j < b ? __ldg(indices + j) : -1;
      v[q] = j < b ? __ldg(values + j) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ix[q] >= 0) tile[ix[q] - base] = v[q];
  }
  __syncthreads();
  float4* d4 = reinterpret_cast<float4*>(dense + base);
  for (int i = threadIdx.x; i < len4; i += kPT) d4[i] = rtile4[i];
}

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// CTAs of the persistent kernel: every one must be resident at once
template <bool MAG>
int prune_grid() {
  static int cached[2][64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int& g = cached[MAG ? 1 : 0][dev];
  if (g == 0) {
    cudaFuncSetAttribute(k_prune<MAG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kFusedSmem));
    cudaFuncSetAttribute(k_prune<MAG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kFusedSmem));
    int per_sm = 0, per_sm_h = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_prune<MAG, false>, kFT, kFusedSmem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_h, k_prune<MAG, true>, kFT, kFusedSmem) ==
            cudaSuccess && per_sm_h >= 1 && per_sm_h < per_sm)
      per_sm = per_sm_h;                                 // both variants co-resident at this grid
    g = per_sm * num_sms();
  }
  return g;
}

struct PruneWs {
  PruneState* st;
  unsigned long long* cta_tot;
  uint2* cands;
  uint2* staged;
  uint2* blist;
  unsigned long long* cta_abv;
};

// state (memset per call) | per-CTA totals | F gather | staged values | staged indices
inline size_t carve(void* ws, int64_t n, int grid, PruneWs* w) {
  const int64_t W = static_cast<int64_t>(grid) * kFW;
  const int64_t nq = (n + kQ - 1) / kQ;
  const int64_t slots = nq * 5 / 2 + kSlack * (W + 1);
  char* base = static_cast<char*>(ws);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* q = base ? base + o : nullptr;
    o += align256(bytes);
    return q;
  };
  PruneWs t;
  t.st = reinterpret_cast<PruneState*>(take(sizeof(PruneState)));
  t.cta_tot = reinterpret_cast<unsigned long long*>(take(2 * grid * sizeof(unsigned long long)));
  t.cands = reinterpret_cast<uint2*>(take(kCandCap * sizeof(uint2)));
  t.staged = reinterpret_cast<uint2*>(take(slots * sizeof(uint2)));
  t.blist = reinterpret_cast<uint2*>(take(kBListCap * sizeof(uint2)));
  t.cta_abv = reinterpret_cast<unsigned long long*>(take(grid * sizeof(unsigned long long)));
  if (w) *w = t;
  return o;
}

template <bool MAG>
int launch_prune(const float* x, int64_t n, int64_t k, float* values, int32_t* indices, int row_len,
                 int32_t* row_ptr, uint32_t* hint, void* ws, cudaStream_t s) {
  const int grid = prune_grid<MAG>();
  PruneWs w;
  carve(ws, n, grid, &w);
  if (hint) {                                           // state in the hint buffer, left zeroed by each call
    PruneState* hs = reinterpret_cast<PruneState*>(reinterpret_cast<char*>(hint) + kHintHeader);
    k_prune<MAG, true><<<grid, kFT, kFusedSmem, s>>>(x, n, static_cast<unsigned long long>(k), hs, w.cta_tot,
                                                     w.cands, w.staged, values, indices, row_len, row_ptr, hint,
                                                     w.blist, w.cta_abv);
    return check_launch();
  }
  if (cudaMemsetAsync(w.st, 0, sizeof(PruneState), s) != cudaSuccess) return check_launch();
  k_prune<MAG, false><<<grid, kFT, kFusedSmem, s>>>(x, n, static_cast<unsigned long long>(k), w.st, w.cta_tot,
                                                      w.cands, w.staged, values, indices, row_len, row_ptr, nullptr,
                                                      w.blist, w.cta_abv);
  return check_launch();
}

}  // namespace sf

using namespace sf;

extern "C" {

size_t sf_prune_workspace_bytes(int64_t n) {
  return carve(nullptr, n > 0 ? n : 1, std::max(prune_grid<true>(), prune_grid<false>()), nullptr);
}

int sf_prune_topk_rows(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                       int32_t* indices, int64_t row_len, int32_t* row_ptr, void* ws, void* stream) {
  if (n <= 0 || k < 1 || k > n || n > 0x7FFFFFFFLL || !x || !values || !indices || !ws)
    return SF_EINVAL;
  if (row_ptr && (row_len <= 0 || row_len > 0x7FFFFFFF || n % row_len)) return SF_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int rl = row_ptr ? static_cast<int>(row_len) : 1;
  if (by_magnitude) return launch_prune<true>(x, n, k, values, indices, rl, row_ptr, nullptr, ws, s);
  return launch_prune<false>(x, n, k, values, indices, rl, row_ptr, nullptr, ws, s);
}

size_t sf_prune_hint_bytes(void) { return kHintHeader + sizeof(PruneState); }

int sf_prune_topk_hint(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                       int32_t* indices, int64_t row_len, int32_t* row_ptr, uint32_t* hint, void* ws,
                       void* stream) {
  if (!hint || (reinterpret_cast<uintptr_t>(hint) & 15u)) return SF_EINVAL;
  if (n <= 0 || k < 1 || k > n || n > 0x7FFFFFFFLL || !x || !values || !indices || !ws)
    return SF_EINVAL;
  if (row_ptr && (row_len <= 0 || row_len > 0x7FFFFFFF || n % row_len)) return SF_EINVAL;
  cudaStream_t s = as_stream(stream);
  const int rl = row_ptr ? static_cast<int>(row_len) : 1;
  if (by_magnitude) return launch_prune<true>(x, n, k, values, indices, rl, row_ptr, hint, ws, s);
  return launch_prune<false>(x, n, k, values, indices, rl, row_ptr, hint, ws, s);
}

int sf_prune_topk(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                  int32_t* indices, void* ws, void* stream) {
  return sf_prune_topk_rows(x, n, k, by_magnitude, values, indices, 0, nullptr, ws, stream);
}

int sf_restore(const float* values, const int32_t* indices, int64_t k, float* dense, int64_t n,
               void* stream) {
  if (n <= 0 || k < 0 || k > n || !dense || (k > 0 && (!values || !indices))) return SF_EINVAL;
  const int64_t ntiles = (n + kRTile - 1) / kRTile;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  k_restore<<<static_cast<unsigned>(ntiles < cap ? ntiles : cap), kPT, 0, as_stream(stream)>>>(values, indices, k,
                                                                                                dense, n);
  return check_launch();
}

int sf_restore_rows(const float* values, const int32_t* indices, int64_t k, const int32_t* row_ptr,
                    int64_t row_len, float* dense, int64_t n, void* stream) {
  if (n <= 0 || k < 0 || k > n || !dense || !row_ptr || (k > 0 && (!values || !indices)) || row_len <= 0 ||
      row_len % 4 || n % row_len || row_len * kRRows * 4 > 48 * 1024 || !aligned16(dense))
    return SF_EINVAL;
  const int64_t rows = n / row_len;
  const int64_t grid = (rows + kRRows - 1) / kRRows;
  if (grid > INT32_MAX) return SF_EINVAL;
  k_restore_rows<<<static_cast<unsigned>(grid), kPT, static_cast<size_t>(row_len) * kRRows * 4,
                   as_stream(stream)>>>(values, indices, row_ptr, rows, static_cast<int>(row_len), dense);
  return check_launch();
}

}  // extern "C"
