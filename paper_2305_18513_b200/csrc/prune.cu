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
// Selection of the k-th largest key T is an 11/11/10-bit MSD radix select
// (three histogram passes, each finished by the last CTA to arrive, so no
// host round trip).  Then a tile pass counts (#u > T, #u == T) per tile, one
// CTA scans the tile counts, and a write pass emits the kept (value, index)
// pairs in ascending index order: every u > T plus the first k - #(u > T)
// elements with u == T in index order (stable ties toward the lower index).
#include "common.cuh"

namespace sf {

constexpr int kPT = 256;                 // threads per CTA
constexpr int kPerThread = 16;           // elements per thread in tile passes
constexpr int kTile = kPT * kPerThread;  // 4096 elements per tile
constexpr int kDigits = 2048;

struct PruneState {
  unsigned int hist[3][kDigits];
  unsigned int ticket[3];
  unsigned int prefix;        // key bits fixed so far
  unsigned int mask;          // which bits of prefix are fixed
  unsigned long long k_rem;   // rank (1-based, from the top) still to find below prefix
  unsigned long long n_gt;    // keys strictly greater than the final threshold
  unsigned long long need_eq; // keys equal to the threshold to keep (index order)
};

__device__ __forceinline__ uint32_t rank_key(float x, bool mag) {
  uint32_t b = __float_as_uint(x);
  if ((b & 0x7FFFFFFFu) > 0x7F800000u) return 0u;   // NaN ranks lowest
  if (mag) return (b & 0x7FFFFFFFu) + 1u;
  if (b == 0x80000000u) b = 0u;                     // -0.0 ties with +0.0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ int pass_shift(int p) { return p == 0 ? 21 : (p == 1 ? 10 : 0); }
__device__ __forceinline__ uint32_t pass_dmask(int p) { return p == 2 ? 0x3FFu : 0x7FFu; }

// One radix pass: histogram of digit p among keys matching the prefix; the
// last CTA picks the digit holding rank k_rem and narrows the prefix.
__global__ void __launch_bounds__(kPT) k_radix_pass(const float* __restrict__ x, int64_t n,
                                                    bool mag, int p, PruneState* st) {
  __shared__ unsigned int sh[kDigits];
  for (int i = threadIdx.x; i < kDigits; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t prefix = st->prefix, mask = st->mask;
  const int shift = pass_shift(p);
  const uint32_t dm = pass_dmask(p);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = aligned16(x);
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += stride) {
    float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
    uint32_t u0 = rank_key(v.x, mag), u1 = rank_key(v.y, mag), u2 = rank_key(v.z, mag),
             u3 = rank_key(v.w, mag);
    if ((u0 & mask) == prefix) atomicAdd(sh + ((u0 >> shift) & dm), 1u);
    if ((u1 & mask) == prefix) atomicAdd(sh + ((u1 >> shift) & dm), 1u);
    if ((u2 & mask) == prefix) atomicAdd(sh + ((u2 >> shift) & dm), 1u);
    if ((u3 & mask) == prefix) atomicAdd(sh + ((u3 >> shift) & dm), 1u);
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    uint32_t u = rank_key(x[i], mag);
    if ((u & mask) == prefix) atomicAdd(sh + ((u >> shift) & dm), 1u);
  }
  __syncthreads();
  unsigned int* gh = st->hist[p];
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
  if (threadIdx.x == 0) {
    // sequential over 256 thread sums (from the top), then inside the thread
    unsigned long long need = st->k_rem, above = 0;
    int t = kPT - 1;
    while (t > 0 && above + tsum[t] < need) above += tsum[t--];
    tsum[0] = above;                 // keys above thread t's digits
    tsum[1] = static_cast<unsigned long long>(t);
  }
  __syncthreads();
  if (threadIdx.x == static_cast<int>(tsum[1])) {
    unsigned long long need = st->k_rem, above = tsum[0];
    int d = kPer - 1;
    while (d > 0 && above + loc[d] < need) above += loc[d--];
    const uint32_t digit = static_cast<uint32_t>(threadIdx.x * kPer + d);
    st->prefix = prefix | (digit << shift);
    st->mask = mask | (dm << shift);
    st->k_rem = need - above;          // rank within the chosen digit
    st->n_gt += above;
    if (p == 2) st->need_eq = st->k_rem;
  }
}

// Zero the selection state; k_rem starts at k (rank from the top, 1-based).
__global__ void k_prune_init(PruneState* st, unsigned long long k) {
  unsigned int* h = &st->hist[0][0];
  for (int i = threadIdx.x; i < 3 * kDigits; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) {
    st->ticket[0] = st->ticket[1] = st->ticket[2] = 0;
    st->prefix = 0;
    st->mask = 0;
    st->k_rem = k;
    st->n_gt = 0;
    st->need_eq = 0;
  }
}

// Per tile: (#u > T, #u == T).  Coalesced layout (order does not matter).
__global__ void __launch_bounds__(kPT) k_tile_count(const float* __restrict__ x, int64_t n,
                                                    bool mag, const PruneState* __restrict__ st,
                                                    unsigned int* __restrict__ tile_gt,
                                                    unsigned int* __restrict__ tile_eq) {
  const uint32_t T = st->prefix;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  unsigned int gt = 0, eq = 0;
#pragma unroll 4
  for (int j = 0; j < kPerThread; ++j) {
    int64_t i = base + j * kPT + threadIdx.x;
    if (i < n) {
      uint32_t u = rank_key(x[i], mag);
      gt += u > T;
      eq += u == T;
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
}

// Exclusive scans over tiles: output offset and equal-keys-before counts.
__global__ void __launch_bounds__(1024) k_tile_scan(int64_t ntiles, const PruneState* st,
                                                    const unsigned int* __restrict__ tile_gt,
                                                    const unsigned int* __restrict__ tile_eq,
                                                    unsigned long long* __restrict__ out_off,
                                                    unsigned long long* __restrict__ eq_before) {
  const unsigned long long need_eq = st->need_eq;
  const int64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
  unsigned long long eqs = 0, gts = 0;
  for (int64_t t = t0; t < t1; ++t) {
    eqs += tile_eq[t];
    gts += tile_gt[t];
  }
  __shared__ unsigned long long se[1024], sg[1024];
  se[threadIdx.x] = eqs;
  sg[threadIdx.x] = gts;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {   // Hillis-Steele inclusive scan
    unsigned long long a = threadIdx.x >= off ? se[threadIdx.x - off] : 0;
    unsigned long long b = threadIdx.x >= off ? sg[threadIdx.x - off] : 0;
    __syncthreads();
    se[threadIdx.x] += a;
    sg[threadIdx.x] += b;
    __syncthreads();
  }
  unsigned long long eb = se[threadIdx.x] - eqs, gb = sg[threadIdx.x] - gts;
  for (int64_t t = t0; t < t1; ++t) {
    eq_before[t] = eb;
    unsigned long long keq_b = eb < need_eq ? eb : need_eq;
    out_off[t] = gb + keq_b;
    eb += tile_eq[t];
    gb += tile_gt[t];
  }
}

// Write pass: thread t of a tile owns elements [base + 16t, base + 16t + 16)
// so per-thread order is index order; a block scan orders the threads.
__global__ void __launch_bounds__(kPT) k_tile_write(const float* __restrict__ x, int64_t n,
                                                    bool mag, const PruneState* __restrict__ st,
                                                    const unsigned long long* __restrict__ out_off,
                                                    const unsigned long long* __restrict__ eq_before,
                                                    float* __restrict__ values,
                                                    int32_t* __restrict__ indices) {
  const uint32_t T = st->prefix;
  const unsigned long long need_eq = st->need_eq;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile + threadIdx.x * kPerThread;
  float v[kPerThread];
  uint32_t u[kPerThread];
  const bool full = base + kPerThread <= n && aligned16(x);
  if (full) {
#pragma unroll
    for (int j = 0; j < kPerThread / 4; ++j) {
      float4 f = __ldg(reinterpret_cast<const float4*>(x + base) + j);
      v[4 * j] = f.x;
      v[4 * j + 1] = f.y;
      v[4 * j + 2] = f.z;
      v[4 * j + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) v[j] = (base + j < n) ? x[base + j] : 0.f;
  }
  unsigned int neq = 0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    u[j] = (base + j < n) ? rank_key(v[j], mag) : 0u;
    neq += (base + j < n) && u[j] == T;
  }
  // block exclusive scan of neq (to rank ties in index order)
  __shared__ unsigned int warp_tot[kPT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int inc = neq;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned int y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  unsigned int wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
  const unsigned long long eq0 = eq_before[blockIdx.x] + wbase + inc - neq;
  // kept flags and count
  unsigned int kept_mask = 0, nk = 0;
  unsigned long long er = eq0;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    bool in = base + j < n;
    bool keep = in && (u[j] > T || (u[j] == T && er < need_eq));
    if (in && u[j] == T) ++er;
    if (keep) {
      kept_mask |= 1u << j;
      ++nk;
    }
  }
  __syncthreads();
  inc = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned int y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += warp_tot[w];
  unsigned long long pos = out_off[blockIdx.x] + wbase + inc - nk;
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    if (kept_mask & (1u << j)) {
      values[pos] = v[j];
      indices[pos] = static_cast<int32_t>(base + j);
      ++pos;
    }
  }
}

// K7: dense = 0 with survivors scattered in.  Each CTA owns a tile of the
// dense output, finds its slice of the (ascending) index list by binary
// search, writes zeros with float4 stores, then scatters its survivors.
__global__ void __launch_bounds__(kPT) k_restore(const float* __restrict__ values,
                                                 const int32_t* __restrict__ indices, int64_t k,
                                                 float* __restrict__ dense, int64_t n) {
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t t1 = min(n, t0 + kTile);
  __shared__ int64_t range[2];
  if (threadIdx.x < 2) {
    const int64_t target = threadIdx.x == 0 ? t0 : t1;
    int64_t lo = 0, hi = k;   // first j with indices[j] >= target
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (static_cast<int64_t>(__ldg(indices + mid)) < target)
        lo = mid + 1;
      else
        hi = mid;
    }
    range[threadIdx.x] = lo;
  }
  if (aligned16(dense) && t1 - t0 == kTile) {
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
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

  k_prune_init<<<1, kPT, 0, s>>>(st, static_cast<unsigned long long>(k));
  const bool mag = by_magnitude != 0;
  const unsigned grid = grid_for((n + 3) / 4, kPT, 4);
  for (int p = 0; p < 3; ++p) k_radix_pass<<<grid, kPT, 0, s>>>(x, n, mag, p, st);
  k_tile_count<<<static_cast<unsigned>(nt), kPT, 0, s>>>(x, n, mag, st, tile_gt, tile_eq);
  k_tile_scan<<<1, 1024, 0, s>>>(nt, st, tile_gt, tile_eq, out_off, eq_before);
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
