// Prune state shared by the prune passes (prune.cu) and the LayerNorm
// forward that can run the first pass fused (layernorm.cu,
// sf_layernorm_fwd_prune_hist): the key bracket, the fine histogram over
// it and the counts, plus the order-preserving key helpers.
#pragma once

#include "common.cuh"

namespace sf {

constexpr int kFine = 4096;              // fine bins inside the bracket

struct PruneState {
  unsigned int lo, hi, shf;       // P1's key bracket and fine-bin shift (written by CTA 0)
  unsigned int T;                 // exact threshold key (P2 finish)
  unsigned int fine_lo, fine_hi;  // key range of the selected fine bin F (written by P2 CTA 0)
  int mode;                       // 0 fast; 2 = bracket missed / F too heavy: the P2 finish
                                  // selects T exactly and counts the tiles itself
  unsigned int cand_count;
  unsigned long long above;       // keys above the bracket (P1 atomics)
  unsigned long long need_f;      // rank (1-based from the top) inside F
  unsigned long long need_eq;     // keys == T to keep, in index order
  unsigned int fine[kFine];
};

template <bool MAG>
__device__ __forceinline__ uint32_t rank_key(float x) {
  uint32_t b = __float_as_uint(x);
  const bool is_nan = (b & 0x7FFFFFFFu) > 0x7F800000u;
  uint32_t u;
  if (MAG) {
    u = (b & 0x7FFFFFFFu) + 1u;
  } else {
    b = b == 0x80000000u ? 0u : b;                                  // -0.0 ties with +0.0
    u = b ^ (static_cast<uint32_t>(static_cast<int32_t>(b) >> 31) | 0x80000000u);
  }
  return is_nan ? 0u : u;                                           // NaN ranks lowest
}

// Magnitude keys without materialising them: with a = bits & 0x7FFFFFFF,
// u = a + 1 for numbers and 0 for NaN, so for any key K
//   u > K  <=>  K <= a <= 0x7F800000  <=>  (a - K) <= (0x7F800000 - K)
// (one subtract and one unsigned compare; NaN fails automatically).
struct MagGt {
  uint32_t sub, lim;
  __device__ __forceinline__ bool operator()(uint32_t a) const { return a - sub <= lim; }
};
__device__ __forceinline__ MagGt mag_gt(uint32_t K) {
  return K <= 0x7F800000u ? MagGt{K, 0x7F800000u - K} : MagGt{0x80000000u, 0u};   // else: none
}
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

// shared-memory histogram increment of bin (d >> shf) when d <= wid: one
// predicated red.shared on a 32-bit shared address (no branch, no generic
// address conversion inside the loop)
__device__ __forceinline__ void red_bin(uint32_t base_s, uint32_t d, uint32_t wid, uint32_t shf) {
  // out-of-bracket keys go to a dummy bin just past the histogram
  // (bins[kFine]): the increment is unconditional, so there is no branch per
  // key, and the warp-aggregated shared increment absorbs the (many) keys
  // that hit the dummy together
  const uint32_t bin = d <= wid ? (d >> shf) : static_cast<uint32_t>(kFine);
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(base_s + (bin << 2)) : "memory");
}

}  // namespace sf
