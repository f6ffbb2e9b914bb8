// Prune state (prune.cu): the grid barrier, the fine histogram over the key
// bracket and the counts, plus the order-preserving key helpers.
#pragma once

#include "common.cuh"

namespace sf {

constexpr int kFine = 2048;              // fine bins inside the key bracket

// Zeroed by the launcher before every call (one memset); the per-CTA
// totals and the staging lists live after it in the workspace.
struct PruneState {
  unsigned int bar;               // grid barrier arrivals
  unsigned int inf_count;         // keys of the threshold bin F gathered
  unsigned long long staged;      // keys >= the bracket's low end (all warps)
  unsigned int blist_n;           // hinted path: keys inside the bracket listed (all CTAs)
  unsigned int blist_ovf;         // hinted path: a CTA's or the global bracket list overflowed
  unsigned int fine[kFine];       // histogram of the keys inside the bracket
  unsigned int rhist[4][256];     // slow path: radix-select rounds over x
  unsigned int done;              // hinted (persistent) state: CTAs finished with it
  unsigned int pad_;
  unsigned long long t[10];       // %globaltimer at phase ends (CTA 0; diagnostics; never reset)
};
// sf_prune_topk_hint: the caller's hint buffer = 4 header words + a
// PruneState that the kernel's last CTA leaves zeroed (no memset per call)
constexpr size_t kHintHeader = 16;

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

}  // namespace sf
