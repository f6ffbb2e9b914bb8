// fp32-accurate dense products on the 5th-generation tensor cores (tcgen05).
//
// Reference: the float32 products of `linear` (tensor.py:337-379: x @ W + b,
// g @ W.T, x.T @ g).  Each fp32 operand is split exactly into three bf16
// terms, x = hi + mid + lo (|mid| <= 2^-8 |hi|, |lo| <= 2^-16 |hi|), and the
// product keeps the six partial products that carry fp32 accuracy:
//
//   A B ~= hi.hi + (hi.mid + mid.hi + mid.mid + hi.lo + lo.hi)
//
// accumulated in TWO fp32 TMEM accumulators (the dominant hi.hi term alone,
// the five small terms together), summed once in the epilogue: a single
// accumulator over all six terms loses ~7x accuracy to the tensor core's
// accumulation (profiles/r01_split_gemm_probe.txt).  Compared with cuBLASLt's
// BF16x9 emulation this issues 6 instead of 9 products and skips its
// inf/NaN scan of the operands; non-finite inputs are not patched (a
// non-finite loss skips the step anyway, trainer.py guard).
//
// Kernel (one 128x128 output tile per CTA, 128 threads, 2 CTAs per SM):
//   thread 0   TMA producer: per 32-wide K block six 128x32 bf16 boxes (A and
//              B, three planes each) into a 3-stage ring (64-byte swizzle);
//   thread 32  MMA issuer: 2 x 6 `tcgen05.mma.kind::f16` (M=128, N=128,
//              K=16) per K block, `tcgen05.commit` frees the stage;
//   all warps  epilogue: `tcgen05.ld` both accumulators (warp w owns TMEM
//              lanes 32w..32w+31 = tile rows), + bias, + beta * C, store.
// Two CTAs per SM overlap one tile's epilogue with the other's main loop.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace sf {
namespace {

constexpr int kBM = 128, kBN = 128, kBK = 32;        // tile; kBK bf16 = 64 bytes (SW64 row)
constexpr int kPlaneBytes = kBM * kBK * 2;           // 8 KB per operand plane box
constexpr int kStageBytes = 6 * kPlaneBytes;         // A hi/mid/lo + B hi/mid/lo
constexpr int smem_bytes(int stages) { return stages * kStageBytes + 1024 + 256; }
constexpr uint32_t kTmemCols = 256;                  // two 128-column fp32 accumulators

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major operand tile, rows of 64 bytes with the 64-byte swizzle; 8-row
// core groups 512 bytes apart (SBO), LBO unused for swizzled K-major.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(4) << 61);
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
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

template <int kStages>
__global__ void __launch_bounds__(128, 1)
    k_gemm_split6(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                  int K, float* __restrict__ C, int64_t ldc, const float* __restrict__ bias, float beta,
                  int kb_per, int64_t split_stride) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gen = smem_raw + (base - raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(gen + kStages * kStageBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + kStages), done = su32(bars + 2 * kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kBN, m0 = blockIdx.y * kBM;
  // split-K: this CTA reduces K blocks [kb0, kb0 + nkb) into partial z
  const int kb0 = blockIdx.z * kb_per;
  const int nkb = min((K + kBK - 1) / kBK - kb0, kb_per);
  C += blockIdx.z * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (threadIdx.x == 0) {
    // TMA producer
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages, kb = kb0 + i;
      if (i >= kStages) mbar_wait(empty0 + 8 * s, ((i / kStages) - 1) & 1);
      const uint32_t full = full0 + 8 * s;
      mbar_expect_tx(full, kStageBytes);
      const uint32_t st = base + s * kStageBytes;
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        tma_load_2d(st + p * kPlaneBytes, &tmA, full, kb * kBK, p * M + m0);
        tma_load_2d(st + (3 + p) * kPlaneBytes, &tmB, full, kb * kBK, p * N + n0);
      }
    }
  } else if (threadIdx.x == 32) {
    // MMA issuer: acc0 (columns 0..127) = hi.hi, acc1 (128..255) = the five small terms
    const uint32_t acc0 = tmem, acc1 = tmem + kBN;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kStages;
      mbar_wait(full0 + 8 * s, (i / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t st = base + s * kStageBytes;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
        const uint32_t off = kk * 32;                    // 16 bf16 along K
        const uint64_t ah = smem_desc(st + 0 * kPlaneBytes + off), am = smem_desc(st + 1 * kPlaneBytes + off),
                       al = smem_desc(st + 2 * kPlaneBytes + off);
        const uint64_t bh = smem_desc(st + 3 * kPlaneBytes + off), bm = smem_desc(st + 4 * kPlaneBytes + off),
                       bl = smem_desc(st + 5 * kPlaneBytes + off);
        const uint32_t acc = (i | kk) != 0;
        mma_bf16(acc0, ah, bh, acc);
        mma_bf16(acc1, ah, bm, acc);
        mma_bf16(acc1, am, bh, 1);
        mma_bf16(acc1, am, bm, 1);
        mma_bf16(acc1, ah, bl, 1);
        mma_bf16(acc1, al, bh, 1);
      }
      mma_commit(empty0 + 8 * s);
    }
    mma_commit(done);
  }
  __syncwarp();

  // epilogue: thread = one tile row
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  float* crow = C + static_cast<int64_t>(row) * ldc;
  const bool vec = ((ldc & 3) == 0) && aligned16(C);
#pragma unroll 1
  for (int c = 0; c < kBN; c += 32) {
    float a0[32], a1[32];
    tmem_ld32(lane_base + c, a0);
    tmem_ld32(lane_base + kBN + c, a1);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < M) {
      const int col0 = n0 + c;
      if (vec && col0 + 32 <= N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o;
          o.x = a0[j] + a1[j];
          o.y = a0[j + 1] + a1[j + 1];
          o.z = a0[j + 2] + a1[j + 2];
          o.w = a0[j + 3] + a1[j + 3];
          if (bias) {
            const float4 b = *reinterpret_cast<const float4*>(bias + col0 + j);
            o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
          }
          float4* dst = reinterpret_cast<float4*>(crow + col0 + j);
          if (beta != 0.0f) {
            const float4 q = *dst;
            o.x += beta * q.x; o.y += beta * q.y; o.z += beta * q.z; o.w += beta * q.w;
          }
          *dst = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (col0 + j < N) {
            float o = a0[j] + a1[j];
            if (bias) o += bias[col0 + j];
            if (beta != 0.0f) o += beta * crow[col0 + j];
            crow[col0 + j] = o;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// Epilogue of one row segment: 32 columns of both accumulators -> C.
__device__ __forceinline__ void store32(const float (&a0)[32], const float (&a1)[32], float* crow, int col0, int N,
                                        bool vec, const float* __restrict__ bias, float beta, float s1 = 1.0f,
                                        float rsc = 1.0f) {
  if (vec && col0 + 32 <= N) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      float4 o;
      o.x = __fmaf_rn(s1, a1[j], a0[j]) * rsc;    // s1 = rsc = 1: exactly a0 + a1
      o.y = __fmaf_rn(s1, a1[j + 1], a0[j + 1]) * rsc;
      o.z = __fmaf_rn(s1, a1[j + 2], a0[j + 2]) * rsc;
      o.w = __fmaf_rn(s1, a1[j + 3], a0[j + 3]) * rsc;
      if (bias) {
        const float4 b = *reinterpret_cast<const float4*>(bias + col0 + j);
        o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
      }
      float4* dst = reinterpret_cast<float4*>(crow + col0 + j);
      if (beta != 0.0f) {
        const float4 q = *dst;
        o.x += beta * q.x; o.y += beta * q.y; o.z += beta * q.z; o.w += beta * q.w;
      }
      *dst = o;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < N) {
        float o = __fmaf_rn(s1, a1[j], a0[j]) * rsc;
        if (bias) o += bias[col0 + j];
        if (beta != 0.0f) o += beta * crow[col0 + j];
        crow[col0 + j] = o;
      }
    }
  }
}

// Persistent form: one CTA per SM loops over (split, m tile, n tile) units.
// Warp 0 lane 0 feeds a 4-stage smem ring by TMA, warp 1 lane 0 issues the
// MMAs into one of two TMEM accumulator pairs (512 columns), warps 2-5 drain
// the other pair -- the epilogue of unit j overlaps the main loop of j + 1.
template <int BN, int P = 3>
struct PCfg {
  static constexpr int kBufs = BN == 128 ? 2 : 1;              // accumulator pairs in 512 TMEM columns
  static constexpr int kStageBytes = P * kBM * kBK * 2 + P * BN * kBK * 2;
  static constexpr int kStages = P == 3 ? (BN == 128 ? 4 : 3) : (BN == 128 ? 6 : 4);
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static constexpr int kSmemTS = kSmem + 2 * kBM * 32 * 4;      // + the TMA-store staging
  // D f32; A/B bf16 (P = 3: hi/mid/lo) or fp16 (P = 2: hi, lo * 2^11)
  static constexpr uint32_t kFmt = P == 3 ? 1u : 0u;
  static constexpr uint32_t kIdesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(kBM >> 4) << 24);
};

__device__ __forceinline__ void mma_bf16_id(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// TS: the epilogue leaves through shared memory and TMA stores (two 16 KB
// 128 x 32 fp32 buffers, 128-byte swizzle): the accumulator pair is handed
// back after its last tcgen05.ld and the stores drain asynchronously under the
// next tile's main loop (beta == 0 products; beta == 1 as TMA reduce-add
// stores: C += the tile in L2).
constexpr int kTsBuf = kBM * 32 * 4;                       // one 128 x 32 fp32 chunk
template <int BN, int P = 3, bool TS = false>
__global__ void __launch_bounds__(192, 1)
    k_gemm_split6_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             int M, int N, int K, float* __restrict__ C, int64_t ldc,
                             const float* __restrict__ bias, float beta, int kb_per, int64_t split_stride,
                             int splits, int batch, int64_t c_bstride, const float* __restrict__ rscale = nullptr,
                             const __grid_constant__ CUtensorMap tmC = CUtensorMap{}) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gen = smem_raw + (base - raw);
  using Cfg = PCfg<BN, P>;
  constexpr int kPStages = Cfg::kStages, kSB = Cfg::kStageBytes, kBufs = Cfg::kBufs;
  constexpr int kAP = kBM * kBK * 2, kBP = BN * kBK * 2;       // plane box bytes
  const uint32_t ts0 = base + kPStages * kSB;                  // TS staging (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(gen + kPStages * kSB + (TS ? 2 * kTsBuf : 0));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kPStages + 4);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + kPStages);
  const uint32_t accf0 = su32(bars + 2 * kPStages), acce0 = su32(bars + 2 * kPStages + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (N + BN - 1) / BN, tiles_m = (M + kBM - 1) / kBM;
  const int units = tiles_n * tiles_m * splits * batch;     // z = batch entry * splits + split
  const int kblocks = (K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 4);        // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
        const int kb0 = (z % splits) * kb_per, nkb = min(kblocks - kb0, kb_per), bi = z / splits;
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % kPStages;
          mbar_wait(empty0 + 8 * s, ((it / kPStages) & 1) ^ 1);
          const uint32_t full = full0 + 8 * s;
          mbar_expect_tx(full, kSB);
          const uint32_t st = base + s * kSB;
#pragma unroll
          for (int p = 0; p < P; ++p) {
            tma_load_3d(st + p * kAP, &tmA, full, (kb0 + i) * kBK, tm * kBM, p * batch + bi);
            tma_load_3d(st + P * kAP + p * kBP, &tmB, full, (kb0 + i) * kBK, tn * BN, p * batch + bi);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, j = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
        const int z = u / (tiles_n * tiles_m);
        const int kb0 = (z % splits) * kb_per, nkb = min(kblocks - kb0, kb_per);
        const uint32_t b = j % kBufs, ph = (j / kBufs) & 1;
        mbar_wait(acce0 + 8 * b, ph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc0 = tmem + b * 2 * BN, acc1 = acc0 + BN;
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % kPStages;
          mbar_wait(full0 + 8 * s, (it / kPStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = base + s * kSB;
          constexpr uint32_t id = Cfg::kIdesc;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint32_t off = kk * 32;
            const uint32_t acc = (i | kk) != 0;
            if constexpr (P == 3) {
              const uint64_t ah = smem_desc(st + 0 * kAP + off), am = smem_desc(st + 1 * kAP + off),
                             al = smem_desc(st + 2 * kAP + off);
              const uint64_t bh = smem_desc(st + 3 * kAP + off), bm = smem_desc(st + 3 * kAP + kBP + off),
                             bl = smem_desc(st + 3 * kAP + 2 * kBP + off);
              mma_bf16_id(acc0, ah, bh, id, acc);
              mma_bf16_id(acc1, ah, bm, id, acc);
              mma_bf16_id(acc1, am, bh, id, 1);
              mma_bf16_id(acc1, am, bm, id, 1);
              mma_bf16_id(acc1, ah, bl, id, 1);
              mma_bf16_id(acc1, al, bh, id, 1);
            } else {                         // fp16 hi, lo * 2^11: hi.hi | hi.lo + lo.hi
              const uint64_t ah = smem_desc(st + off), al = smem_desc(st + kAP + off);
              const uint64_t bh = smem_desc(st + 2 * kAP + off), bl = smem_desc(st + 2 * kAP + kBP + off);
              mma_bf16_id(acc0, ah, bh, id, acc);
              mma_bf16_id(acc1, ah, bl, id, acc);
              mma_bf16_id(acc1, al, bh, id, 1);
            }
          }
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(accf0 + 8 * b);
      }
    }
  } else {
    // epilogue warps 2..5: TMEM lane quadrant = warp % 4
    const int q = warp & 3;
    const bool vec = ((ldc & 3) == 0) && aligned16(C);
    constexpr float s1 = P == 3 ? 1.0f : 0x1p-11f;
    uint32_t j = 0, cc = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
      const uint32_t b = j % kBufs;
      mbar_wait(accf0 + 8 * b, (j / kBufs) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int r = q * 32 + lane, row = tm * kBM + r;
      const float rsc = (rscale && row < M) ? rscale[row] : 1.0f;   // A's per-row scale 2^-e
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * 2 * BN;
      float* crow = C + (z % splits) * split_stride + (z / splits) * c_bstride + static_cast<int64_t>(row) * ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32, ++cc) {
        float a0[32], a1[32];
        tmem_ld32(lane_base + c, a0);
        tmem_ld32(lane_base + BN + c, a1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == BN - 32) {
          // last TMEM read of this pair: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce0 + 8 * b) : "memory");
        }
        if constexpr (TS) {
          const int col0 = tn * BN + c;
          if (col0 >= N) continue;                             // uniform: whole chunk past N
          const uint32_t buf = ts0 + (cc & 1) * kTsBuf;
          if (threadIdx.x == 64 && cc >= 2)                    // the store of chunk cc - 2 has read its buffer
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            float4 o;
            o.x = __fmaf_rn(s1, a1[4 * k4], a0[4 * k4]) * rsc;
            o.y = __fmaf_rn(s1, a1[4 * k4 + 1], a0[4 * k4 + 1]) * rsc;
            o.z = __fmaf_rn(s1, a1[4 * k4 + 2], a0[4 * k4 + 2]) * rsc;
            o.w = __fmaf_rn(s1, a1[4 * k4 + 3], a0[4 * k4 + 3]) * rsc;
            if (bias) {
              const int cb = col0 + 4 * k4;
              o.x += cb < N ? bias[cb] : 0.f;
              o.y += cb + 1 < N ? bias[cb + 1] : 0.f;
              o.z += cb + 2 < N ? bias[cb + 2] : 0.f;
              o.w += cb + 3 < N ? bias[cb + 3] : 0.f;
            }
            const uint32_t a = buf + r * 128u + ((k4 ^ (r & 7)) << 4);      // 128-byte swizzle
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w)
                         : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (threadIdx.x == 64) {
            if (beta != 0.0f)                                  // beta == 1: C += the tile (reduce-add in L2)
              asm volatile(
                  "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];"
                  ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(buf), "r"(col0), "r"(tm * kBM), "r"(z)
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                  ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(buf), "r"(col0), "r"(tm * kBM), "r"(z)
                  : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {
          if (row < M) store32(a0, a1, crow, tn * BN + c, N, vec, bias, beta, s1, rsc);
        }
      }
    }
    if (TS && threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// x (rows x cols, leading dimension ld) -> planes [3][rows][cols] bf16 with
// x = hi + mid + lo exactly (round-to-nearest at each step).
__device__ __forceinline__ void split3(float x, __nv_bfloat16& h, __nv_bfloat16& m, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(h);
  m = __float2bfloat16_rn(r);
  l = __float2bfloat16_rn(r - __bfloat162float(m));
}

__device__ __forceinline__ uint32_t pack2(__nv_bfloat16 a, __nv_bfloat16 b) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(a)) | (static_cast<uint32_t>(__bfloat16_as_ushort(b)) << 16);
}

// Eight consecutive values -> 16 bytes in each plane.
__device__ __forceinline__ void split8_store(const float (&v)[8], __nv_bfloat16* __restrict__ out, int64_t plane,
                                             int64_t o) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __nv_bfloat16 h0, m0, l0, h1, m1, l1;
    split3(v[2 * j], h0, m0, l0);
    split3(v[2 * j + 1], h1, m1, l1);
    h[j] = pack2(h0, h1);
    m[j] = pack2(m0, m1);
    l[j] = pack2(l0, l1);
  }
  *reinterpret_cast<uint4*>(out + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(out + plane + o) = make_uint4(m[0], m[1], m[2], m[3]);
  *reinterpret_cast<uint4*>(out + 2 * plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// Contiguous x (ld == cols, rows * cols % 8 == 0): flat, 8 values per thread.
__global__ void k_split3_flat(const float* __restrict__ x, int64_t n, __nv_bfloat16* __restrict__ out,
                              int64_t plane) {
  const int64_t n8 = n >> 3;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = ld_stream(reinterpret_cast<const float4*>(x) + 2 * i);
    const float4 b = ld_stream(reinterpret_cast<const float4*>(x) + 2 * i + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    split8_store(v, out, plane, 8 * i);
  }
}

__global__ void k_split3(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                         __nv_bfloat16* __restrict__ out, int64_t plane) {
  const int64_t n4 = plane >> 2;                          // cols % 4 == 0 (host checks)
  const int64_t c4 = cols >> 2;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / c4, c = (i - r * c4) * 4;
    const float4 v = *reinterpret_cast<const float4*>(x + r * ld + c);
    __nv_bfloat16 h[4], m[4], l[4];
    split3(v.x, h[0], m[0], l[0]);
    split3(v.y, h[1], m[1], l[1]);
    split3(v.z, h[2], m[2], l[2]);
    split3(v.w, h[3], m[3], l[3]);
    const int64_t o = r * cols + c;
    *reinterpret_cast<uint2*>(out + o) = *reinterpret_cast<uint2*>(h);
    *reinterpret_cast<uint2*>(out + plane + o) = *reinterpret_cast<uint2*>(m);
    *reinterpret_cast<uint2*>(out + 2 * plane + o) = *reinterpret_cast<uint2*>(l);
  }
}

// Transposing split: x (rows x cols) -> planes [3][cols][rows] (K-major for
// operands whose reduction dimension is x's row dimension).  64 x 32 tiles
// through shared memory; each thread splits 8 consecutive rows of one column
// and stores 16 bytes per plane (128-byte rows per warp quarter).
__global__ void __launch_bounds__(256) k_split3_t(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                  int64_t ld, __nv_bfloat16* __restrict__ out, int64_t plane,
                                                  int64_t x_bstride = 0, int64_t out_bstride = 0) {
  __shared__ float tile[64][33];
  x += blockIdx.z * x_bstride;                      // batched: one matrix per grid.z
  out += blockIdx.z * out_bstride;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int t = threadIdx.x;
  const bool full = r0 + 64 <= rows && c0 + 32 <= cols;
  if (full && (ld & 3) == 0 && aligned16(x)) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (t >> 3) + 32 * h, c = 4 * (t & 7);
      const float4 v = ld_stream(reinterpret_cast<const float4*>(x + (r0 + r) * ld + c0 + c));
      tile[r][c] = v.x; tile[r][c + 1] = v.y; tile[r][c + 2] = v.z; tile[r][c + 3] = v.w;
    }
  } else {
    for (int i = t; i < 64 * 32; i += 256) {
      const int r = i >> 5, c = i & 31;
      tile[r][c] = (r0 + r < rows && c0 + c < cols) ? x[(r0 + r) * ld + c0 + c] : 0.0f;
    }
  }
  __syncthreads();
  const int c = t >> 3, q = t & 7;                        // output row c0 + c, rows r0 + 8q .. + 7
  const int64_t oc = c0 + c, orow = r0 + 8 * q;
  if (oc >= cols) return;
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = tile[8 * q + j][c];
  const int64_t o = oc * rows + orow;
  if (orow + 8 <= rows && (rows & 7) == 0 && (plane & 7) == 0) {
    split8_store(v, out, plane, o);
  } else {
    for (int j = 0; j < 8 && orow + j < rows; ++j) {
      __nv_bfloat16 h, m, l;
      split3(v[j], h, m, l);
      out[o + j] = h;
      out[plane + o + j] = m;
      out[2 * plane + o + j] = l;
    }
  }
}

// ---- two fp16 planes: x = hi + lo * 2^-11 (hi = RN_f16(x), lo = RN_f16((x - hi) * 2^11);
// x - hi is exact and |x - hi| <= 2^-11 |x|, so lo has hi's range): 22
// significant bits for 2^-14 <= |x| < 65504, absolute error <= 2^-35 below.
// The product keeps hi.hi + 2^-11 (hi.lo + lo.hi) (f16x3: three MMAs).
constexpr float kLoScale = 2048.0f;

__device__ __forceinline__ void split8_store_h(const float (&v)[8], __half* __restrict__ out, int64_t plane, int64_t o) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split_pair2h(v[2 * j], v[2 * j + 1], h[j], l[j]);
  *reinterpret_cast<uint4*>(out + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(out + plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

__global__ void k_split2h_flat(const float* __restrict__ x, int64_t n, __half* __restrict__ out, int64_t plane) {
  const int64_t n8 = n >> 3;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = ld_stream(reinterpret_cast<const float4*>(x) + 2 * i);
    const float4 b = ld_stream(reinterpret_cast<const float4*>(x) + 2 * i + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    split8_store_h(v, out, plane, 8 * i);
  }
}

__global__ void k_split2h(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                          __half* __restrict__ out, int64_t plane) {
  const int64_t c4 = cols >> 2, n4 = rows * c4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / c4, c = (i - r * c4) * 4;
    const float4 v = *reinterpret_cast<const float4*>(x + r * ld + c);
    uint32_t h0, l0, h1, l1;
    split_pair2h(v.x, v.y, h0, l0);
    split_pair2h(v.z, v.w, h1, l1);
    const int64_t o = r * cols + c;
    *reinterpret_cast<uint2*>(out + o) = make_uint2(h0, h1);
    *reinterpret_cast<uint2*>(out + plane + o) = make_uint2(l0, l1);
  }
}

// transposing form (as k_split3_t): x (rows x cols) -> planes [2][cols][rows]
__global__ void __launch_bounds__(256) k_split2h_t(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                   int64_t ld, __half* __restrict__ out, int64_t plane) {
  __shared__ float tile[64][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int t = threadIdx.x;
  for (int i = t; i < 64 * 32; i += 256) {
    const int r = i >> 5, c = i & 31;
    tile[r][c] = (r0 + r < rows && c0 + c < cols) ? x[(r0 + r) * ld + c0 + c] : 0.0f;
  }
  __syncthreads();
  const int c = t >> 3, q = t & 7;
  const int64_t oc = c0 + c, orow = r0 + 8 * q;
  if (oc >= cols) return;
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = tile[8 * q + j][c];
  const int64_t o = oc * rows + orow;
  if (orow + 8 <= rows && (rows & 7) == 0 && (plane & 7) == 0) {
    split8_store_h(v, out, plane, o);
  } else {
    for (int j = 0; j < 8 && orow + j < rows; ++j) planes_store1h(v[j], out, plane, o + j);
  }
}

// Row-scaled form for operands that span fp16's range (gradients): row r is
// split as x * 2^e_r with e_r = 14 - floor(log2 max|x_r|) (the row maximum
// lands in [2^14, 2^15)), and rscale[r] = 2^-e_r multiplies the product's
// row in the GEMM epilogue (exact: powers of two).  One CTA per row: the
// row's maximum, then its split (the second read hits L1).
constexpr int kRowT = 256;
__global__ void __launch_bounds__(kRowT) k_split2h_rows(const float* __restrict__ x, int64_t cols, int64_t ld,
                                                        __half* __restrict__ out, int64_t plane,
                                                        float* __restrict__ rscale) {
  const int64_t r = blockIdx.x;
  const float* row = x + r * ld;
  const int64_t c4 = cols >> 2;
  float m = 0.0f;
  for (int64_t i = threadIdx.x; i < c4; i += kRowT) {
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * i);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  __shared__ float sm[kRowT / 32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  m = sm[0];
#pragma unroll
  for (int w = 1; w < kRowT / 32; ++w) m = fmaxf(m, sm[w]);
  int e;
  const float sc = row_scale_exp(m, e);
  if (threadIdx.x == 0) rscale[r] = __int_as_float((127 - e) << 23);
  for (int64_t i = threadIdx.x; i < c4; i += kRowT) {
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * i);
    planes_store4h(make_float4(v.x * sc, v.y * sc, v.z * sc, v.w * sc), out, plane, r * cols + 4 * i);
  }
}

// Same persistent GEMM with the A operand read as fp32 (row-major, K
// contiguous) and split into its bf16 planes inside the kernel: warps 6-9
// convert each TMA-loaded 128x32 fp32 tile into the three 64-byte-swizzled
// bf16 planes the MMAs read (no separate split pass over A: 4 bytes per
// element read instead of 4 + 6 written + 6 read).  BN = 128, 3 stages of
// (fp32 A 16 KB + A planes 24 KB + B planes 24 KB).
constexpr int kCStages = 3;                                // plane stages (A + B planes)
#ifndef SF_A32_FSTAGES
#define SF_A32_FSTAGES 4
#endif
constexpr int kCFStages = SF_A32_FSTAGES;                  // fp32 A stages (run ahead of the planes)
constexpr int kCF32 = kBM * kBK * 4;                       // fp32 A tile
constexpr int kCStage = 6 * kPlaneBytes;
constexpr int kCSmem = kCFStages * kCF32 + kCStages * kCStage + 1024 + 512;

#ifndef SF_A32_CONV_WARPS
#define SF_A32_CONV_WARPS 8
#endif
constexpr int kConvWarps = SF_A32_CONV_WARPS;              // warps 6 .. 5 + kConvWarps
constexpr int kCRows = kBM / kConvWarps;                   // tile rows per converter warp
constexpr int kFWarp = 6 + kConvWarps;                     // fp32 A producer warp
constexpr int kCThreads = 32 * (kFWarp + 1);

// exact 3-term split of two floats with packed conversions
__device__ __forceinline__ void split3x2(float x0, float x1, uint32_t& h, uint32_t& m, uint32_t& l) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
  float r0 = x0 - __uint_as_float(h << 16), r1 = x1 - __uint_as_float(h & 0xFFFF0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(m) : "f"(r1), "f"(r0));
  r0 -= __uint_as_float(m << 16);
  r1 -= __uint_as_float(m & 0xFFFF0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(r1), "f"(r0));
}

// byte offset of bf16 element (row, k) in a 128 x 32 plane with the 64-byte
// swizzle (16-byte chunk index XOR row bits 1-2)
__device__ __forceinline__ uint32_t sw64_off(int row, int k) {
  const int chunk = (k >> 3) ^ ((row >> 1) & 3);
  return static_cast<uint32_t>(row * 64 + chunk * 16 + (k & 7) * 2);
}

__global__ void __launch_bounds__(kCThreads, 1)
    k_gemm_split6_a32(const __grid_constant__ CUtensorMap tmA32, const __grid_constant__ CUtensorMap tmB, int M,
                      int N, int K, float* __restrict__ C, int64_t ldc, const float* __restrict__ bias, float beta,
                      int kb_per, int64_t split_stride, int splits) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gen = smem_raw + (base - raw);
  // [fp32 A ring][plane ring][barriers]
  const uint32_t pbase = base + kCFStages * kCF32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gen + kCFStages * kCF32 + kCStages * kCStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kCStages + 2 * kCFStages + 4);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + kCStages);
  const uint32_t fullf0 = su32(bars + 2 * kCStages), emptyf0 = su32(bars + 2 * kCStages + kCFStages);
  const uint32_t accf0 = su32(bars + 2 * kCStages + 2 * kCFStages), acce0 = accf0 + 16;
  constexpr int BN = kBN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (N + BN - 1) / BN, tiles_m = (M + kBM - 1) / kBM;
  const int units = tiles_n * tiles_m * splits;
  const int kblocks = (K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kCStages; ++s) {
      mbar_init(full0 + 8 * s, 1 + kConvWarps);   // B planes (TMA) + the converter warps
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int s = 0; s < kCFStages; ++s) {
      mbar_init(fullf0 + 8 * s, 1);
      mbar_init(emptyf0 + 8 * s, kConvWarps);     // converter warps done reading
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA32)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == kFWarp) {
    // warp 0: B planes into the plane ring; the last warp: fp32 A tiles into their own ring
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
        const int kb0 = z * kb_per, nkb = min(kblocks - kb0, kb_per);
        for (int i = 0; i < nkb; ++i, ++it) {
          if (warp == kFWarp) {
            const uint32_t sf = it % kCFStages;
            mbar_wait(emptyf0 + 8 * sf, ((it / kCFStages) & 1) ^ 1);
            mbar_expect_tx(fullf0 + 8 * sf, kCF32);
            tma_load_2d(base + sf * kCF32, &tmA32, fullf0 + 8 * sf, (kb0 + i) * kBK, tm * kBM);
          } else {
            const uint32_t s = it % kCStages;
            mbar_wait(empty0 + 8 * s, ((it / kCStages) & 1) ^ 1);
            mbar_expect_tx(full0 + 8 * s, 3 * kPlaneBytes);
            const uint32_t st = pbase + s * kCStage;
#pragma unroll
            for (int p = 0; p < 3; ++p)
              tma_load_2d(st + (3 + p) * kPlaneBytes, &tmB, full0 + 8 * s, (kb0 + i) * kBK, p * N + tn * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t it = 0, j = 0;
      constexpr uint32_t id = kIdesc;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
        const int z = u / (tiles_n * tiles_m);
        const int kb0 = z * kb_per, nkb = min(kblocks - kb0, kb_per);
        const uint32_t b = j & 1, ph = (j >> 1) & 1;
        mbar_wait(acce0 + 8 * b, ph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc0 = tmem + b * 2 * BN, acc1 = acc0 + BN;
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % kCStages;
          mbar_wait(full0 + 8 * s, (it / kCStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = pbase + s * kCStage;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t ah = smem_desc(st + 0 * kPlaneBytes + off), am = smem_desc(st + 1 * kPlaneBytes + off),
                           al = smem_desc(st + 2 * kPlaneBytes + off);
            const uint64_t bh = smem_desc(st + 3 * kPlaneBytes + off), bm = smem_desc(st + 4 * kPlaneBytes + off),
                           bl = smem_desc(st + 5 * kPlaneBytes + off);
            const uint32_t acc = (i | kk) != 0;
            mma_bf16_id(acc0, ah, bh, id, acc);
            mma_bf16_id(acc1, ah, bm, id, acc);
            mma_bf16_id(acc1, am, bh, id, 1);
            mma_bf16_id(acc1, am, bm, id, 1);
            mma_bf16_id(acc1, ah, bl, id, 1);
            mma_bf16_id(acc1, al, bh, id, 1);
          }
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(accf0 + 8 * b);
      }
    }
  } else if (warp >= 6) {
    // converters: lane -> (row (lane >> 3) + 4 i, float4 chunk lane & 7); warp w covers kCRows rows
    const int cw = warp - 6;
    const int c = lane & 7;
    uint32_t it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int z = u / (tiles_n * tiles_m);
      const int kb0 = z * kb_per, nkb = min(kblocks - kb0, kb_per);
      for (int i = 0; i < nkb; ++i, ++it) {
        const uint32_t sf = it % kCFStages, s = it % kCStages;
        mbar_wait(fullf0 + 8 * sf, (it / kCFStages) & 1);
        const uint8_t* f32 = gen + sf * kCF32;
        float4 v[kCRows / 4];
#pragma unroll
        for (int r8 = 0; r8 < kCRows / 4; ++r8)
          v[r8] = *reinterpret_cast<const float4*>(f32 + (cw * kCRows + r8 * 4 + (lane >> 3)) * 128 + c * 16);
        // order these generic-proxy reads before the next TMA (async-proxy) write of the stage
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(emptyf0 + 8 * sf) : "memory");
        mbar_wait(empty0 + 8 * s, ((it / kCStages) & 1) ^ 1);   // the MMAs are done with these planes
        uint8_t* pl = gen + kCFStages * kCF32 + s * kCStage;
#pragma unroll
        for (int r8 = 0; r8 < kCRows / 4; ++r8) {
          const int row = cw * kCRows + r8 * 4 + (lane >> 3);
          uint32_t h0, m0, l0, h1, m1, l1;
#ifdef SF_A32_SCALAR
          {
            __nv_bfloat16 h[4], m[4], l[4];
            split3(v[r8].x, h[0], m[0], l[0]);
            split3(v[r8].y, h[1], m[1], l[1]);
            split3(v[r8].z, h[2], m[2], l[2]);
            split3(v[r8].w, h[3], m[3], l[3]);
            h0 = pack2(h[0], h[1]); h1 = pack2(h[2], h[3]);
            m0 = pack2(m[0], m[1]); m1 = pack2(m[2], m[3]);
            l0 = pack2(l[0], l[1]); l1 = pack2(l[2], l[3]);
          }
#else
          split3x2(v[r8].x, v[r8].y, h0, m0, l0);
          split3x2(v[r8].z, v[r8].w, h1, m1, l1);
#endif
          const uint32_t o = sw64_off(row, 4 * c);
          *reinterpret_cast<uint2*>(pl + o) = make_uint2(h0, h1);
          *reinterpret_cast<uint2*>(pl + kPlaneBytes + o) = make_uint2(m0, m1);
          *reinterpret_cast<uint2*>(pl + 2 * kPlaneBytes + o) = make_uint2(l0, l1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * s) : "memory");
      }
    }
  } else {
    // epilogue warps 2..5
    const int q = warp & 3;
    const bool vec = ((ldc & 3) == 0) && aligned16(C);
    uint32_t j = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++j) {
      const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
      const uint32_t b = j & 1;
      mbar_wait(accf0 + 8 * b, (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = tm * kBM + q * 32 + lane;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * 2 * BN;
      float* crow = C + z * split_stride + static_cast<int64_t>(row) * ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float a0[32], a1[32];
        tmem_ld32(lane_base + c, a0);
        tmem_ld32(lane_base + BN + c, a1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == BN - 32) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce0 + 8 * b) : "memory");
        }
        if (row < M) store32(a0, a1, crow, tn * BN + c, N, vec, bias, beta);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Split-K finish: C = sum_z partial[z] (fixed order) + bias + beta * C.
__global__ void k_splitk_reduce(const float* __restrict__ ws, int splits, int64_t M, int64_t N,
                                float* __restrict__ C, int64_t ldc, const float* __restrict__ bias, float beta) {
  const int64_t n4 = N >> 2, total = M * n4, plane = M * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / n4, c = (i - r * n4) * 4;
    float4 o = *reinterpret_cast<const float4*>(ws + r * N + c);
    for (int z = 1; z < splits; ++z) {
      const float4 q = *reinterpret_cast<const float4*>(ws + z * plane + r * N + c);
      o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
    }
    if (bias) {
      const float4 b = *reinterpret_cast<const float4*>(bias + c);
      o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
    }
    float4* dst = reinterpret_cast<float4*>(C + r * ldc + c);
    if (beta != 0.0f) {
      const float4 q = *dst;
      o.x += beta * q.x; o.y += beta * q.y; o.z += beta * q.z; o.w += beta * q.w;
    }
    *dst = o;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// planes [3][rows][k] bf16 as one (3 rows) x k matrix; box 128 rows x 32.
bool make_map(CUtensorMap* map, const void* planes, int64_t rows, int64_t k, uint32_t box_rows = kBM) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(3 * rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
  cuuint32_t box[2] = {kBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(planes), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_tc_stages = 0;    // 0/1: persistent kernel, N = 128 / 256 tiles; 2..4: one tile per CTA, that many stages

// planes [3][batch][rows][k] bf16 as a (3 batch) x rows x k tensor; box box_rows x 32 x 1
// (rows past `rows` are zero-filled, never another plane's or entry's rows).
bool make_map3(CUtensorMap* map, const void* planes, int64_t rows, int64_t k, int64_t batch, uint32_t box_rows,
               int nplanes = 3) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(nplanes * batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(k) * 2, static_cast<cuuint64_t>(rows * k) * 2};
  cuuint32_t box[3] = {kBK, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(planes), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 row-major A (rows x k, leading dimension ld): box 128 rows x 32, no swizzle.
bool make_map_f32(CUtensorMap* map, const float* a, int64_t rows, int64_t k, int64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {kBK, kBM};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- CTA-pair (cta_group::2) form of the f16x3 product (opt-in, see
// g_gemm_pair): 256 x 256 tiles,
// each CTA of a 2-CTA cluster stages its 128 rows of A and its 128-column
// half of B (32 KB per K block instead of 48 KB), the leader issues
// tcgen05.mma.cta_group::2 (M = 256): each SM reads half of the B operand,
// which lifts the shared-memory bound of the N = 256 single-CTA tile.  Both
// CTAs' TMA loads complete on the leader's stage barrier; the leader's
// commits free the stage in both CTAs and signal both epilogues; both
// epilogues hand the accumulators back on the leader's barrier.  Each SM
// drains its own 128 x 256 accumulators through the TMA-store epilogue.
// PBN = 256: one accumulator pair per SM (512 TMEM columns); PBN = 128: two
// pairs, the epilogue of tile j overlapping the main loop of tile j + 1.
template <int PBN>
struct PairCfg {
  static constexpr int kHalfB = PBN / 2;                                 // B rows staged per CTA
  static constexpr int kStageBytes = 2 * kBM * kBK * 2 + 2 * kHalfB * kBK * 2;
  static constexpr int kStages = PBN == 256 ? 6 : 8;
  static constexpr int kBufs = PBN == 256 ? 1 : 2;
  static constexpr int kSmem = kStages * kStageBytes + 2 * kTsBuf + 1024 + 256;
};

__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_to(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"(static_cast<uint16_t>(3))
               : "memory");
}

template <int PBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_gemm_f16x3_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, int M, int N, int K, float beta, int kb_per,
                      int splits, const float* __restrict__ bias, const float* __restrict__ rscale) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gen = smem_raw + (base - raw);
  using Cfg = PairCfg<PBN>;
  constexpr int kPairStages = Cfg::kStages, kPairStageBytes = Cfg::kStageBytes, kHalfB = Cfg::kHalfB;
  constexpr int kBufs = Cfg::kBufs;
  constexpr int kAP = kBM * kBK * 2, kBP = kHalfB * kBK * 2;    // plane boxes: A 128 rows, B half
  const uint32_t ts0 = base + kPairStages * kPairStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gen + kPairStages * kPairStageBytes + 2 * kTsBuf);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kPairStages + 4);
  const uint32_t full0 = su32(bars), empty0 = su32(bars + kPairStages);
  const uint32_t accf0 = su32(bars + 2 * kPairStages), acce0 = accf0 + 16;
  const uint32_t rank = cta_rank_in_cluster();
  const bool leader = rank == 0;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_n = (N + PBN - 1) / PBN, tiles_m = (M + 255) / 256;
  const int units = tiles_n * tiles_m * splits;
  const int kblocks = (K + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(full0 + 8 * s, 1);                       // leader: its expect_tx arrival (+ both CTAs' bytes)
      mbar_init(empty0 + 8 * s, 1);                      // the leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 8);                       // leader: 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();                                    // both CTAs' barriers exist before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_l = mapa_to(full0, 0), acce_l0 = mapa_to(acce0, 0);

  if (warp == 0) {
    if (lane == 0) {                                     // TMA producer (both CTAs): own A rows, own B half
      uint32_t it = 0;
      for (int u = cl; u < units; u += ncl) {
        const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
        const int kb0 = z * kb_per, nkb = min(kblocks - kb0, kb_per);
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % kPairStages;
          mbar_wait(empty0 + 8 * s, ((it / kPairStages) & 1) ^ 1);
          const uint32_t fullr = full_l + 8 * s;
          if (leader) mbar_expect_tx(full0 + 8 * s, 2 * kPairStageBytes);
          const uint32_t st = base + s * kPairStageBytes;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            tma_load_3d_pair(st + p * kAP, &tmA, fullr, (kb0 + i) * kBK, tm * 256 + 128 * rank, p);
            tma_load_3d_pair(st + 2 * kAP + p * kBP, &tmB, fullr, (kb0 + i) * kBK, tn * PBN + kHalfB * rank, p);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {                           // MMA issuer: the leader only
      constexpr uint32_t id = (1u << 4) | ((static_cast<uint32_t>(PBN) >> 3) << 17) | ((256u >> 4) << 24);   // M 256
      uint32_t it = 0, j = 0;
      for (int u = cl; u < units; u += ncl, ++j) {
        const int z = u / (tiles_n * tiles_m);
        const int kb0 = z * kb_per, nkb = min(kblocks - kb0, kb_per);
        const uint32_t b = j % kBufs;
        mbar_wait(acce0 + 8 * b, ((j / kBufs) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc0 = tmem + b * 2 * PBN, acc1 = acc0 + PBN;
        for (int i = 0; i < nkb; ++i, ++it) {
          const uint32_t s = it % kPairStages;
          mbar_wait(full0 + 8 * s, (it / kPairStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = base + s * kPairStageBytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint32_t off = kk * 32;
            const uint32_t acc = (i | kk) != 0;
            const uint64_t ah = smem_desc(st + off), al = smem_desc(st + kAP + off);
            const uint64_t bh = smem_desc(st + 2 * kAP + off), bl = smem_desc(st + 2 * kAP + kBP + off);
            umma_pair(acc0, ah, bh, id, acc);
            umma_pair(acc1, ah, bl, id, acc);
            umma_pair(acc1, al, bh, id, 1);
          }
          commit_pair(empty0 + 8 * s);                   // frees stage s in both CTAs
        }
        commit_pair(accf0 + 8 * b);                      // both epilogues may drain
      }
    }
  } else {
    // epilogue warps 2..5 of each CTA: its 128 rows (TMEM lanes) x 256 columns
    const int q = warp & 3;
    uint32_t j = 0, cc = 0;
    for (int u = cl; u < units; u += ncl, ++j) {
      const int tn = u % tiles_n, tm = (u / tiles_n) % tiles_m, z = u / (tiles_n * tiles_m);
      const uint32_t b = j % kBufs;
      mbar_wait(accf0 + 8 * b, (j / kBufs) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int r = q * 32 + lane, row0 = tm * 256 + 128 * static_cast<int>(rank), row = row0 + r;
      const float rsc = (rscale && row < M) ? rscale[row] : 1.0f;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * 2 * PBN;
#pragma unroll 1
      for (int c = 0; c < PBN; c += 32, ++cc) {
        float a0[32], a1[32];
        tmem_ld32(lane_base + c, a0);
        tmem_ld32(lane_base + PBN + c, a1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == PBN - 32) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acce_l0 + 8 * b) : "memory");
        }
        const int col0 = tn * PBN + c;
        if (col0 >= N) continue;
        const uint32_t buf = ts0 + (cc & 1) * kTsBuf;
        if (threadIdx.x == 64 && cc >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          float4 o;
          o.x = __fmaf_rn(0x1p-11f, a1[4 * k4], a0[4 * k4]) * rsc;
          o.y = __fmaf_rn(0x1p-11f, a1[4 * k4 + 1], a0[4 * k4 + 1]) * rsc;
          o.z = __fmaf_rn(0x1p-11f, a1[4 * k4 + 2], a0[4 * k4 + 2]) * rsc;
          o.w = __fmaf_rn(0x1p-11f, a1[4 * k4 + 3], a0[4 * k4 + 3]) * rsc;
          if (bias) {
            const int cb = col0 + 4 * k4;
            o.x += cb < N ? bias[cb] : 0.f;
            o.y += cb + 1 < N ? bias[cb + 1] : 0.f;
            o.z += cb + 2 < N ? bias[cb + 2] : 0.f;
            o.w += cb + 3 < N ? bias[cb + 3] : 0.f;
          }
          const uint32_t a = buf + r * 128u + ((k4 ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w)
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          if (beta != 0.0f)
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];"
                ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(buf), "r"(col0), "r"(row0), "r"(z)
                : "memory");
          else
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                ::"l"(reinterpret_cast<uint64_t>(&tmC)), "r"(buf), "r"(col0), "r"(row0), "r"(z)
                : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();                                    // the peer no longer reads this CTA's smem / barriers
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// fp32 C (M x N, leading dimension ldc) x `splits` partials sstride apart as
// a 3-D tensor for the TMA-store epilogue: box 32 columns x 128 rows,
// 128-byte swizzle; rows / columns past M / N are clipped by the map.
bool make_map_c(CUtensorMap* map, float* c, int64_t M, int64_t N, int64_t ldc, int64_t splits, int64_t sstride) {
  auto fn = encode_fn();
  if (!fn || (ldc & 3) || (splits > 1 && (sstride & 3)) || !aligned16(c)) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(splits)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldc) * 4,
                           static_cast<cuuint64_t>(splits > 1 ? sstride : M * ldc) * 4};
  cuuint32_t box[3] = {32, kBM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool g_tma_store = true;   // sf_gemm_set_tma_store
// sf_gemm_set_pair: f16x3 products on CTA pairs, 256 x 128 (1) or 256 x 256 (2)
// tiles.  Off by default: measured no faster than the single-CTA 128 x 256
// tile with the TMA-store epilogue at every step shape (the single-CTA form is
// not shared-memory bound; `profiles/r02_kernel_bench_v9_pair.txt`).
bool g_gemm_pair = false;
int g_pair_bn = 128;

}  // namespace
}  // namespace sf

extern "C" {

int sf_gemm_set_tma_store(int on) {
  sf::g_tma_store = on != 0;
  return SF_OK;
}

int sf_gemm_set_pair(int on) {
  if (on < 0 || on > 2) return SF_EINVAL;
  sf::g_gemm_pair = on != 0;
  sf::g_pair_bn = on == 2 ? 256 : 128;
  return SF_OK;
}

int sf_gemm_split6_set_stages(int stages) {
  if (stages < 0 || stages > 4) return SF_EINVAL;
  sf::g_tc_stages = stages;
  return SF_OK;
}

int sf_split3_bf16_ex(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                      int64_t plane_stride, void* stream) {
  using namespace sf;
  if (rows < 0 || cols < 0 || ld < cols || (rows * cols > 0 && (!x || !planes)) || plane_stride < rows * cols)
    return SF_EINVAL;
  if (rows * cols == 0) return SF_OK;
  auto* out = static_cast<__nv_bfloat16*>(planes);
  const bool p16 = aligned16(planes) && (plane_stride & 7) == 0;
  if (!transpose) {
    if ((cols & 3) || (ld & 3) || !aligned16(x) || (reinterpret_cast<uintptr_t>(planes) & 7) || (plane_stride & 3))
      return SF_EINVAL;
    if (ld == cols && ((rows * cols) & 7) == 0 && p16)
      k_split3_flat<<<grid_for(rows * cols / 8, 256, 4), 256, 0, as_stream(stream)>>>(x, rows * cols, out,
                                                                                       plane_stride);
    else
      k_split3<<<grid_for(rows * cols / 4, 256), 256, 0, as_stream(stream)>>>(x, rows, cols, ld, out, plane_stride);
  } else {
    if (!aligned16(planes)) return SF_EINVAL;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 63) / 64));
    if (grid.y > 65535u) return SF_EINVAL;
    k_split3_t<<<grid, 256, 0, as_stream(stream)>>>(x, rows, cols, ld, out, plane_stride);
  }
  return check_launch();
}

int sf_split3_bf16(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                   void* stream) {
  return sf_split3_bf16_ex(x, rows, cols, ld, transpose, planes, rows * cols, stream);
}

int sf_split2_f16_ex(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                     int64_t plane_stride, void* stream) {
  using namespace sf;
  if (rows < 0 || cols < 0 || ld < cols || (rows * cols > 0 && (!x || !planes)) || plane_stride < rows * cols)
    return SF_EINVAL;
  if (rows * cols == 0) return SF_OK;
  auto* out = static_cast<__half*>(planes);
  if (!transpose) {
    if ((cols & 3) || (ld & 3) || !aligned16(x) || (reinterpret_cast<uintptr_t>(planes) & 7) || (plane_stride & 3))
      return SF_EINVAL;
    if (ld == cols && ((rows * cols) & 7) == 0 && aligned16(planes) && (plane_stride & 7) == 0)
      k_split2h_flat<<<grid_for(rows * cols / 8, 256, 4), 256, 0, as_stream(stream)>>>(x, rows * cols, out,
                                                                                        plane_stride);
    else
      k_split2h<<<grid_for(rows * cols / 4, 256), 256, 0, as_stream(stream)>>>(x, rows, cols, ld, out, plane_stride);
  } else {
    if (!aligned16(planes)) return SF_EINVAL;
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 63) / 64));
    if (grid.y > 65535u) return SF_EINVAL;
    k_split2h_t<<<grid, 256, 0, as_stream(stream)>>>(x, rows, cols, ld, out, plane_stride);
  }
  return check_launch();
}

int sf_split2_f16(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                  void* stream) {
  return sf_split2_f16_ex(x, rows, cols, ld, transpose, planes, rows * cols, stream);
}

int sf_split2_f16_rows(const float* x, int64_t rows, int64_t cols, int64_t ld, void* planes, float* row_scale,
                       void* stream) {
  using namespace sf;
  if (rows < 0 || cols < 0 || ld < cols || (rows * cols > 0 && (!x || !planes || !row_scale))) return SF_EINVAL;
  if (rows * cols == 0) return SF_OK;
  if ((cols & 3) || (ld & 3) || !aligned16(x) || (reinterpret_cast<uintptr_t>(planes) & 7) || rows > INT32_MAX)
    return SF_EINVAL;
  k_split2h_rows<<<static_cast<unsigned>(rows), kRowT, 0, as_stream(stream)>>>(
      x, cols, ld, static_cast<__half*>(planes), rows * cols, row_scale);
  return check_launch();
}

int64_t sf_gemm_split6_splits(int64_t m, int64_t n, int64_t k) {
  using namespace sf;
  const int64_t kblocks = (k + kBK - 1) / kBK;
  const int64_t tiles = ((m + kBM - 1) / kBM) * ((n + kBN - 1) / kBN);
  // accuracy: the tensor core truncates while accumulating, so the error
  // grows linearly in the K run of one accumulator -> at most kMaxRun K per
  // partial: up to K = 3072 one run (<= 1.5x strict SGEMM's error, no
  // partial traffic for the forward / input-gradient products), longer
  // reductions (weight gradients over B*T tokens) in runs of <= 1024;
  // occupancy: ~2 CTAs per SM when the tile grid is small, partials no
  // shorter than kMinRun
  constexpr int64_t kOneRun = 3072 / kBK, kMaxRun = 1024 / kBK, kMinRun = 512 / kBK;
  int64_t splits = kblocks <= kOneRun ? 1 : (kblocks + kMaxRun - 1) / kMaxRun;
  const int64_t want = (2 * static_cast<int64_t>(num_sms()) + tiles - 1) / tiles;
  const int64_t cap = kblocks / kMinRun > 1 ? kblocks / kMinRun : 1;
  const int64_t occ = want < cap ? want : cap;
  if (occ > splits) splits = occ;
  if (splits > 32) splits = 32;
  const int64_t per = (kblocks + splits - 1) / splits;
  return (kblocks + per - 1) / per;                  // no empty partials
}

int64_t sf_gemm_split6_ws_bytes(int64_t m, int64_t n, int64_t k) {
  const int64_t s = sf_gemm_split6_splits(m, n, k);
  return s > 1 ? s * m * n * 4 : 0;
}

int sf_gemm_split6(int64_t m, int64_t n, int64_t k, const void* a_planes, const void* b_planes, float* c,
                   int64_t ldc, const float* bias, float beta, void* ws, int64_t ws_bytes, void* stream) {
  using namespace sf;
  if (m < 0 || n < 0 || k < 0 || ldc < n) return SF_EINVAL;
  if (m == 0 || n == 0) return SF_OK;
  if (!a_planes || !b_planes || !c || k == 0 || (k & 7) || 3 * m > INT32_MAX || 3 * n > INT32_MAX ||
      !aligned16(a_planes) || !aligned16(b_planes))
    return SF_EINVAL;
  CUtensorMap ta, tb;
  if (!make_map(&ta, a_planes, m, k) || !make_map(&tb, b_planes, n, k)) return SF_EUNAVAILABLE;
  dim3 grid(static_cast<unsigned>((n + kBN - 1) / kBN), static_cast<unsigned>((m + kBM - 1) / kBM));
  if (grid.y > 65535u) return SF_EINVAL;
  const int64_t splits = sf_gemm_split6_splits(m, n, k);
  const int kb_per = static_cast<int>(((k + kBK - 1) / kBK + splits - 1) / splits);
  float* out = c;
  int64_t ldo = ldc, sstride = 0;
  const float* ob = bias;
  float obeta = beta;
  if (splits > 1) {
    if (!ws || ws_bytes < splits * m * n * 4 || !aligned16(ws) || (n & 3) || (ldc & 3) || !aligned16(c))
      return SF_EINVAL;
    out = static_cast<float*>(ws);
    ldo = n;
    sstride = m * n;
    ob = nullptr;
    obeta = 0.0f;
  }
  grid.z = static_cast<unsigned>(splits);
  static unsigned long long optin2 = 0, optin3 = 0, optin4 = 0, optinp = 0, optinw = 0;
  const int mi = static_cast<int>(m), ni = static_cast<int>(n), ki = static_cast<int>(k);
  switch (g_tc_stages) {
    case 0:
    case 1: {
      // persistent: N = 128 tiles with two accumulator pairs (epilogue
      // overlapped) or N = 256 tiles with one (half the A-operand smem reads)
      // auto (0): N = 256 when one unit's K run is long enough (>= 2048) to
      // amortise its un-overlapped epilogue (measured, tools/tc_gemm_probe.py)
      const bool wide = g_tc_stages == 1 || (g_tc_stages == 0 && static_cast<int64_t>(kb_per) * kBK >= 2048 && n >= 256);
      const int64_t tn = wide ? (n + 255) / 256 : grid.x;
      const int64_t units = tn * grid.y * splits;
      const unsigned ctas = static_cast<unsigned>(units < num_sms() ? units : num_sms());
      CUtensorMap ta3, tb3;
      if (!make_map3(&ta3, a_planes, m, k, 1, kBM) || !make_map3(&tb3, b_planes, n, k, 1, wide ? 256 : kBN))
        return SF_EUNAVAILABLE;
      if (wide) {
        smem_optin(k_gemm_split6_persistent<256>, PCfg<256>::kSmem, optinw);
        k_gemm_split6_persistent<256><<<ctas, 192, PCfg<256>::kSmem, as_stream(stream)>>>(
            ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0);
      } else {
        CUtensorMap tc3;
        if (g_tma_store && (obeta == 0.0f || obeta == 1.0f) && make_map_c(&tc3, out, m, n, ldo, splits, sstride)) {
          static unsigned long long optints = 0;
          smem_optin(k_gemm_split6_persistent<128, 3, true>, PCfg<128, 3>::kSmemTS, optints);
          k_gemm_split6_persistent<128, 3, true><<<ctas, 192, PCfg<128, 3>::kSmemTS, as_stream(stream)>>>(
              ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0, nullptr,
              tc3);
        } else {
          smem_optin(k_gemm_split6_persistent<128>, PCfg<128>::kSmem, optinp);
          k_gemm_split6_persistent<128><<<ctas, 192, PCfg<128>::kSmem, as_stream(stream)>>>(
              ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0);
        }
      }
      break;
    }
    case 2:
      smem_optin(k_gemm_split6<2>, smem_bytes(2), optin2);
      k_gemm_split6<2><<<grid, 128, smem_bytes(2), as_stream(stream)>>>(ta, tb, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride);
      break;
    case 4:
      smem_optin(k_gemm_split6<4>, smem_bytes(4), optin4);
      k_gemm_split6<4><<<grid, 128, smem_bytes(4), as_stream(stream)>>>(ta, tb, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride);
      break;
    default:
      smem_optin(k_gemm_split6<3>, smem_bytes(3), optin3);
      k_gemm_split6<3><<<grid, 128, smem_bytes(3), as_stream(stream)>>>(ta, tb, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride);
  }
  if (splits > 1) {
    const int rc = check_launch();
    if (rc != SF_OK) return rc;
    k_splitk_reduce<<<grid_for(m * n / 4, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const float*>(ws), static_cast<int>(splits), m, n, c, ldc, bias, beta);
  }
  return check_launch();
}

int sf_gemm_f16x3(int64_t m, int64_t n, int64_t k, const void* a_planes, const float* a_row_scale,
                  const void* b_planes, float* c, int64_t ldc, const float* bias, float beta, void* ws,
                  int64_t ws_bytes, void* stream) {
  using namespace sf;
  if (m < 0 || n < 0 || k < 0 || ldc < n) return SF_EINVAL;
  if (m == 0 || n == 0) return SF_OK;
  if (!a_planes || !b_planes || !c || k == 0 || (k & 7) || 2 * m > INT32_MAX || 2 * n > INT32_MAX ||
      !aligned16(a_planes) || !aligned16(b_planes))
    return SF_EINVAL;
  const int64_t tiles_m = (m + kBM - 1) / kBM;
  if (tiles_m > 65535) return SF_EINVAL;
  const int64_t splits = sf_gemm_split6_splits(m, n, k);
  const int kb_per = static_cast<int>(((k + kBK - 1) / kBK + splits - 1) / splits);
  float* out = c;
  int64_t ldo = ldc, sstride = 0;
  const float* ob = bias;
  float obeta = beta;
  if (splits > 1) {
    if (!ws || ws_bytes < splits * m * n * 4 || !aligned16(ws) || (n & 3) || (ldc & 3) || !aligned16(c))
      return SF_EINVAL;
    out = static_cast<float*>(ws);
    ldo = n;
    sstride = m * n;
    ob = nullptr;
    obeta = 0.0f;
  }
  static unsigned long long optinp = 0, optinw = 0;
  const int mi = static_cast<int>(m), ni = static_cast<int>(n), ki = static_cast<int>(k);
  // N = 256 tiles: the smem traffic per MMA of three products over two planes
  // per operand is 4/3 of the six-product form's, the wider B tile cuts the
  // A reads in half (g_tc_stages 0: auto, N >= 256 -> wide)
  const bool wide = g_tc_stages == 1 || (g_tc_stages == 0 && n >= 256);
  const int64_t tn = wide ? (n + 255) / 256 : (n + kBN - 1) / kBN;
  const int64_t units = tn * tiles_m * splits;
  const unsigned ctas = static_cast<unsigned>(units < num_sms() ? units : num_sms());
  CUtensorMap ta3, tb3;
  if (!make_map3(&ta3, a_planes, m, k, 1, kBM, 2) || !make_map3(&tb3, b_planes, n, k, 1, wide ? 256 : kBN, 2))
    return SF_EUNAVAILABLE;
  CUtensorMap tc3;
  const bool ts = g_tma_store && (obeta == 0.0f || obeta == 1.0f) && make_map_c(&tc3, out, m, n, ldo, splits, sstride);
  if (ts && g_gemm_pair && g_tc_stages == 0 && m >= 256 && n >= 256 && num_sms() >= 2) {
    const int pbn = g_pair_bn;
    CUtensorMap ta2, tb2;
    if (!make_map3(&ta2, a_planes, m, k, 1, kBM, 2) || !make_map3(&tb2, b_planes, n, k, 1, pbn / 2, 2))
      return SF_EUNAVAILABLE;
    const int64_t units2 = ((m + 255) / 256) * ((n + pbn - 1) / pbn) * splits;
    const int64_t ncl = units2 < num_sms() / 2 ? units2 : num_sms() / 2;
    if (pbn == 256) {
      static unsigned long long optinpair = 0;
      smem_optin(k_gemm_f16x3_pair<256>, PairCfg<256>::kSmem, optinpair);
      k_gemm_f16x3_pair<256><<<static_cast<unsigned>(2 * ncl), 192, PairCfg<256>::kSmem, as_stream(stream)>>>(
          ta2, tb2, tc3, mi, ni, ki, obeta, kb_per, static_cast<int>(splits), ob, a_row_scale);
    } else {
      static unsigned long long optinpair = 0;
      smem_optin(k_gemm_f16x3_pair<128>, PairCfg<128>::kSmem, optinpair);
      k_gemm_f16x3_pair<128><<<static_cast<unsigned>(2 * ncl), 192, PairCfg<128>::kSmem, as_stream(stream)>>>(
          ta2, tb2, tc3, mi, ni, ki, obeta, kb_per, static_cast<int>(splits), ob, a_row_scale);
    }
  } else if (wide && ts) {
    static unsigned long long optints = 0;
    smem_optin(k_gemm_split6_persistent<256, 2, true>, PCfg<256, 2>::kSmemTS, optints);
    k_gemm_split6_persistent<256, 2, true><<<ctas, 192, PCfg<256, 2>::kSmemTS, as_stream(stream)>>>(
        ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0, a_row_scale, tc3);
  } else if (!wide && ts) {
    static unsigned long long optints = 0;
    smem_optin(k_gemm_split6_persistent<128, 2, true>, PCfg<128, 2>::kSmemTS, optints);
    k_gemm_split6_persistent<128, 2, true><<<ctas, 192, PCfg<128, 2>::kSmemTS, as_stream(stream)>>>(
        ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0, a_row_scale, tc3);
  } else if (wide) {
    smem_optin(k_gemm_split6_persistent<256, 2>, PCfg<256, 2>::kSmem, optinw);
    k_gemm_split6_persistent<256, 2><<<ctas, 192, PCfg<256, 2>::kSmem, as_stream(stream)>>>(
        ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0, a_row_scale);
  } else {
    smem_optin(k_gemm_split6_persistent<128, 2>, PCfg<128, 2>::kSmem, optinp);
    k_gemm_split6_persistent<128, 2><<<ctas, 192, PCfg<128, 2>::kSmem, as_stream(stream)>>>(
        ta3, tb3, mi, ni, ki, out, ldo, ob, obeta, kb_per, sstride, static_cast<int>(splits), 1, 0, a_row_scale);
  }
  if (splits > 1) {
    const int rc = check_launch();
    if (rc != SF_OK) return rc;
    k_splitk_reduce<<<grid_for(m * n / 4, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const float*>(ws), static_cast<int>(splits), m, n, c, ldc, bias, beta);
  }
  return check_launch();
}

int sf_gemm_split6_a32(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda, const void* b_planes,
                       float* c, int64_t ldc, const float* bias, float beta, void* ws, int64_t ws_bytes,
                       void* stream) {
  using namespace sf;
  if (m < 0 || n < 0 || k < 0 || ldc < n || lda < k) return SF_EINVAL;
  if (m == 0 || n == 0) return SF_OK;
  if (!a || !b_planes || !c || k == 0 || (k & 7) || (lda & 3) || 3 * n > INT32_MAX || m > INT32_MAX ||
      !aligned16(a) || !aligned16(b_planes))
    return SF_EINVAL;
  CUtensorMap ta, tb;
  if (!make_map_f32(&ta, a, m, k, lda) || !make_map(&tb, b_planes, n, k)) return SF_EUNAVAILABLE;
  const int64_t tiles = ((n + kBN - 1) / kBN) * ((m + kBM - 1) / kBM);
  const int64_t splits = sf_gemm_split6_splits(m, n, k);
  const int kb_per = static_cast<int>(((k + kBK - 1) / kBK + splits - 1) / splits);
  float* out = c;
  int64_t ldo = ldc, sstride = 0;
  const float* ob = bias;
  float obeta = beta;
  if (splits > 1) {
    if (!ws || ws_bytes < splits * m * n * 4 || !aligned16(ws) || (n & 3) || (ldc & 3) || !aligned16(c))
      return SF_EINVAL;
    out = static_cast<float*>(ws);
    ldo = n;
    sstride = m * n;
    ob = nullptr;
    obeta = 0.0f;
  }
  static unsigned long long optin = 0;
  smem_optin(k_gemm_split6_a32, kCSmem, optin);
  const int64_t units = tiles * splits;
  const unsigned ctas = static_cast<unsigned>(units < num_sms() ? units : num_sms());
  k_gemm_split6_a32<<<ctas, kCThreads, kCSmem, as_stream(stream)>>>(ta, tb, static_cast<int>(m), static_cast<int>(n),
                                                               static_cast<int>(k), out, ldo, ob, obeta, kb_per,
                                                               sstride, static_cast<int>(splits));
  if (splits > 1) {
    const int rc = check_launch();
    if (rc != SF_OK) return rc;
    k_splitk_reduce<<<grid_for(m * n / 4, 256), 256, 0, as_stream(stream)>>>(
        static_cast<const float*>(ws), static_cast<int>(splits), m, n, c, ldc, bias, beta);
  }
  return check_launch();
}

int sf_gemm_split6_batched(int64_t m, int64_t n, int64_t k, int64_t batch, const void* a_planes,
                           const void* b_planes, float* c, int64_t c_bstride, void* stream) {
  using namespace sf;
  if (m < 0 || n < 0 || k < 0 || batch < 0 || c_bstride < m * n) return SF_EINVAL;
  if (m == 0 || n == 0 || batch == 0) return SF_OK;
  if (!a_planes || !b_planes || !c || k == 0 || (k & 7) || m > INT32_MAX || n > INT32_MAX || 3 * batch > INT32_MAX ||
      !aligned16(a_planes) || !aligned16(b_planes))
    return SF_EINVAL;
  CUtensorMap ta3, tb3;
  if (!make_map3(&ta3, a_planes, m, k, batch, kBM) || !make_map3(&tb3, b_planes, n, k, batch, kBN))
    return SF_EUNAVAILABLE;
  const int64_t units = ((n + kBN - 1) / kBN) * ((m + kBM - 1) / kBM) * batch;
  if (units > INT32_MAX) return SF_EINVAL;
  static unsigned long long optin = 0;
  smem_optin(k_gemm_split6_persistent<128>, PCfg<128>::kSmem, optin);
  const unsigned ctas = static_cast<unsigned>(units < num_sms() ? units : num_sms());
  k_gemm_split6_persistent<128><<<ctas, 192, PCfg<128>::kSmem, as_stream(stream)>>>(
      ta3, tb3, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), c, n, nullptr, 0.0f,
      static_cast<int>((k + kBK - 1) / kBK), 0, 1, static_cast<int>(batch), c_bstride);
  return check_launch();
}

int sf_split3_bf16_batched(const float* x, int64_t batch, int64_t rows, int64_t cols, int64_t ld,
                           int64_t x_bstride, void* planes, void* stream) {
  using namespace sf;
  if (batch < 0 || rows < 0 || cols < 0 || ld < cols || batch > 65535) return SF_EINVAL;
  if (batch * rows * cols == 0) return SF_OK;
  if (!x || !planes || !aligned16(planes)) return SF_EINVAL;
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 63) / 64),
            static_cast<unsigned>(batch));
  if (grid.y > 65535u) return SF_EINVAL;
  k_split3_t<<<grid, 256, 0, as_stream(stream)>>>(x, rows, cols, ld, static_cast<__nv_bfloat16*>(planes),
                                                   batch * rows * cols, x_bstride, rows * cols);
  return check_launch();
}

}  // extern "C"
