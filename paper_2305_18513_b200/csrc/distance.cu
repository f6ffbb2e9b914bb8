// K8 per-layer update distance (numpy-pairwise exact) and K9 the fused
// f32 AdamW step that produces it without a before-copy.  Two launches: the
// chunk kernel (update + exact chunk subtrees) and one CTA per layer for
// the combine trees above the chunks and the layer's fold.
//
// Reference: layer_distance / update_distances (scheduler.py:92-120),
// OptimizerState.step (trainer.py:50-76), fine_tune (trainer.py:194-200).
//
// numpy's float64 add-reduce over a contiguous array is a recursive pairwise
// sum: blocks of n <= 128 are summed with 8 interleaved accumulators
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail
// (n < 8: plain sequential sum), larger n split at n/2 rounded down to a
// multiple of 8.  The host cuts each parameter's tree into subtrees of at
// most SF_DIST_CHUNK elements ("chunks"); one CTA evaluates one chunk
// exactly (8 lanes per leaf, shuffles in numpy's combine order, then the
// subtree recursion), and one CTA per parameter evaluates the tree above
// the chunks level by level.  No floating-point atomics anywhere, so the
// result is bit-identical to np.sum on every run.
//
// This translation unit is compiled with -fmad=false: AdamW must round
// every f32 multiply and add separately, as numpy does.
#include "common.cuh"

namespace sf {

constexpr int kDT = 256;
constexpr int kChunk = SF_DIST_CHUNK;
constexpr int kMaxLeaves = 64;    // leaves of a <= 4096-element subtree hold >= 64 elements
constexpr int kProgMax = 4 + 2 * kMaxLeaves + 2 * kMaxLeaves + 16;
constexpr double kGuard = 1.0e-12;

// Slot-table words (per call, one row of SF_SLOT_WORDS int64 per active slot)
__device__ __forceinline__ float lo_f(int64_t w) {
  return __uint_as_float(static_cast<uint32_t>(static_cast<uint64_t>(w) & 0xFFFFFFFFu));
}
__device__ __forceinline__ float hi_f(int64_t w) {
  return __uint_as_float(static_cast<uint32_t>(static_cast<uint64_t>(w) >> 32));
}

__device__ __forceinline__ double rel_change(float before, float after) {
  const double pb = static_cast<double>(before), pa = static_cast<double>(after);
  return fabs(pa - pb) / (fabs(pb) + kGuard);
}

struct AdamC {
  float b1, ob1, b2, ob2, bc1, bc2, eps, wd, lr;
};

// trainer.py:67-74, every op rounded separately (this TU is -fmad=false);
// returns the pre-update value's relative change as float64
__device__ __forceinline__ double adam_one(float& p, float g, float& m, float& v, const AdamC& c) {
  const float mm = c.b1 * m + c.ob1 * g;
  const float vv = c.b2 * v + (c.ob2 * g) * g;
  const float mh = mm / c.bc1;
  const float vh = vv / c.bc2;
  const float u = mh / (sqrtf(vh) + c.eps) + c.wd * p;
  const float pn = p - c.lr * u;
  const double e = rel_change(p, pn);
  m = mm;
  v = vv;
  p = pn;
  return e;
}

// trainer.py:63-64 (SGD): p - f32(lr * g), numpy's weak-scalar promotion
// keeps both ops in f32, each rounded (-fmad=false)
__device__ __forceinline__ double sgd_one(float& p, float g, float lr) {
  const float pn = p - lr * g;
  const double e = rel_change(p, pn);
  p = pn;
  return e;
}

// One CTA = one chunk: a complete subtree of numpy's pairwise reduction.
// Its shape comes from a host-built program shared by all chunks of the
// same length: leaves (offset, length) and the level-ordered internal nodes.
//   prog = [nleaves, nnodes, nlevels, 0, leaves.., nodes.., level bounds..]
// UPD: SF_UPDATE_NONE (distance of before/after), SF_UPDATE_ADAMW,
// SF_UPDATE_SGD (update the parameter, distance from the value in registers)
template <int UPD>
__global__ void __launch_bounds__(kDT) k_dist_chunks(const int64_t* __restrict__ slots,
                                                     int32_t n_active,
                                                     const int32_t* __restrict__ chunk_tab,
                                                     const int32_t* __restrict__ prog_tab,
                                                     double* __restrict__ chunk_sum,
                                                     const float* __restrict__ guard) {
  pdl_trigger();
  // a non-finite loss (trainer.py: TrainingDiverged is raised before the
  // optimizer runs) leaves parameters, moments and distances untouched
  if (guard && !isfinite(__ldg(guard))) return;
  __shared__ double e[kChunk];
  __shared__ double val[2 * kMaxLeaves];     // leaf sums then internal nodes
  __shared__ __align__(16) int prog[kProgMax];
  __shared__ int s_slot;
  const int64_t b = blockIdx.x;
  if (threadIdx.x < 32) {   // last slot whose chunk base <= b (warp-parallel search)
    int lo = 0, hi = n_active - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (slots[static_cast<int64_t>(mid) * SF_SLOT_WORDS + SF_SLOT_CBASE] <= b)
        lo = mid;
      else
        hi = mid - 1;
    }
    if (threadIdx.x == 0) s_slot = lo;
  }
  __syncthreads();
  const int64_t* sl = slots + static_cast<int64_t>(s_slot) * SF_SLOT_WORDS;
  const int64_t c = b - sl[SF_SLOT_CBASE];
  const int4 ch = reinterpret_cast<const int4*>(chunk_tab)[sl[SF_SLOT_CHUNK0] + c];
  const int off = ch.x, len = ch.y;
  {
    const int* pg = prog_tab + ch.z;
    const int plen = 4 + 2 * pg[0] + 2 * pg[1] + pg[2] + 1;
    for (int i = threadIdx.x; i < plen; i += kDT) prog[i] = pg[i];
  }

  float* A = reinterpret_cast<float*>(sl[SF_SLOT_A]) + off;
  const float* B = reinterpret_cast<const float*>(sl[SF_SLOT_B]) + off;
  // chunk offsets are multiples of 8 elements, so float4 access is aligned
  // whenever the parameter's base pointer is
  const bool vec = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0;
  if (UPD == SF_UPDATE_ADAMW) {
    float* M = reinterpret_cast<float*>(sl[SF_SLOT_M]) + off;
    float* V = reinterpret_cast<float*>(sl[SF_SLOT_V]) + off;
    AdamC cc;
    cc.b1 = lo_f(sl[SF_SLOT_BETA1]);
    cc.ob1 = hi_f(sl[SF_SLOT_BETA1]);
    cc.b2 = lo_f(sl[SF_SLOT_BETA2]);
    cc.ob2 = hi_f(sl[SF_SLOT_BETA2]);
    cc.bc1 = lo_f(sl[SF_SLOT_BC]);
    cc.bc2 = hi_f(sl[SF_SLOT_BC]);
    cc.eps = lo_f(sl[SF_SLOT_EPSWD]);
    cc.wd = hi_f(sl[SF_SLOT_EPSWD]);
    cc.lr = lo_f(sl[SF_SLOT_LR]);
    const bool vec4 = vec && ((reinterpret_cast<uintptr_t>(M) | reinterpret_cast<uintptr_t>(V)) & 15u) == 0;
    const int n4 = vec4 ? len / 4 : 0;
    for (int i = threadIdx.x; i < n4; i += kDT) {
      float4 p = reinterpret_cast<float4*>(A)[i];
      const float4 g = __ldg(reinterpret_cast<const float4*>(B) + i);
      float4 m = reinterpret_cast<float4*>(M)[i];
      float4 v = reinterpret_cast<float4*>(V)[i];
      e[4 * i] = adam_one(p.x, g.x, m.x, v.x, cc);
      e[4 * i + 1] = adam_one(p.y, g.y, m.y, v.y, cc);
      e[4 * i + 2] = adam_one(p.z, g.z, m.z, v.z, cc);
      e[4 * i + 3] = adam_one(p.w, g.w, m.w, v.w, cc);
      reinterpret_cast<float4*>(A)[i] = p;
      reinterpret_cast<float4*>(M)[i] = m;
      reinterpret_cast<float4*>(V)[i] = v;
    }
    for (int i = 4 * n4 + threadIdx.x; i < len; i += kDT) {
      float p = A[i], m = M[i], v = V[i];
      e[i] = adam_one(p, B[i], m, v, cc);
      A[i] = p;
      M[i] = m;
      V[i] = v;
    }
  } else if (UPD == SF_UPDATE_SGD) {
    const float lr = lo_f(sl[SF_SLOT_LR]);
    const bool full = vec && len == kChunk;
    if (full) {
      constexpr int kQ = kChunk / kDT / 4;
      float4 p[kQ], g[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int i = threadIdx.x + q * kDT;
        p[q] = reinterpret_cast<float4*>(A)[i];
        g[q] = __ldg(reinterpret_cast<const float4*>(B) + i);
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int i = threadIdx.x + q * kDT;
        e[4 * i] = sgd_one(p[q].x, g[q].x, lr);
        e[4 * i + 1] = sgd_one(p[q].y, g[q].y, lr);
        e[4 * i + 2] = sgd_one(p[q].z, g[q].z, lr);
        e[4 * i + 3] = sgd_one(p[q].w, g[q].w, lr);
        reinterpret_cast<float4*>(A)[i] = p[q];
      }
    }
    const int n4 = vec && !full ? len / 4 : 0;
    for (int i = threadIdx.x; i < n4; i += kDT) {
      float4 p = reinterpret_cast<float4*>(A)[i];
      const float4 g = __ldg(reinterpret_cast<const float4*>(B) + i);
      e[4 * i] = sgd_one(p.x, g.x, lr);
      e[4 * i + 1] = sgd_one(p.y, g.y, lr);
      e[4 * i + 2] = sgd_one(p.z, g.z, lr);
      e[4 * i + 3] = sgd_one(p.w, g.w, lr);
      reinterpret_cast<float4*>(A)[i] = p;
    }
    for (int i = (full ? len : 4 * n4) + threadIdx.x; i < len; i += kDT) {
      float p = A[i];
      e[i] = sgd_one(p, B[i], lr);
      A[i] = p;
    }
  } else {
    const int n4 = vec ? len / 4 : 0;
    for (int i = threadIdx.x; i < n4; i += kDT) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(A) + i);
      const float4 z = __ldg(reinterpret_cast<const float4*>(B) + i);
      e[4 * i] = rel_change(a.x, z.x);
      e[4 * i + 1] = rel_change(a.y, z.y);
      e[4 * i + 2] = rel_change(a.z, z.z);
      e[4 * i + 3] = rel_change(a.w, z.w);
    }
    for (int i = 4 * n4 + threadIdx.x; i < len; i += kDT) e[i] = rel_change(A[i], B[i]);
  }
  __syncthreads();
  const int nl = prog[0], nn = prog[1], nlev = prog[2];
  const int2* leaves = reinterpret_cast<const int2*>(prog + 4);
  const int2* nodes = reinterpret_cast<const int2*>(prog + 4 + 2 * nl);
  const int* levels = prog + 4 + 2 * nl + 2 * nn;
  // leaf sums: 8 lanes per leaf, lane j owns numpy's accumulator r[j]
  const int sub = threadIdx.x & 7;
  for (int l0 = threadIdx.x >> 3; l0 < ((nl + 3) & ~3); l0 += kDT / 8) {
    const bool valid = l0 < nl;
    const int2 lf = valid ? leaves[l0] : make_int2(0, 0);
    const double* a = e + lf.x;
    const int n = lf.y;
    double r = 0.0;
    if (valid && n >= 8) {
      r = a[sub];
      for (int i = 8; i < n - (n % 8); i += 8) r = r + a[i + sub];
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) across the 8-lane group
    r = r + __shfl_xor_sync(0xFFFFFFFFu, r, 1);
    r = r + __shfl_xor_sync(0xFFFFFFFFu, r, 2);
    r = r + __shfl_xor_sync(0xFFFFFFFFu, r, 4);
    if (valid && sub == 0) {
      double res;
      if (n < 8) {
        res = 0.0;
        for (int i = 0; i < n; ++i) res = res + a[i];
      } else {
        res = r;
        for (int i = n - (n % 8); i < n; ++i) res = res + a[i];
      }
      val[l0] = res;
    }
  }
  __syncthreads();
  // internal nodes, one level at a time (children always on earlier levels)
  for (int lv = 0; lv < nlev; ++lv) {
    for (int i = levels[lv] + threadIdx.x; i < levels[lv + 1]; i += kDT) {
      const int2 lr = nodes[i];
      val[nl + i] = val[lr.x] + val[lr.y];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) chunk_sum[b] = nn ? val[nl + nn - 1] : val[0];
}

// The combine tree above one slot's chunks, level by level.  When the
// slot's chunk sums and tree fit (<= kTreeCap each), they are staged in
// shared memory first (every load in flight at once) and the levels run on
// shared memory alone; otherwise the nodes live in `node_val`.
constexpr int kTreeCap = 8192;
constexpr size_t kTreeSmem = size_t(kTreeCap) * (2 * sizeof(double) + sizeof(int2)) + 64 * sizeof(int);

__device__ double slot_tree(const int64_t* __restrict__ sl, const int32_t* __restrict__ tree_tab,
                            const int32_t* __restrict__ level_tab, const double* __restrict__ chunk_sum,
                            double* __restrict__ node_val, unsigned char* smem) {
  __shared__ double s_res;
  const int64_t cbase = sl[SF_SLOT_CBASE];
  const int nchunk = static_cast<int>(sl[SF_SLOT_NCHUNK]);
  const int64_t t0 = sl[SF_SLOT_TREE0];
  const int nnode = static_cast<int>(sl[SF_SLOT_NNODE]);
  const int64_t l0 = sl[SF_SLOT_LEVEL0];
  const int nlevel = static_cast<int>(sl[SF_SLOT_NLEVEL]);
  if (nnode == 0) return __ldcg(chunk_sum + cbase);
  const int2* tree = reinterpret_cast<const int2*>(tree_tab) + t0;
  if (nchunk <= kTreeCap && nnode <= kTreeCap && nlevel < 64) {
    double* sc = reinterpret_cast<double*>(smem);
    double* nv = sc + kTreeCap;
    int2* tr = reinterpret_cast<int2*>(nv + kTreeCap);
    int* lvl = reinterpret_cast<int*>(tr + kTreeCap);
    constexpr int kB = 8;
    for (int i0 = 0; i0 < nchunk; i0 += kB * blockDim.x) {
      double c[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = i0 + threadIdx.x + q * blockDim.x;
        c[q] = i < nchunk ? __ldcg(chunk_sum + cbase + i) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = i0 + threadIdx.x + q * blockDim.x;
        if (i < nchunk) sc[i] = c[q];
      }
    }
    for (int i0 = 0; i0 < nnode; i0 += kB * blockDim.x) {
      int2 c[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = i0 + threadIdx.x + q * blockDim.x;
        c[q] = i < nnode ? __ldg(tree + i) : make_int2(0, 0);
      }
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = i0 + threadIdx.x + q * blockDim.x;
        if (i < nnode) tr[i] = c[q];
      }
    }
    for (int i = threadIdx.x; i <= nlevel; i += blockDim.x) lvl[i] = __ldg(level_tab + l0 + i);
    __syncthreads();
    for (int lv = 0; lv < nlevel; ++lv) {
      for (int i = lvl[lv] + threadIdx.x; i < lvl[lv + 1]; i += blockDim.x) {
        const int2 lr = tr[i];
        nv[i] = (lr.x < nchunk ? sc[lr.x] : nv[lr.x - nchunk]) + (lr.y < nchunk ? sc[lr.y] : nv[lr.y - nchunk]);
      }
      __syncthreads();
    }
    const double r = nv[nnode - 1];
    __syncthreads();
    return r;
  }
  double* nv = node_val + t0;
  for (int lv = 0; lv < nlevel; ++lv) {
    const int a = __ldg(level_tab + l0 + lv), z = __ldg(level_tab + l0 + lv + 1);
    for (int i = a + threadIdx.x; i < z; i += blockDim.x) {
      const int2 lr = __ldg(tree + i);
      const double L = lr.x < nchunk ? __ldcg(chunk_sum + cbase + lr.x) : __ldcg(nv + lr.x - nchunk);
      const double R = lr.y < nchunk ? __ldcg(chunk_sum + cbase + lr.y) : __ldcg(nv + lr.y - nchunk);
      nv[i] = L + R;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) s_res = __ldcg(nv + nnode - 1);
  __syncthreads();
  const double r = s_res;
  __syncthreads();
  return r;
}

// One CTA per active layer: d[layer] = (((0.0 + S0) + S1) + ...) / count,
// a Python-float left fold over the layer's parameters in registry order
// (scheduler.py:100-105), each S the combine tree above the parameter's
// chunks.  A parameter the step did not move (no gradient) has S = 0.0
// exactly and is left out of the fold (x + 0.0 == x for the non-negative
// partials) but counted in `count`; a layer with no moved parameter gets 0.0.
__global__ void __launch_bounds__(kDT) k_dist_layers(const int64_t* __restrict__ slots,
                                                     const int32_t* __restrict__ tree_tab,
                                                     const int32_t* __restrict__ level_tab,
                                                     const double* __restrict__ chunk_sum,
                                                     double* __restrict__ node_val,
                                                     const int32_t* __restrict__ layers,
                                                     const int64_t* __restrict__ counts,
                                                     double* __restrict__ d_out,
                                                     const float* __restrict__ guard) {
  extern __shared__ __align__(16) unsigned char tsm[];
  pdl_wait();
  if (guard && !isfinite(__ldg(guard))) return;
  const int i = blockIdx.x;
  const int j0 = layers[3 * i], nr = layers[3 * i + 1], out = layers[3 * i + 2];
  double total = 0.0;
  for (int j = 0; j < nr; ++j)
    total = total + slot_tree(slots + static_cast<int64_t>(j0 + j) * SF_SLOT_WORDS, tree_tab, level_tab,
                              chunk_sum, node_val, tsm);
  if (threadIdx.x == 0) {
    const int64_t c = counts[i];
    d_out[out] = c > 0 ? total / static_cast<double>(c) : 0.0;
  }
}

inline size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace sf

using namespace sf;

extern "C" {

size_t sf_distance_workspace_bytes(int64_t total_chunks, int32_t n_active, int64_t total_nodes) {
  return a256(static_cast<size_t>(total_chunks > 0 ? total_chunks : 1) * sizeof(double)) +
         a256(static_cast<size_t>(n_active > 0 ? n_active : 1) * sizeof(double)) +
         a256(static_cast<size_t>(total_nodes > 0 ? total_nodes : 1) * sizeof(double));
}

int sf_layer_distance(const int64_t* slots, int32_t n_active, int64_t total_chunks,
                      const int32_t* chunk_tab, const int32_t* prog_tab, const int32_t* tree_tab,
                      const int32_t* level_tab, int64_t total_nodes, const int32_t* layers,
                      const int64_t* layer_counts, int32_t n_layers, double* d_out, int update,
                      const float* guard, void* ws, void* stream) {
  if (n_active < 0 || total_chunks < 0 || n_layers < 0 || !ws) return SF_EINVAL;
  if (update != SF_UPDATE_NONE && update != SF_UPDATE_ADAMW && update != SF_UPDATE_SGD) return SF_EINVAL;
  if (n_layers > 0 && (!layers || !layer_counts || !d_out)) return SF_EINVAL;
  cudaStream_t s = as_stream(stream);
  static unsigned long long smem_done = 0;
  smem_optin(k_dist_layers, kTreeSmem, smem_done);
  if (n_active == 0 || total_chunks == 0) {
    // active layers none of whose parameters moved: d = 0.0 (scheduler.py:100-105)
    if (n_layers > 0)
      k_dist_layers<<<n_layers, kDT, 0, s>>>(nullptr, nullptr, nullptr, nullptr, nullptr, layers, layer_counts,
                                             d_out, guard);
    return n_layers > 0 ? check_launch() : SF_OK;
  }
  if (!slots || !chunk_tab || !prog_tab || !tree_tab || !level_tab) return SF_EINVAL;
  if (total_chunks > 0x7FFFFFFFLL) return SF_EINVAL;
  char* w = static_cast<char*>(ws);
  double* chunk_sum = reinterpret_cast<double*>(w);
  w += a256(static_cast<size_t>(total_chunks) * sizeof(double));
  w += a256(static_cast<size_t>(n_active) * sizeof(double));     // (per-slot totals: unused, layout kept)
  double* node_val = reinterpret_cast<double*>(w);
  (void)total_nodes;
  if (update == SF_UPDATE_ADAMW)
    k_dist_chunks<SF_UPDATE_ADAMW><<<static_cast<unsigned>(total_chunks), kDT, 0, s>>>(
        slots, n_active, chunk_tab, prog_tab, chunk_sum, guard);
  else if (update == SF_UPDATE_SGD)
    k_dist_chunks<SF_UPDATE_SGD><<<static_cast<unsigned>(total_chunks), kDT, 0, s>>>(
        slots, n_active, chunk_tab, prog_tab, chunk_sum, guard);
  else
    k_dist_chunks<SF_UPDATE_NONE><<<static_cast<unsigned>(total_chunks), kDT, 0, s>>>(
        slots, n_active, chunk_tab, prog_tab, chunk_sum, guard);
  if (n_layers > 0)
    launch_pdl(k_dist_layers, dim3(static_cast<unsigned>(n_layers)), dim3(kDT), kTreeSmem, s,
               static_cast<const int64_t*>(slots), tree_tab, level_tab, static_cast<const double*>(chunk_sum),
               node_val, layers, layer_counts, d_out, guard);
  return check_launch();
}

}  // extern "C"
