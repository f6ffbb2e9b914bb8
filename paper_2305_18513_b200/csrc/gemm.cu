// Dense fp32 GEMMs of the encoder step (the model's Linear layers and the
// attention score/context batched products, tensor.py:290-379 in the
// reference, which computes them with numpy/OpenBLAS in float32).
//
// These are the only tensor-core-shaped work in the step and, per the
// north_star, they are left to cuBLAS: this file is a thin C-ABI over
// cuBLASLt.  The one B200-specific choice is the arithmetic mode:
//
//   SF_GEMM_FP32     CUBLAS_COMPUTE_32F            (SIMT FFMA, ~75 TF/s)
//   SF_GEMM_BF16X9   CUBLAS_COMPUTE_32F_EMULATED_16BFX9: each fp32 operand
//                    is split into three bf16 terms and the products are
//                    accumulated in fp32 on the 5th-gen tensor cores —
//                    fp32-accurate results at tensor-core throughput
//   SF_GEMM_TF32     CUBLAS_COMPUTE_32F_FAST_TF32  (one pass, 10-bit mantissa;
//                    opt-in only, not fp32-accurate)
//
// BF16x9 emulation exists in cuBLASLt >= 12.9.  PyTorch ships and loads its
// own cuBLASLt 12.8 (no emulation), so the toolkit's 12.9 library is opened
// privately by absolute path with RTLD_LOCAL | RTLD_DEEPBIND (its internal
// references bind to itself, never to torch's copy; it only depends on libc)
// and every entry point is taken with dlsym from that handle.
//
// Row-major convention (PyTorch's): C[b] = op(A[b]) @ op(B[b]) (+ bias[col])
// (+ beta * C[b]).  cuBLAS is column-major, so the call is issued as
// C^T = op(B)^T op(A)^T with the operands swapped.
#include <cublasLt.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace sf {
namespace {

using PFN_create = cublasStatus_t (*)(cublasLtHandle_t*);
using PFN_desc_create = cublasStatus_t (*)(cublasLtMatmulDesc_t*, cublasComputeType_t, cudaDataType_t);
using PFN_desc_set = cublasStatus_t (*)(cublasLtMatmulDesc_t, cublasLtMatmulDescAttributes_t, const void*,
                                        size_t);
using PFN_layout_create = cublasStatus_t (*)(cublasLtMatrixLayout_t*, cudaDataType, uint64_t, uint64_t,
                                             int64_t);
using PFN_layout_set = cublasStatus_t (*)(cublasLtMatrixLayout_t, cublasLtMatrixLayoutAttribute_t,
                                          const void*, size_t);
using PFN_pref_create = cublasStatus_t (*)(cublasLtMatmulPreference_t*);
using PFN_pref_set = cublasStatus_t (*)(cublasLtMatmulPreference_t, cublasLtMatmulPreferenceAttributes_t,
                                        const void*, size_t);
using PFN_heur = cublasStatus_t (*)(cublasLtHandle_t, cublasLtMatmulDesc_t, cublasLtMatrixLayout_t,
                                    cublasLtMatrixLayout_t, cublasLtMatrixLayout_t, cublasLtMatrixLayout_t,
                                    cublasLtMatmulPreference_t, int, cublasLtMatmulHeuristicResult_t*, int*);
using PFN_matmul = cublasStatus_t (*)(cublasLtHandle_t, cublasLtMatmulDesc_t, const void*, const void*,
                                      cublasLtMatrixLayout_t, const void*, cublasLtMatrixLayout_t, const void*,
                                      const void*, cublasLtMatrixLayout_t, void*, cublasLtMatrixLayout_t,
                                      const cublasLtMatmulAlgo_t*, void*, size_t, cudaStream_t);
using PFN_version = size_t (*)(void);

struct Lt {
  void* dl = nullptr;
  cublasLtHandle_t handle = nullptr;
  size_t version = 0;
  PFN_desc_create desc_create = nullptr;
  PFN_desc_set desc_set = nullptr;
  PFN_layout_create layout_create = nullptr;
  PFN_layout_set layout_set = nullptr;
  PFN_pref_create pref_create = nullptr;
  PFN_pref_set pref_set = nullptr;
  PFN_heur heur = nullptr;
  PFN_matmul matmul = nullptr;
  char error[256] = {0};
};

const char* kCandidates[] = {
    "/usr/local/cuda/lib64/libcublasLt.so.12",
    "/usr/local/cuda/targets/x86_64-linux/lib/libcublasLt.so.12",
    "/usr/local/cuda-12.9/lib64/libcublasLt.so.12",
};

Lt& lt_state() {
  static Lt lt;
  return lt;
}

Lt* lt_load() {
  Lt& lt = lt_state();
  static std::once_flag once;
  std::call_once(once, [&lt] {
    const char* env = getenv("SLIMFIT_CUBLASLT");
    void* h = nullptr;
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND);
    for (const char* p : kCandidates) {
      if (h) break;
      h = dlopen(p, RTLD_NOW | RTLD_LOCAL | RTLD_DEEPBIND);
    }
    if (!h) {
      snprintf(lt.error, sizeof lt.error, "cannot dlopen the toolkit cuBLASLt: %s", dlerror());
      return;
    }
    auto create = reinterpret_cast<PFN_create>(dlsym(h, "cublasLtCreate"));
    auto ver = reinterpret_cast<PFN_version>(dlsym(h, "cublasLtGetVersion"));
    lt.desc_create = reinterpret_cast<PFN_desc_create>(dlsym(h, "cublasLtMatmulDescCreate"));
    lt.desc_set = reinterpret_cast<PFN_desc_set>(dlsym(h, "cublasLtMatmulDescSetAttribute"));
    lt.layout_create = reinterpret_cast<PFN_layout_create>(dlsym(h, "cublasLtMatrixLayoutCreate"));
    lt.layout_set = reinterpret_cast<PFN_layout_set>(dlsym(h, "cublasLtMatrixLayoutSetAttribute"));
    lt.pref_create = reinterpret_cast<PFN_pref_create>(dlsym(h, "cublasLtMatmulPreferenceCreate"));
    lt.pref_set = reinterpret_cast<PFN_pref_set>(dlsym(h, "cublasLtMatmulPreferenceSetAttribute"));
    lt.heur = reinterpret_cast<PFN_heur>(dlsym(h, "cublasLtMatmulAlgoGetHeuristic"));
    lt.matmul = reinterpret_cast<PFN_matmul>(dlsym(h, "cublasLtMatmul"));
    if (!create || !ver || !lt.desc_create || !lt.desc_set || !lt.layout_create || !lt.layout_set ||
        !lt.pref_create || !lt.pref_set || !lt.heur || !lt.matmul) {
      snprintf(lt.error, sizeof lt.error, "cuBLASLt lacks an entry point");
      return;
    }
    lt.version = ver();
    if (create(&lt.handle) != CUBLAS_STATUS_SUCCESS) {
      snprintf(lt.error, sizeof lt.error, "cublasLtCreate failed (no CUDA device?)");
      lt.handle = nullptr;
      return;
    }
    lt.dl = h;
  });
  return lt.handle ? &lt : nullptr;
}

struct Key {
  int64_t v[14];
  bool operator==(const Key& o) const { return memcmp(v, o.v, sizeof v) == 0; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    size_t h = 1469598103934665603ull;
    for (int64_t x : k.v) h = (h ^ static_cast<size_t>(x)) * 1099511628211ull;
    return h;
  }
};

constexpr int kMaxAlgos = 8;

struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo;
  size_t ws = 0;
  bool ok = false;
  // the heuristic's candidates, timed once on the first beta == 0 call
  // when SLIMFIT_GEMM_AUTOTUNE=1.  Off by default: a timing-based choice can
  // differ between processes, and different kernels round differently, so
  // runs would stop being bit-reproducible (the heuristic's first choice is
  // deterministic); measured gain 0-6% per shape
  int n_cand = 0;
  cublasLtMatmulAlgo_t cand[kMaxAlgos];
  size_t cand_ws[kMaxAlgos];
  bool tuned = false;
};

bool autotune_on() {
  static const int on = [] {
    const char* e = getenv("SLIMFIT_GEMM_AUTOTUNE");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return on != 0;
}

std::mutex g_mu;
std::unordered_map<Key, Plan, KeyHash> g_plans;
int g_last_status = 0;

cublasComputeType_t compute_of(int mode) {
  switch (mode) {
    case SF_GEMM_BF16X9: return CUBLAS_COMPUTE_32F_EMULATED_16BFX9;
    case SF_GEMM_TF32: return CUBLAS_COMPUTE_32F_FAST_TF32;
    default: return CUBLAS_COMPUTE_32F;
  }
}

// Build (once per shape) the Lt descriptors in cuBLAS's column-major view.
Plan* plan_for(Lt* lt, int ta, int tb, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t sa, int64_t ldb,
               int64_t sb, int64_t ldc, int64_t sc, int64_t batch, int has_bias, int has_beta, int mode,
               size_t ws_bytes, int device) {
  Key key{{ta, tb, m, n, k, lda, sa, ldb, sb, ldc, sc, batch,
           (int64_t)has_bias | ((int64_t)has_beta << 1) | ((int64_t)mode << 2) | ((int64_t)device << 8),
           (int64_t)ws_bytes}};
  auto it = g_plans.find(key);
  if (it != g_plans.end()) return &it->second;
  Plan& p = g_plans[key];
  // column-major: C^T (n x m, ld ldc) = op(B)^T (n x k) * op(A)^T (k x m)
  // row-major X (r x c, ld) is column-major X^T (c x r, ld).
  cublasOperation_t opA = tb ? CUBLAS_OP_T : CUBLAS_OP_N;   // applies to the stored B
  cublasOperation_t opB = ta ? CUBLAS_OP_T : CUBLAS_OP_N;   // applies to the stored A
  uint64_t a_rows = tb ? k : n, a_cols = tb ? n : k;        // stored B, column-major view
  uint64_t b_rows = ta ? m : k, b_cols = ta ? k : m;        // stored A, column-major view
  cublasStatus_t st = lt->desc_create(&p.desc, compute_of(mode), CUDA_R_32F);
  if (st == CUBLAS_STATUS_SUCCESS) st = lt->desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof opA);
  if (st == CUBLAS_STATUS_SUCCESS) st = lt->desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof opB);
  if (st == CUBLAS_STATUS_SUCCESS && has_bias) {
    cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_BIAS;
    st = lt->desc_set(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof epi);
  }
  if (st == CUBLAS_STATUS_SUCCESS) st = lt->layout_create(&p.a, CUDA_R_32F, a_rows, a_cols, ldb);
  if (st == CUBLAS_STATUS_SUCCESS) st = lt->layout_create(&p.b, CUDA_R_32F, b_rows, b_cols, lda);
  if (st == CUBLAS_STATUS_SUCCESS) st = lt->layout_create(&p.c, CUDA_R_32F, n, m, ldc);
  if (st == CUBLAS_STATUS_SUCCESS && batch > 1) {
    int32_t bc = static_cast<int32_t>(batch);
    cublasLtMatrixLayout_t ls[3] = {p.a, p.b, p.c};
    int64_t strides[3] = {sb, sa, sc};
    for (int i = 0; i < 3 && st == CUBLAS_STATUS_SUCCESS; ++i) {
      st = lt->layout_set(ls[i], CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof bc);
      if (st == CUBLAS_STATUS_SUCCESS)
        st = lt->layout_set(ls[i], CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &strides[i], sizeof(int64_t));
    }
  }
  if (st == CUBLAS_STATUS_SUCCESS) {
    cublasLtMatmulPreference_t pref = nullptr;
    st = lt->pref_create(&pref);
    uint64_t wsb = ws_bytes;
    if (st == CUBLAS_STATUS_SUCCESS)
      st = lt->pref_set(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof wsb);
    cublasLtMatmulHeuristicResult_t res[kMaxAlgos];
    int found = 0;
    if (st == CUBLAS_STATUS_SUCCESS)
      st = lt->heur(lt->handle, p.desc, p.a, p.b, p.c, p.c, pref, autotune_on() ? kMaxAlgos : 1, res, &found);
    if (st == CUBLAS_STATUS_SUCCESS && found > 0) {
      p.algo = res[0].algo;
      p.ws = res[0].workspaceSize;
      p.ok = true;
      p.n_cand = 0;
      for (int i = 0; i < found && i < kMaxAlgos; ++i) {
        if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
        p.cand[p.n_cand] = res[i].algo;
        p.cand_ws[p.n_cand] = res[i].workspaceSize;
        ++p.n_cand;
      }
      p.tuned = p.n_cand <= 1;
    } else if (st == CUBLAS_STATUS_SUCCESS) {
      st = CUBLAS_STATUS_NOT_SUPPORTED;
    }
    // the preference object is tiny; it is deliberately not destroyed
    // (cublasLtMatmulPreferenceDestroy is not bound), one per shape
  }
  g_last_status = static_cast<int>(st);
  return &p;
}

}  // namespace
}  // namespace sf

extern "C" {

int sf_gemm_available(int mode) {
  sf::Lt* lt = sf::lt_load();
  if (!lt) return 0;
  if (mode == SF_GEMM_BF16X9) return lt->version >= 120900 ? 1 : 0;
  return 1;
}

size_t sf_gemm_lt_version(void) {
  sf::Lt* lt = sf::lt_load();
  return lt ? lt->version : 0;
}

int sf_gemm_last_status(void) { return sf::g_last_status; }

const char* sf_gemm_lt_error(void) {
  sf::lt_load();
  return sf::lt_state().error;
}

int sf_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, int64_t stride_a,
                const float* B, int64_t ldb, int64_t stride_b, float* C, int64_t ldc, int64_t stride_c,
                int64_t batch, const float* bias, float beta, int mode, void* workspace, size_t ws_bytes,
                void* stream) {
  if (m < 0 || n < 0 || k < 0 || batch < 1 || mode < SF_GEMM_FP32 || mode > SF_GEMM_TF32) return SF_EINVAL;
  if (m == 0 || n == 0) return SF_OK;
  sf::Lt* lt = sf::lt_load();
  if (!lt) return SF_EUNAVAILABLE;
  if (mode == SF_GEMM_BF16X9 && lt->version < 120900) return SF_EUNAVAILABLE;
  int dev = 0;
  cudaGetDevice(&dev);
  // one lock over plan lookup, bias-pointer update and the (asynchronous)
  // enqueue: the plan's descriptor is shared by every caller of that shape
  std::lock_guard<std::mutex> g(sf::g_mu);
  sf::Plan* p = sf::plan_for(lt, ta, tb, m, n, k, lda, stride_a, ldb, stride_b, ldc, stride_c, batch,
                             bias != nullptr, beta != 0.0f, mode, ws_bytes, dev);
  if (!p->ok) return SF_EUNAVAILABLE;
  if (bias) {
    cublasStatus_t st = lt->desc_set(p->desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof bias);
    if (st != CUBLAS_STATUS_SUCCESS) return SF_EINVAL;
  }
  const float one = 1.0f;
  cudaStream_t cs = sf::as_stream(stream);
  if (!p->tuned && beta == 0.0f) {
    // first call of this shape: time each candidate once (after one warm
    // run) on the real operands and keep the fastest.  Trials overwrite C,
    // which the real call below rewrites; beta != 0 calls never tune.
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    int besti = 0;
    for (int i = 0; i < p->n_cand; ++i) {
      if (p->cand_ws[i] > ws_bytes) continue;
      bool ok = lt->matmul(lt->handle, p->desc, &one, B, p->a, A, p->b, &beta, C, p->c, C, p->c, &p->cand[i],
                           workspace, p->cand_ws[i], cs) == CUBLAS_STATUS_SUCCESS;
      cudaEventRecord(e0, cs);
      ok = ok && lt->matmul(lt->handle, p->desc, &one, B, p->a, A, p->b, &beta, C, p->c, C, p->c, &p->cand[i],
                            workspace, p->cand_ws[i], cs) == CUBLAS_STATUS_SUCCESS;
      cudaEventRecord(e1, cs);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      if (ok && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess && ms < best) {
        best = ms;
        besti = i;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGetLastError();                  // a rejected candidate must not poison later checks
    p->algo = p->cand[besti];
    p->ws = p->cand_ws[besti];
    p->tuned = true;
  }
  cublasStatus_t st = lt->matmul(lt->handle, p->desc, &one, B, p->a, A, p->b, &beta, C, p->c, C, p->c, &p->algo,
                                 workspace, p->ws, cs);
  sf::g_last_status = static_cast<int>(st);
  if (st != CUBLAS_STATUS_SUCCESS) return SF_ECUDA;
  return sf::check_launch();
}

}  // extern "C"
