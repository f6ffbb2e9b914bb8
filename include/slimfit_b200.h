/*
 * slimfit_b200.h — C ABI of the B200 (sm_100a) kernels behind the SlimFit
 * activation-memory hot path.  This is the drop-in boundary: a plain
 * `extern "C"` shared library (libslimfit_b200.so) with raw device pointers,
 * element counts and a cudaStream_t passed as `void*`.  No torch types.
 *
 * Every entry point
 *   - is stream-ordered and asynchronous (no host synchronisation unless the
 *     comment says so), never allocates device memory (callers pass the
 *     workspace sized by the matching *_workspace_bytes query), and keeps no
 *     global mutable state, so it is re-entrant across host threads;
 *   - returns SF_OK or an error code; on SF_ECUDA the CUDA error is kept in a
 *     thread-local slot readable with sf_last_cuda_error().
 *
 * The reference functions each call replaces are cited as file:line under
 * /root/reference/pkg/src/slimfit/ (the reference is pure Python/numpy, so
 * "replaces" means: same inputs, same outputs, bit-for-bit where noted).
 */
#ifndef SLIMFIT_B200_H
#define SLIMFIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SF_OK = 0,
  SF_EINVAL = 1, /* bad argument: Python side raises CodecError / ShapeError */
  SF_ERANGE = 2, /* value outside a codec's code range (pack4)               */
  SF_ECUDA = 3,  /* CUDA runtime/launch error, see sf_last_cuda_error()     */
  SF_EUNAVAILABLE = 4 /* a required library/mode is absent (no fallback)    */
};

int sf_abi_version(void);
int sf_last_cuda_error(void);
const char* sf_strerror(int code);

/* ---- K1 / K2: 8-bit fixed point --------------------------------------------
 * sf_quant8 replaces compression.quantize (compression.py:66-74) for 8-bit
 * specs, as called by CompressedActivation.quantized (:193-197) from
 * tensor._save_maybe_quant8 (tensor.py:280-283):
 *   code = clamp(round_half_away(x * 2^fb), code_min, code_max), NaN -> 0.
 * codes are int8 (is_signed) or uint8, same logical (C) order as x.
 * sf_dequant8 replaces dequantize (compression.py:77-79) / the quant8 branch
 * of CompressedActivation.decompress (:214-215): y = code * 2^-fb (exact).
 */
int sf_quant8(const float* x, void* codes, int64_t n, int fb, int is_signed, void* stream);
/* general form of K1 for any reference spec (bits in {4, 8}): codes are one
 * int8/uint8 per element, clamped to the spec's code range (compression.py:66). */
int sf_quantize(const float* x, void* codes, int64_t n, int bits, int fb, int is_signed,
                void* stream);
/* As sf_quantize for a float64 array (compression.quantize scales and rounds
 * in float64, compression.py:66-74): codes are exact for float64 inputs
 * (no float32 narrowing before the half-code decision). */
int sf_quantize_f64(const double* x, void* codes, int64_t n, int bits, int fb, int is_signed,
                    void* stream);
int sf_dequant8(const void* codes, float* y, int64_t n, int fb, int is_signed, void* stream);

/* ---- K3: percentile power-of-two prescale ------------------------------------
 * Replaces choose_prescale_exp (compression.py:111-124) with numpy 2.3.5
 * percentile(method="linear") semantics.  q is the quantile exactly as numpy
 * forms it (np.true_divide(pct, 100)); value_max is the spec's largest value
 * (1.75 for Q2.2).  Writes s = max(0, ceil(log2(p / value_max))) (0 for empty,
 * p <= 0, non-finite p, any NaN in x) to *s_dev.  Optional p_dev receives p
 * as float64 when it was materialised (NaN otherwise).  ws must hold
 * sf_prescale_workspace_bytes(n) bytes.
 */
size_t sf_prescale_workspace_bytes(int64_t n);
int sf_prescale_exp(const float* x, int64_t n, double q, float value_max, int32_t* s_dev,
                    double* p_dev, void* ws, void* stream);

/* ---- K4 / K5: 4-bit packed fixed point -----------------------------------------
 * sf_quant4_pack replaces quantize(x / 2^s, spec) + pack4 (compression.py:205,
 * :82-95): byte i = (c[2i] & 0xF) | (c[2i+1] & 0xF) << 4, odd n pads the high
 * nibble with 0.  s is read from device memory (s_dev, produced by K3).
 * sf_unpack4_dequant replaces unpack4 + dequantize * 2^s (compression.py:98-108,
 * :216-219).  packed holds (n + 1) / 2 bytes.
 */
int sf_quant4_pack(const float* x, uint8_t* packed, int64_t n, const int32_t* s_dev, int fb,
                   void* stream);
int sf_unpack4_dequant(const uint8_t* packed, float* y, int64_t n, const int32_t* s_dev, int fb,
                       void* stream);

/* ---- K6 / K7: global top-k magnitude pruning ----------------------------------
 * sf_prune_topk replaces prune_topk (compression.py:137-162): keeps the k
 * largest keys (|x| if by_magnitude, else x) over the whole flat tensor; ties
 * go to the lower index; NaN ranks below every number; indices are written
 * ascending (int32) with values[j] = x[indices[j]].  k = ceil(keep_frac * n)
 * is formed on the host in float64 exactly as the reference does.
 * sf_restore replaces restore (compression.py:165-169): dense = 0, then
 * dense[indices] = values.  Both reject n <= 0 or k outside [1, n].
 */
size_t sf_prune_workspace_bytes(int64_t n);
int sf_prune_topk(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                  int32_t* indices, void* ws, void* stream);
int sf_restore(const float* values, const int32_t* indices, int64_t k, float* dense, int64_t n,
               void* stream);
/* Same as sf_prune_topk, and when row_ptr != NULL also writes the CSR row
 * pointers of the kept set for rows of row_len elements (n % row_len == 0):
 * row_ptr[r] = #kept with index < r * row_len, row_ptr[n / row_len] = k
 * (int32, n / row_len + 1 entries) — what sf_layernorm_bwd's sparse path
 * consumes, produced in the write pass at no extra read. */
int sf_prune_topk_rows(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                       int32_t* indices, int64_t row_len, int32_t* row_ptr, void* ws,
                       void* stream);
/* sf_prune_topk_rows with a per-call-site hint: `hint` is
 * sf_prune_hint_bytes() of device memory (16-byte aligned), zeroed by the
 * caller once and then used by one call at a time (stream order); every call
 * rewrites its first 4 words with its threshold key and bracket half width,
 * and the rest holds the kernel's grid state, which each call leaves zeroed
 * (no memset per call).  With a valid hint
 * (by_magnitude only) the kernel skips the sample and the two inner grid
 * barriers (the bracket is T_prev -+ half); a hint that misses rank k falls
 * back to the general path inside the same launch.  Output identical to
 * sf_prune_topk_rows for every input.  row_ptr may be NULL. */
size_t sf_prune_hint_bytes(void);
int sf_prune_topk_hint(const float* x, int64_t n, int64_t k, int by_magnitude, float* values,
                       int32_t* indices, int64_t row_len, int32_t* row_ptr, uint32_t* hint, void* ws,
                       void* stream);
/* sf_restore with the CSR row pointers sf_prune_topk_rows wrote (row_len % 4
 * == 0, row_len <= 1536, dense 16-byte aligned): each CTA takes its rows'
 * slice of the pairs straight from row_ptr -- no search over the indices. */
int sf_restore_rows(const float* values, const int32_t* indices, int64_t k, const int32_t* row_ptr,
                    int64_t row_len, float* dense, int64_t n, void* stream);
/* ---- LayerNorm with the semi-static x~ cache (tensor.py:447-494) -------------
 * Forward over `rows` rows of width H: mean, population variance,
 * rstd = 1/sqrt(var + eps), x~ = (x - mean) * rstd, y = x~ * gamma + beta.
 * xtilde may be NULL (frozen + pruned: the caller prunes from a transient).
 * Backward (tensor.py:481-490): gg = gamma * g * rstd / H,
 *   dx = H*gg - sum(gg) - x~ * sum(gg * x~)   (row sums),
 * with x~ either dense (xtilde != NULL) or the pruned pair (values, indices,
 * k) consumed directly (fused K7, no dense restore); row_ptr (may be NULL:
 * then derived from the indices) are that pair's CSR row pointers as
 * sf_prune_topk_rows writes them.  dgamma / dbeta (may be NULL = frozen)
 * get column sums of x~*g and g.  ws: sf_layernorm_bwd_workspace_bytes.
 */
int sf_layernorm_fwd(const float* x, const float* gamma, const float* beta, float* y,
                     float* xtilde, float* rstd, int64_t rows, int64_t H, float eps, void* stream);
/* Residual LayerNorm: the row is res + (x + bias) -- the residual add
 * after a projection (tensor.py:337-379 `x @ W + b`, then model.py's
 * `x = x + a`) whose bias was left out of the GEMM, rounded in that order --
 * then the sf_layernorm_fwd outputs.  sum (may be NULL) receives the row
 * sum itself (pre-norm keeps it as the residual stream). */
int sf_layernorm_fwd_residual(const float* res, const float* x, const float* bias, const float* gamma,
                              const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                              int64_t rows, int64_t H, float eps, void* stream);
size_t sf_layernorm_bwd_workspace_bytes(int64_t rows, int64_t H);
int sf_layernorm_bwd(const float* g, const float* gamma, const float* xtilde,
                     const float* values, const int32_t* indices, int64_t k,
                     const int32_t* row_ptr, const float* rstd, float* dx, float* dgamma,
                     float* dbeta, int64_t rows, int64_t H, void* ws, void* stream);

/* ---- attention head layout (model.py:202-238 reshape/transpose) ------------
 * sf_split_heads: y (B, T, heads*dh) row-major -> out (B, heads, T, dh),
 * adding the projection bias (length heads*dh; may be NULL) on the way
 * (tensor.py:337-379 `x @ W + b` with the bias left out of the GEMM); when
 * codes != NULL also writes the 8-bit fixed-point codes of out (same layout,
 * = sf_quantize(out, bits 8, fb, is_signed)) for the matmul cache
 * (tensor.py:290-334).  sf_merge_heads is the inverse move (no bias).
 * dh % 4 == 0, pointers 16-byte aligned (codes 4-byte). */
int sf_split_heads(const float* y, const float* bias, float* out, void* codes, int64_t B, int64_t T,
                   int64_t heads, int64_t dh, int fb, int is_signed, void* stream);
int sf_merge_heads(const float* x, float* out, int64_t B, int64_t T, int64_t heads, int64_t dh,
                   void* stream);
/* the same move into rows of out_ld floats (>= heads*dh, % 4 == 0): the
 * q/k/v gradients merged side by side into one (B*T, 3H) operand so the
 * three projections' input gradient is one K = 3H GEMM */
int sf_merge_heads_ld(const float* x, float* out, int64_t B, int64_t T, int64_t heads, int64_t dh,
                      int64_t out_ld, void* stream);

/* ---- embedding backward ------------------------------------------------------
 * Replaces the table gradient of `embedding` (tensor.py:497-520, np.add.at):
 * dw[v] = sum over positions p with ids[p] == v of g[p], added in position
 * order, every row written (zeros where v does not occur).  perm: positions
 * stably sorted by id; starts: V + 1 segment bounds into perm (both int64,
 * computed on the device, no host round trip).  H % 4 == 0, H <= 1024. */
int sf_embedding_bwd(const float* g, const int64_t* perm, const int64_t* starts, float* dw, int64_t V,
                     int64_t H, void* stream);
/* the whole table gradient from the raw ids (int64, n of them): a stable
 * LSD radix sort of (id, position) pairs, segment bounds by binary search,
 * then the position-ordered sums -- all on the stream, no host round trip.
 * ws: sf_embedding_grad_workspace_bytes(n, V). */
size_t sf_embedding_grad_workspace_bytes(int64_t n, int64_t V);
int sf_embedding_grad(const int64_t* ids, int64_t n, const float* g, float* dw, int64_t V, int64_t H, void* ws,
                      void* stream);

/* ---- GELU (tanh form, tensor.py:382-410) with the packed4 cache fused -------
 * sf_gelu_fwd: y = 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))).
 * sf_gelu_bwd: dx = g * (0.5 (1 + t) + 0.5 x (1 - t^2) du) from raw x.
 * sf_gelu_bwd_packed4: same, decoding x from the packed4 cache on the fly
 * (fused K5; the decoded fp32 x never touches HBM).
 */
int sf_gelu_fwd(const float* x, float* y, int64_t n, void* stream);
/* GELU forward fused with K3's histogram pass over its input: one read of x
 * writes y and decides the packed4 prescale exponent of x (= sf_prescale_exp
 * semantics, s_dev / ws as there; x and y 16-byte aligned). */
int sf_gelu_fwd_prescale(const float* x, float* y, int64_t n, double q, float value_max,
                         int32_t* s_dev, void* ws, void* stream);
/* Same with the FFN projection's bias (tensor.py:337-379) fused: x holds the
 * GEMM output without bias, rows of row_len (n % row_len == 0, row_len % 4
 * == 0); x is overwritten in place with x + bias (the GELU input the packed4
 * cache then encodes), y = gelu(x + bias), s as sf_prescale_exp of x + bias. */
int sf_gelu_fwd_prescale_bias(float* x, const float* bias, int64_t row_len, float* y, int64_t n,
                              double q, float value_max, int32_t* s_dev, void* ws, void* stream);
int sf_gelu_bwd(const float* g, const float* x, float* dx, int64_t n, void* stream);
int sf_gelu_bwd_packed4(const float* g, const uint8_t* packed, const int32_t* s_dev, int fb,
                        float* dx, int64_t n, void* stream);

/* ---- Softmax writing fp32 probs and their 8-bit codes in one pass ----------
 * (tensor.py:413-444 + _save_maybe_quant8, with the preceding scale op
 * tensor.py:583-593 folded in): rows of width W of raw scores s;
 * p = softmax(s * scale); probs (may be NULL) receives p, codes receives
 * quantize(p, spec).  Backward sf_softmax_bwd_q8:
 * ds = (p * (g - sum(g * p))) * scale with p decoded from codes.
 */
int sf_softmax_fwd_q8(const float* s, float* probs, void* codes, int64_t rows, int64_t W,
                      float scale, int fb, int is_signed, void* stream);
int sf_softmax_bwd_q8(const float* g, const void* codes, float* ds, int64_t rows, int64_t W,
                      int fb, int is_signed, float scale, void* stream);

/* ---- K8 / K9: per-layer update distance, fused AdamW ---------------------------
 * Distances replace layer_distance / update_distances (scheduler.py:92-120):
 *   d[layer] = (((0.0 + S_param0) + S_param1) + ...) / count,
 *   S = numpy pairwise sum of |after - before| / (|before| + 1e-12) in fp64,
 * reproduced bit-for-bit (leaf/tree order of numpy's add-reduce).  With
 * update = SF_UPDATE_ADAMW or SF_UPDATE_SGD the same call first applies
 * OptimizerState.step (trainer.py:50-76; AdamW: f32, every op rounded,
 * per-layer bias correction constants supplied per slot; SGD: p - f32(lr g))
 * to each slot and measures the distance between the pre- and post-update
 * values it holds in registers, which removes the clone_layer_data copy
 * (trainer.py:194-200) for both optimizers.
 *
 * Static tables (device memory, built once per model by the host):
 *   chunk_tab int32[4 * n]: (offset, length, program offset, 0) of each
 *             pairwise subtree of <= SF_DIST_CHUNK elements, in depth-first
 *             order per parameter;
 *   prog_tab  int32: per distinct chunk length, the subtree's shape
 *             [nleaves, nnodes, nlevels, 0, (off, len) x nleaves,
 *              (left, right) x nnodes, level bounds x (nlevels + 1)];
 *   tree_tab  int32[2 * n]: (left, right) operand ids of the combine tree
 *             above the chunks, level-ordered (id < nchunk = chunk partial,
 *             else internal node id - nchunk); the last node is the root;
 *   level_tab int32: per parameter nlevel + 1 bounds into its tree nodes.
 * Per call: `slots` int64[n_active * SF_SLOT_WORDS] (device), one row per
 * parameter processed; `layers` int32[3 * n_layers] = (first slot row j0,
 * number of rows nr >= 0, output index): rows j0 .. j0+nr-1 are the layer's
 * moved parameters in registry order; layer_counts int64[n_layers] counts
 * ALL the layer's elements (a parameter without a gradient did not move and
 * adds 0.0 to the sum, scheduler.py:100-105; nr = 0 gives d = 0.0); d_out is
 * written at the output indices only (frozen entries untouched).  n_active =
 * 0 with n_layers > 0 only writes those zero distances.  guard (device float, may
 * be NULL): when it holds a non-finite value (the step's loss) nothing is
 * written at all -- the reference raises TrainingDiverged before its
 * optimizer step (trainer.py:175-190), so the host can check the loss after
 * the launch instead of synchronising before it.  ws holds
 * sf_distance_workspace_bytes(total_chunks, n_active, total_nodes) bytes.
 */
#define SF_DIST_CHUNK 4096
enum { SF_UPDATE_NONE = 0, SF_UPDATE_ADAMW = 1, SF_UPDATE_SGD = 2 };
enum {
  SF_SLOT_A = 0,       /* before (distance) or param p (AdamW, updated), float*  */
  SF_SLOT_B = 1,       /* after (distance) or grad g (AdamW), float*             */
  SF_SLOT_M = 2,       /* AdamW first moment, float* (updated)                   */
  SF_SLOT_V = 3,       /* AdamW second moment, float* (updated)                  */
  SF_SLOT_N = 4,       /* element count                                          */
  SF_SLOT_CHUNK0 = 5,  /* first row of this parameter in chunk_tab               */
  SF_SLOT_NCHUNK = 6,  /* number of chunks                                       */
  SF_SLOT_TREE0 = 7,   /* first row in tree_tab (and in the node workspace)      */
  SF_SLOT_NNODE = 8,   /* number of internal combine nodes                       */
  SF_SLOT_LEVEL0 = 9,  /* first entry in level_tab                               */
  SF_SLOT_NLEVEL = 10, /* number of levels                                       */
  SF_SLOT_CBASE = 11,  /* prefix sum of nchunk over the preceding rows (this call)*/
  SF_SLOT_BETA1 = 12,  /* f32 pair: beta1 | (1 - beta1) << 32                    */
  SF_SLOT_BETA2 = 13,  /* f32 pair: beta2 | (1 - beta2) << 32                    */
  SF_SLOT_BC = 14,     /* f32 pair: 1 - beta1^t | (1 - beta2^t) << 32            */
  SF_SLOT_EPSWD = 15,  /* f32 pair: eps | weight_decay << 32                     */
  SF_SLOT_LR = 16,     /* f32: lr (low word), AdamW and SGD                      */
  SF_SLOT_WORDS = 17
};
size_t sf_distance_workspace_bytes(int64_t total_chunks, int32_t n_active, int64_t total_nodes);
int sf_layer_distance(const int64_t* slots, int32_t n_active, int64_t total_chunks,
                      const int32_t* chunk_tab, const int32_t* prog_tab, const int32_t* tree_tab,
                      const int32_t* level_tab, int64_t total_nodes, const int32_t* layers,
                      const int64_t* layer_counts, int32_t n_layers, double* d_out, int update,
                      const float* guard, void* ws, void* stream);

/* ---- fused self-attention core with the matsoft8 caches --------------------
 * Replaces, per head, `q @ k^T` (matmul, tensor.py:290-334), softmax with
 * the scale op (tensor.py:413-444) and `probs @ v` (matmul), including the
 * four 8-bit caches those ops store (compression.quantize of q, k^T (stored
 * as k's codes), probs, v; compression.py:66-74), and their backward
 * (decoded operands, SavedValue.get tensor.py:132-135).
 * sf_attention_fwd: y3 = (3, B*T, heads*dh) q/k/v projections without bias
 *   (bq/bk/bv added as the head split does), ctx = (B*T, heads*dh) merged;
 *   q/k/v codes (B, heads, T, dh) int8, p codes (B, heads, T, T) int8 of
 *   the spec Q(8-fb).fb signed.
 * sf_attention_bwd: g = (B*T, heads*dh) merged context gradient; writes
 *   dq | dk | dv side by side into gcat (B*T, 3*heads*dh); `ws` holds
 *   sf_attention_bwd_workspace_bytes(B, T, heads) bytes (0 -- ws may be
 *   NULL -- for the one-head kernels, T <= 128 with T % 4 == 0).
 * Limits: dh == 64, T <= 384 (SF_EINVAL otherwise: the host keeps the
 * unfused ops).  T <= 128 with T % 4 == 0 runs one CTA per head; other T
 * run query-tiled kernels (64 query rows per CTA; backward in two kernels,
 * dq per query tile and dk | dv per key tile). */
int sf_attention_fwd(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                     int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                     void* v_codes, void* p_codes, void* stream);
/* kernel selection (process-wide): 1 = tcgen05 with TMEM accumulators
 * (default): the one-head forward (T <= 128, T % 4 == 0) on two fp16 planes
 * per fp32 operand (22-bit split, two CTAs per SM), its backward and the
 * query-tiled kernels (other T) on exact three-term bf16 splits; 3 = the same
 * with the one-head forward on three bf16 planes; 2 = mma.sync only; 0 =
 * FP32 FMA kernels.  SLIMFIT_ATTN_TC=0 / 2 / 3 in the environment sets it
 * before first use. */
int sf_attention_set_impl(int tensor_cores);
size_t sf_attention_bwd_workspace_bytes(int64_t B, int64_t T, int64_t heads);
int sf_attention_bwd(const float* g, const void* q_codes, const void* k_codes, const void* v_codes,
                     const void* p_codes, int64_t B, int64_t T, int64_t heads, int64_t dh, float scale, int fb,
                     float* gcat, void* ws, void* stream);

/* ---- producers that also write the next GEMM's operand planes ---------------
 * Same as the functions without `_p`, and when the extra `*_planes` pointer
 * is non-NULL the kernel also writes its fp32 output split exactly into three
 * bf16 planes [3][rows][cols] (plane stride = the output's element count;
 * x = hi + mid + lo, bit-identical to sf_split3_bf16), the A operand of the
 * next sf_gemm_split6 product (the layer's input in the forward, the
 * input-gradient product's g in the backward) -- so that product needs no
 * split pass over its A operand.  Planes pointers 8-byte aligned. */
int sf_layernorm_fwd_p(const float* x, const float* gamma, const float* beta, float* y,
                       float* xtilde, float* rstd, int64_t rows, int64_t H, float eps, void* y_planes,
                       void* stream);
int sf_layernorm_fwd_residual_p(const float* res, const float* x, const float* bias, const float* gamma,
                                const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                                int64_t rows, int64_t H, float eps, void* y_planes, void* stream);
int sf_layernorm_bwd_p(const float* g, const float* gamma, const float* xtilde,
                       const float* values, const int32_t* indices, int64_t k,
                       const int32_t* row_ptr, const float* rstd, float* dx, float* dgamma,
                       float* dbeta, int64_t rows, int64_t H, void* ws, void* dx_planes, void* stream);
int sf_gelu_fwd_prescale_bias_p(float* x, const float* bias, int64_t row_len, float* y, int64_t n,
                                double q, float value_max, int32_t* s_dev, void* ws, void* y_planes,
                                void* stream);
int sf_gelu_bwd_packed4_p(const float* g, const uint8_t* packed, const int32_t* s_dev, int fb,
                          float* dx, int64_t n, void* dx_planes, void* stream);
int sf_attention_fwd_p(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                       int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                       void* v_codes, void* p_codes, void* ctx_planes, void* stream);
int sf_attention_bwd_p(const float* g, const void* q_codes, const void* k_codes, const void* v_codes,
                       const void* p_codes, int64_t B, int64_t T, int64_t heads, int64_t dh, float scale, int fb,
                       float* gcat, void* ws, void* gcat_planes, void* stream);
/* The forward producers with the planes' form chosen: planes_format 0 = the
 * three bf16 planes above (the `_p` functions), 1 = the two fp16 planes of
 * sf_split2_f16 ([2][rows][cols], x = hi + 2^-11 lo), the A operand of the
 * next sf_gemm_f16x3 product. */
int sf_layernorm_fwd_pf(const float* x, const float* gamma, const float* beta, float* y,
                        float* xtilde, float* rstd, int64_t rows, int64_t H, float eps, void* y_planes,
                        int planes_format, void* stream);
int sf_layernorm_fwd_residual_pf(const float* res, const float* x, const float* bias, const float* gamma,
                                 const float* beta, float* y, float* sum, float* xtilde, float* rstd,
                                 int64_t rows, int64_t H, float eps, void* y_planes, int planes_format,
                                 void* stream);
/* (y may be NULL when y_planes != NULL: only the next product's planes are
 * written -- the caller's projection is frozen and caches nothing) */
int sf_gelu_fwd_prescale_bias_pf(float* x, const float* bias, int64_t row_len, float* y, int64_t n,
                                 double q, float value_max, int32_t* s_dev, void* ws, void* y_planes,
                                 int planes_format, void* stream);
int sf_attention_fwd_pf(const float* y3, const float* bq, const float* bk, const float* bv, int64_t B, int64_t T,
                        int64_t heads, int64_t dh, float scale, int fb, float* ctx, void* q_codes, void* k_codes,
                        void* v_codes, void* p_codes, void* ctx_planes, int planes_format, void* stream);
/* Backward producers with the planes' form chosen: 0 = three bf16 planes
 * (the `_p` functions), 2 = two fp16 planes scaled per row (as
 * sf_split2_f16_rows: the row's maximum lands in [2^14, 2^15), 2^-e per row
 * into *_row_scale, rows floats), the A operand of the input-gradient
 * sf_gemm_f16x3 product. */
int sf_layernorm_bwd_pf(const float* g, const float* gamma, const float* xtilde,
                        const float* values, const int32_t* indices, int64_t k,
                        const int32_t* row_ptr, const float* rstd, float* dx, float* dgamma,
                        float* dbeta, int64_t rows, int64_t H, void* ws, void* dx_planes, int planes_format,
                        float* dx_row_scale, void* stream);
/* (planes_format 2: dx may be NULL -- only the row-scaled planes are written,
 * for an input-gradient product that is dx's only reader) */
int sf_gelu_bwd_packed4_pf(const float* g, const uint8_t* packed, const int32_t* s_dev, int fb,
                           float* dx, int64_t n, int64_t row_len, void* dx_planes, int planes_format,
                           float* dx_row_scale, void* stream);

/* ---- dense fp32 GEMMs (cuBLASLt) ---------------------------------------------
 * The step's GEMMs: Linear forward/backward (`x @ W + b`, `g @ W^T`,
 * `x^T @ g`; tensor.py:337-379) and the attention score/context batched
 * products (`matmul`, tensor.py:290-334).  The reference computes them in
 * float32 with numpy/OpenBLAS; they are the tensor-core-shaped part of the
 * step and go to cuBLASLt (the toolkit's 12.9 library, opened privately).
 * Row-major: C[b] = op(A[b]) @ op(B[b]) + bias (broadcast over rows, may be
 * NULL) + beta * C[b]; op = transpose when ta/tb.  mode:
 *   SF_GEMM_FP32   strict fp32 (CUBLAS_COMPUTE_32F)
 *   SF_GEMM_BF16X9 fp32 emulated with 3 bf16 terms per operand on the tensor
 *                  cores (CUBLAS_COMPUTE_32F_EMULATED_16BFX9): fp32-accurate
 *   SF_GEMM_TF32   one-pass TF32 (opt-in, not fp32-accurate)
 * workspace: caller-provided device buffer of ws_bytes (32 MiB suffices).
 * Returns SF_EUNAVAILABLE when cuBLASLt or the mode is missing (no fallback).
 */
enum { SF_GEMM_FP32 = 0, SF_GEMM_BF16X9 = 1, SF_GEMM_TF32 = 2 };
int sf_gemm_available(int mode);
size_t sf_gemm_lt_version(void);
int sf_gemm_last_status(void);
const char* sf_gemm_lt_error(void); /* why cuBLASLt did not load ("" when it did) */
int sf_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, int64_t stride_a,
                const float* B, int64_t ldb, int64_t stride_b, float* C, int64_t ldc, int64_t stride_c,
                int64_t batch, const float* bias, float beta, int mode, void* workspace, size_t ws_bytes,
                void* stream);

/* ---- dense fp32 GEMMs on tcgen05 (our kernel, csrc/gemm_tc.cu) ----------------
 * Same products as above (tensor.py:337-379), fp32-accurate from bf16 tensor
 * core MMAs.  sf_split3_bf16 splits x (rows x cols, leading dimension ld)
 * exactly into three bf16 planes x = hi + mid + lo, written [3][rows][cols]
 * or, with transpose, [3][cols][rows] (cols % 4 == 0 and ld % 4 == 0 without
 * transpose).  sf_gemm_split6: C = A @ B^T (+ bias) (+ beta * C) from A planes
 * [3][m][k] and B planes [3][n][k] (both K-major, k % 8 == 0) with the six
 * partial products hh + (hm + mh + mm + hl + lh) in two TMEM accumulators;
 * long reductions / small tile grids run split-K into `ws`
 * (sf_gemm_split6_ws_bytes(m, n, k) bytes, n % 4 == 0 then) and a fixed-order
 * reduce.  Non-finite inputs are not patched (the step skips on a non-finite
 * loss).  sf_gemm_split6_set_stages selects the smem pipeline depth (2..4). */
int sf_split3_bf16(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                   void* stream);
/* As sf_split3_bf16 with an explicit distance (elements) between the three
 * planes (>= rows * cols): room for extra operand rows, e.g. the row of ones
 * that turns the weight-gradient GEMM x^T g into [x^T; 1] g = [dW; db]. */
int sf_split3_bf16_ex(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                      int64_t plane_stride, void* stream);
int64_t sf_gemm_split6_splits(int64_t m, int64_t n, int64_t k);
int64_t sf_gemm_split6_ws_bytes(int64_t m, int64_t n, int64_t k);
int sf_gemm_split6(int64_t m, int64_t n, int64_t k, const void* a_planes, const void* b_planes, float* c,
                   int64_t ldc, const float* bias, float beta, void* ws, int64_t ws_bytes, void* stream);
int sf_gemm_split6_set_stages(int stages);
/* 1 (default): products with beta == 0 (or 1: TMA reduce-add stores) leave
 * the persistent kernels through shared memory and TMA stores (the accumulators return to the MMA issuer
 * after their last tcgen05.ld, the stores drain under the next tile); 0: the
 * threads store C directly. */
int sf_gemm_set_tma_store(int on);
/* f16x3 products with m, n >= 256 on CTA pairs (tcgen05.mma.cta_group::2,
 * M = 256, each SM staging half of B): 1 = 256 x 128 tiles (two accumulator
 * pairs per SM), 2 = 256 x 256 tiles; 0 (default) = single-CTA 128 x 256
 * tiles, measured at least as fast at every step shape.  Same sums. */
int sf_gemm_set_pair(int on);
/* f16x3 form (the forward products, whose operands -- activations and
 * weights -- stay below fp16's 65504): sf_split2_f16 splits x into two fp16
 * planes x = hi + 2^-11 lo (hi = RN_f16(x), lo = RN_f16((x - hi) 2^11)),
 * [2][rows][cols] or transposed [2][cols][rows] (same layout rules as
 * sf_split3_bf16); sf_gemm_f16x3: C = A @ B^T (+ bias) (+ beta * C) from A
 * planes [2][m][k] and B planes [2][n][k] with the three products
 * hh + 2^-11 (hl + lh) in two TMEM accumulators (22-bit operands: error at
 * strict SGEMM's level), same split-K rule and workspace as sf_gemm_split6.
 * |x| >= 65504 overflows hi: the product is non-finite (the step guard then
 * skips the step; SLIMFIT_GEMM_FWD=bf16x6 keeps the three-plane form). */
int sf_split2_f16(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                  void* stream);
int sf_split2_f16_ex(const float* x, int64_t rows, int64_t cols, int64_t ld, int transpose, void* planes,
                     int64_t plane_stride, void* stream);
int sf_gemm_f16x3(int64_t m, int64_t n, int64_t k, const void* a_planes, const float* a_row_scale,
                  const void* b_planes, float* c, int64_t ldc, const float* bias, float beta, void* ws,
                  int64_t ws_bytes, void* stream);
/* Row-scaled split for A operands spanning fp16's range (gradients): row r
 * is split as x 2^e_r, e_r = 15 - ceil-exponent of max|x_r| (the row maximum
 * lands in [2^14, 2^15)), row_scale[r] = 2^-e_r; pass row_scale as
 * sf_gemm_f16x3's a_row_scale (NULL there: unscaled planes). */
int sf_split2_f16_rows(const float* x, int64_t rows, int64_t cols, int64_t ld, void* planes, float* row_scale,
                       void* stream);
/* Batched form (the attention products `matmul`, tensor.py:290-334, at
 * T > 128): planes [3][batch][m][k] and [3][batch][n][k], C entries c_bstride
 * apart (ldc = n), no bias / accumulation / split-K.  sf_split3_bf16_batched:
 * the transposing split of `batch` matrices (rows x cols, ld, x_bstride
 * apart) into planes [3][batch][cols][rows]. */
int sf_gemm_split6_batched(int64_t m, int64_t n, int64_t k, int64_t batch, const void* a_planes,
                           const void* b_planes, float* c, int64_t c_bstride, void* stream);
int sf_split3_bf16_batched(const float* x, int64_t batch, int64_t rows, int64_t cols, int64_t ld,
                           int64_t x_bstride, void* planes, void* stream);
/* Same product with A given as fp32 (row-major m x k, lda % 4 == 0, 16-byte
 * aligned): the kernel splits each TMA-loaded A tile into its planes in
 * shared memory (converter warps), no separate split pass over A. */
int sf_gemm_split6_a32(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda, const void* b_planes,
                       float* c, int64_t ldc, const float* bias, float beta, void* ws, int64_t ws_bytes,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SLIMFIT_B200_H */
