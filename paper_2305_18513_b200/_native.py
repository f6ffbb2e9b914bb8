"""ctypes binding of libslimfit_b200.so (include/slimfit_b200.h).

The product path has no fallback: if the library is missing or fails to load,
every codec/op call raises `NativeUnavailable`.  There is no CPU or eager
PyTorch substitute for the kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CodecError, ShapeError, SlimfitError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLIMFIT_LIB") or os.path.join(_HERE, "libslimfit_b200.so")

SF_OK, SF_EINVAL, SF_ERANGE, SF_ECUDA, SF_EUNAVAILABLE = 0, 1, 2, 3, 4

# int64 words per row of the distance slot table (include/slimfit_b200.h)
SLOT = dict(A=0, B=1, M=2, V=3, N=4, CHUNK0=5, NCHUNK=6, TREE0=7, NNODE=8, LEVEL0=9,
            NLEVEL=10, CBASE=11, BETA1=12, BETA2=13, BC=14, EPSWD=15, LR=16)
SLOT_WORDS = 17
DIST_CHUNK = 4096
UPDATE_NONE, UPDATE_ADAMW, UPDATE_SGD = 0, 1, 2      # sf_layer_distance `update`


class NativeUnavailable(SlimfitError):
    """The CUDA kernel library could not be loaded (no fallback exists)."""


class KernelError(SlimfitError):
    """A CUDA launch or runtime error reported by the kernel library."""


_lock = threading.Lock()
_lib = None

_I64, _I32, _P, _D, _F, _SZ = (ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double,
                               ctypes.c_float, ctypes.c_size_t)
_INT = ctypes.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "sf_abi_version": (_INT, []),
    "sf_last_cuda_error": (_INT, []),
    "sf_strerror": (ctypes.c_char_p, [_INT]),
    "sf_quant8": (_INT, [_P, _P, _I64, _INT, _INT, _P]),
    "sf_quantize": (_INT, [_P, _P, _I64, _INT, _INT, _INT, _P]),
    "sf_quantize_f64": (_INT, [_P, _P, _I64, _INT, _INT, _INT, _P]),
    "sf_dequant8": (_INT, [_P, _P, _I64, _INT, _INT, _P]),
    "sf_prescale_workspace_bytes": (_SZ, [_I64]),
    "sf_prescale_exp": (_INT, [_P, _I64, _D, _F, _P, _P, _P, _P]),
    "sf_quant4_pack": (_INT, [_P, _P, _I64, _P, _INT, _P]),
    "sf_unpack4_dequant": (_INT, [_P, _P, _I64, _P, _INT, _P]),
    "sf_prune_workspace_bytes": (_SZ, [_I64]),
    "sf_prune_topk": (_INT, [_P, _I64, _I64, _INT, _P, _P, _P, _P]),
    "sf_prune_topk_rows": (_INT, [_P, _I64, _I64, _INT, _P, _P, _I64, _P, _P, _P]),
    "sf_prune_hint_bytes": (_SZ, []),
    "sf_prune_topk_hint": (_INT, [_P, _I64, _I64, _INT, _P, _P, _I64, _P, _P, _P, _P]),
    "sf_restore": (_INT, [_P, _P, _I64, _P, _I64, _P]),
    "sf_layernorm_fwd": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P]),
    "sf_layernorm_fwd_residual": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P]),
    "sf_layernorm_bwd_workspace_bytes": (_SZ, [_I64, _I64]),
    "sf_layernorm_bwd": (_INT, [_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _I64, _I64, _P, _P]),
    "sf_gelu_fwd": (_INT, [_P, _P, _I64, _P]),
    "sf_gelu_fwd_prescale": (_INT, [_P, _P, _I64, _D, _F, _P, _P, _P]),
    "sf_gelu_fwd_prescale_bias": (_INT, [_P, _P, _I64, _P, _I64, _D, _F, _P, _P, _P]),
    "sf_split_heads": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _INT, _P]),
    "sf_merge_heads": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _P]),
    "sf_embedding_bwd": (_INT, [_P, _P, _P, _P, _I64, _I64, _P]),
    "sf_embedding_grad_workspace_bytes": (_SZ, [_I64, _I64]),
    "sf_embedding_grad": (_INT, [_P, _I64, _P, _P, _I64, _I64, _P, _P]),
    "sf_merge_heads_ld": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _I64, _P]),
    "sf_gelu_bwd": (_INT, [_P, _P, _P, _I64, _P]),
    "sf_gelu_bwd_packed4": (_INT, [_P, _P, _P, _INT, _P, _I64, _P]),
    "sf_softmax_fwd_q8": (_INT, [_P, _P, _P, _I64, _I64, _F, _INT, _INT, _P]),
    "sf_softmax_bwd_q8": (_INT, [_P, _P, _P, _I64, _I64, _INT, _INT, _F, _P]),
    "sf_distance_workspace_bytes": (_SZ, [_I64, _I32, _I64]),
    "sf_layer_distance": (_INT, [_P, _I32, _I64, _P, _P, _P, _P, _I64, _P, _P, _I32, _P, _INT, _P,
                                 _P, _P]),
    "sf_attention_fwd": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _F, _INT, _P, _P, _P, _P, _P, _P]),
    "sf_attention_set_impl": (_INT, [_INT]),
    "sf_attention_bwd": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _F, _INT, _P, _P, _P]),
    "sf_attention_bwd_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "sf_layernorm_fwd_p": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P, _P]),
    "sf_layernorm_fwd_residual_p": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P, _P]),
    "sf_layernorm_bwd_p": (_INT, [_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P]),
    "sf_gelu_fwd_prescale_bias_p": (_INT, [_P, _P, _I64, _P, _I64, _D, _F, _P, _P, _P, _P]),
    "sf_gelu_bwd_packed4_p": (_INT, [_P, _P, _P, _INT, _P, _I64, _P, _P]),
    "sf_attention_fwd_p": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _F, _INT, _P, _P, _P, _P, _P, _P, _P]),
    "sf_attention_bwd_p": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _F, _INT, _P, _P, _P, _P]),
    "sf_layernorm_fwd_pf": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P, _INT, _P]),
    "sf_layernorm_fwd_residual_pf": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _F, _P, _INT, _P]),
    "sf_gelu_fwd_prescale_bias_pf": (_INT, [_P, _P, _I64, _P, _I64, _D, _F, _P, _P, _P, _INT, _P]),
    "sf_attention_fwd_pf": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _F, _INT, _P, _P, _P, _P, _P, _P, _INT,
                                   _P]),
    "sf_layernorm_bwd_pf": (_INT, [_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _INT, _P, _P]),
    "sf_gelu_bwd_packed4_pf": (_INT, [_P, _P, _P, _INT, _P, _I64, _I64, _P, _INT, _P, _P]),
    "sf_gemm_available": (_INT, [_INT]),
    "sf_gemm_lt_version": (_SZ, []),
    "sf_gemm_last_status": (_INT, []),
    "sf_gemm_lt_error": (ctypes.c_char_p, []),
    "sf_gemm_f32": (_INT, [_INT, _INT, _I64, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64,
                           _I64, _P, _F, _INT, _P, _SZ, _P]),
    "sf_split3_bf16": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _P]),
    "sf_split3_bf16_ex": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _I64, _P]),
    "sf_split3_bf16_batched": (_INT, [_P, _I64, _I64, _I64, _I64, _I64, _P, _P]),
    "sf_gemm_split6_batched": (_INT, [_I64, _I64, _I64, _I64, _P, _P, _P, _I64, _P]),
    "sf_gemm_split6": (_INT, [_I64, _I64, _I64, _P, _P, _P, _I64, _P, _F, _P, _I64, _P]),
    "sf_gemm_f16x3": (_INT, [_I64, _I64, _I64, _P, _P, _P, _P, _I64, _P, _F, _P, _I64, _P]),
    "sf_split2_f16_rows": (_INT, [_P, _I64, _I64, _I64, _P, _P, _P]),
    "sf_gemm_set_tma_store": (_INT, [_INT]),
    "sf_gemm_set_pair": (_INT, [_INT]),
    "sf_restore_rows": (_INT, [_P, _P, _I64, _P, _I64, _P, _I64, _P]),
    "sf_split2_f16": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _P]),
    "sf_split2_f16_ex": (_INT, [_P, _I64, _I64, _I64, _INT, _P, _I64, _P]),
    "sf_gemm_split6_splits": (_I64, [_I64, _I64, _I64]),
    "sf_gemm_split6_a32": (_INT, [_I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _F, _P, _I64, _P]),
    "sf_gemm_split6_ws_bytes": (_I64, [_I64, _I64, _I64]),
    "sf_gemm_split6_set_stages": (_INT, [_INT]),
}


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing; build it with `python -m paper_2305_18513_b200.build` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols(path: str = LIB_PATH):
    """Names from SIGNATURES that the shared object exports (no GPU needed)."""
    lib = ctypes.CDLL(path)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(rc: int, what: str):
    if rc == SF_OK:
        return
    lib = load()
    if rc == SF_ECUDA:
        err = lib.sf_last_cuda_error()
        raise KernelError(f"{what}: CUDA error {err}: {lib.sf_strerror(rc).decode()}")
    if rc == SF_ERANGE:
        raise CodecError(f"{what}: value outside the codec range")
    if rc == SF_EINVAL:
        raise CodecError(f"{what}: invalid argument")
    if rc == SF_EUNAVAILABLE:
        raise NativeUnavailable(f"{what}: required library or mode unavailable "
                                f"(cuBLASLt status {lib.sf_gemm_last_status()})")
    raise KernelError(f"{what}: error code {rc}")


# kernels each entry point launches (main path; tails of unaligned sizes add one)
KERNELS_PER_CALL = {
    "sf_quant8": 1, "sf_quantize": 1, "sf_quantize_f64": 1, "sf_dequant8": 1, "sf_prescale_exp": 3, "sf_quant4_pack": 1,
    "sf_unpack4_dequant": 1, "sf_prune_topk": 1, "sf_prune_topk_rows": 1, "sf_prune_topk_hint": 1, "sf_prune_hint_bytes": 0, "sf_restore": 1, "sf_layernorm_fwd": 1, "sf_layernorm_fwd_residual": 1,
    "sf_gelu_fwd_prescale_bias": 3, "sf_split_heads": 1, "sf_merge_heads": 1, "sf_embedding_grad": 4, "sf_merge_heads_ld": 1,
    "sf_layernorm_bwd": 1, "sf_gelu_fwd": 1, "sf_gelu_fwd_prescale": 3, "sf_gelu_bwd": 1,
    "sf_gelu_bwd_packed4": 1,
    "sf_softmax_fwd_q8": 1, "sf_softmax_bwd_q8": 1, "sf_layer_distance": 2,
    "sf_gemm_f32": 0,     # cuBLASLt's kernels, not ours
    "sf_split3_bf16": 1, "sf_split3_bf16_ex": 1, "sf_split3_bf16_batched": 1, "sf_gemm_split6_batched": 1, "sf_gemm_split6": 1, "sf_gemm_split6_set_stages": 0, "sf_gemm_split6_splits": 0,
    "sf_gemm_split6_ws_bytes": 0, "sf_gemm_split6_a32": 1, "sf_gemm_f16x3": 1, "sf_split2_f16": 1, "sf_split2_f16_rows": 1, "sf_gemm_set_tma_store": 0, "sf_gemm_set_pair": 0, "sf_restore_rows": 1,
    "sf_split2_f16_ex": 1,
}

launch_count = 0          # running total of kernels launched through `call`
call_count: dict = {}
distance_params = 0       # elements in the last sf_layer_distance call (set by DistancePlan)


def _alg_bytes(name, a):
    """Algorithmic HBM bytes of one call (SURVEY.md §8(d) per-element figures)."""
    if name in ("sf_quant8", "sf_quantize", "sf_dequant8"):
        return 5 * a[2]
    if name == "sf_prescale_exp":
        return 4 * a[1]
    if name in ("sf_quant4_pack", "sf_unpack4_dequant"):
        return 4.5 * a[2]
    if name in ("sf_prune_topk", "sf_prune_topk_rows", "sf_prune_topk_hint"):
        return 4 * a[1] + 8 * a[2]
    if name == "sf_restore":
        return 4 * a[4] + 8 * a[2]
    if name == "sf_layernorm_fwd":
        return (12 if a[4] else 8) * a[6] * a[7]
    if name == "sf_layernorm_fwd_residual":      # res + x in, y (+ x~, + sum) out
        return (12 + (4 if a[7] else 0) + (4 if a[6] else 0)) * a[9] * a[10]
    if name == "sf_gelu_fwd_prescale_bias":      # x in, x + b and y out (y NULL: planes only)
        return (12 if a[3] else 8) * a[4]
    if name == "sf_split_heads":
        return (8 + (1 if a[3] else 0)) * a[4] * a[5] * a[6] * a[7]
    if name in ("sf_merge_heads", "sf_merge_heads_ld"):
        return 8 * a[2] * a[3] * a[4] * a[5]
    if name == "sf_layernorm_bwd":
        n = a[11] * a[12]
        return 8 * n + (4 * n if a[2] else 8 * a[5])
    if name in ("sf_gelu_fwd", "sf_gelu_fwd_prescale"):
        return 8 * a[2]
    if name == "sf_gelu_bwd":
        return 12 * a[3]
    if name == "sf_gelu_bwd_packed4":               # g + codes in, dx out (dx NULL: planes only)
        return (8.5 if a[4] else 4.5) * a[5]
    if name in ("sf_softmax_fwd_q8", "sf_softmax_bwd_q8"):
        return 9 * a[3] * a[4]
    if name == "sf_layer_distance":
        return {UPDATE_ADAMW: 28, UPDATE_SGD: 12}.get(a[12], 8) * distance_params
    if name == "sf_attention_fwd":               # flops: 2 products of T x T x dh per head
        return 4.0 * a[4] * a[6] * a[5] * a[5] * a[7]
    if name == "sf_attention_bwd":               # 4 products per head
        return 8.0 * a[5] * a[7] * a[6] * a[6] * a[8]
    if name == "sf_gemm_f32":                   # flops, not bytes: 2 m n k batch
        return 2.0 * a[2] * a[3] * a[4] * a[14]
    if name in ("sf_gemm_split6", "sf_gemm_split6_a32", "sf_gemm_f16x3"):   # fp32 flops of the emulated product: 2 m n k
        return 2.0 * a[0] * a[1] * a[2]
    if name == "sf_gemm_split6_batched":
        return 2.0 * a[0] * a[1] * a[2] * a[3]
    if name == "sf_split3_bf16_batched":
        return 10 * a[1] * a[2] * a[3]
    if name in ("sf_split3_bf16", "sf_split3_bf16_ex"):   # x in, three bf16 planes out
        return 10 * a[1] * a[2]
    if name in ("sf_split2_f16", "sf_split2_f16_ex", "sf_split2_f16_rows"):   # x in, two fp16 planes out
        return 8 * a[1] * a[2]
    return 0


class KernelTimer:
    """Optional CUDA-event timing of every C-ABI call on the launching
    stream (used by bench.py for the live per-kernel roofline)."""

    def __init__(self):
        self.records = []      # (name, alg_bytes, start, end)

    def summary(self):
        import torch
        torch.cuda.synchronize()
        out = {}
        for name, nb, a, b in self.records:
            ms = a.elapsed_time(b)
            s = out.setdefault(name, {"calls": 0, "ms": 0.0, "bytes": 0.0})
            s["calls"] += 1
            s["ms"] += ms
            s["bytes"] += nb
        return out


timer: KernelTimer | None = None


# `_p` producers (they also write the next GEMM's operand planes): position of
# the planes argument and the output's element count, for the kernel table
# (timed under the base name; +6 algorithmic bytes per element when planes
# are written)
_PLANES = {
    "sf_layernorm_fwd_p": (9, lambda a: a[6] * a[7]),
    "sf_layernorm_fwd_residual_p": (12, lambda a: a[9] * a[10]),
    "sf_layernorm_bwd_p": (14, lambda a: a[11] * a[12]),
    "sf_gelu_fwd_prescale_bias_p": (9, lambda a: a[4]),
    "sf_gelu_bwd_packed4_p": (6, lambda a: a[5]),
    "sf_attention_fwd_p": (15, None),            # tensor-bound: flops, not bytes
    "sf_attention_bwd_p": (13, None),
    # `_pf`: planes pointer then the planes' form (0: three bf16 planes, 1: two fp16 planes)
    "sf_layernorm_fwd_pf": (9, lambda a: a[6] * a[7]),
    "sf_layernorm_fwd_residual_pf": (12, lambda a: a[9] * a[10]),
    "sf_gelu_fwd_prescale_bias_pf": (9, lambda a: a[4]),
    "sf_attention_fwd_pf": (15, None),
    "sf_layernorm_bwd_pf": (14, lambda a: a[11] * a[12]),
    "sf_gelu_bwd_packed4_pf": (7, lambda a: a[5]),
}


def _base_name(name: str) -> str:
    return name[:-3] if name.endswith("_pf") else name[:-2]


def call(name: str, *args):
    """Invoke `name` and raise on a non-zero return code."""
    global launch_count
    lib = load()
    if timer is not None:
        import torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        check(getattr(lib, name)(*args), name)
        b.record()
        base, bargs, extra = name, args, 0.0
        if name in _PLANES:
            i, elems = _PLANES[name]
            pf = name.endswith("_pf")
            base, bargs = _base_name(name), args[:i] + args[i + 1 + pf:]
            if args[i] and elems is not None:
                extra = (4.0 if pf and args[i + 1] else 6.0) * elems(args)
        tag = base
        if base == "sf_layernorm_bwd":           # frozen (pruned or dense x~) vs active (with dgamma/dbeta)
            tag = base + (":active" if bargs[9] else (":sparse" if bargs[2] is None else ":dense"))
        timer.records.append((tag, _alg_bytes(base, bargs) + extra, a, b))
    else:
        check(getattr(lib, name)(*args), name)
    launch_count += KERNELS_PER_CALL.get(_base_name(name) if name in _PLANES else name, 1)
    if (name == "sf_gemm_split6" and args[10]) or (name in ("sf_gemm_split6_a32", "sf_gemm_f16x3") and args[11]):  # split-K reduce
        launch_count += 1
    call_count[name] = call_count.get(name, 0) + 1


def shape_error(msg: str):
    return ShapeError(msg)
