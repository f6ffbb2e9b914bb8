"""Freeze-aware, codec-aware ops as torch.autograd Functions, plus the
cached-activation ledger — the drop-in for the reference's tensor module
(tensor.py under /root/reference/pkg/src/slimfit).

Each Function saves for backward exactly what the reference op caches
(tensor.py:290-520), encoded by the active `CompressionConfig` through the
sm_100a kernels, and nothing else: the fp32 forward outputs are released as
soon as their consumers have run, so the allocator peak reflects the
reference's caching policy.  Frozen layers (parameters with
requires_grad=False) neither cache their dynamic inputs nor produce weight
gradients — the wgrad GEMM is skipped, not computed and discarded.

The generic plumbing ops of the reference (add, reshape, transpose,
first_token, tanh, cross_entropy, row_slice: tensor.py:523-674) are PyTorch's
own autograd ops; they cache the same things (tanh its output, the loss its
probabilities and labels) and the ledger records them with the reference's
names and byte counts.
"""

from __future__ import annotations

import itertools
import math
import os
import threading
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import _native as N
from . import compression as Cz
from . import gemm as G
from .compression import CompressedActivation, FixedPointSpec, Q2_2, Q4_4
from .errors import ShapeError, SlimfitError

# SLIMFIT_ATTN_TC (csrc/attention.cu attn_impl): 1 tcgen05 (default), 2 mma.sync, 0 FP32 FMA
_ATTN_IMPL = os.environ.get("SLIMFIT_ATTN_TC", "1")[:1] or "1"

SQRT_2_OVER_PI = math.sqrt(2.0 / math.pi)   # tensor.py:27
GELU_CUBIC = 0.044715                       # tensor.py:28


@dataclass
class CompressionConfig:
    """Which cached activations are encoded and how (tensor.py:31-57).

    quant_dense: the 4H-wide FFN output-dense input (8-bit);
    quant_matmul_softmax: attention score/probability operands (8-bit);
    quant_gelu: the GELU input (4-bit packed, power-of-two prescale);
    prune_layernorm: top-k pruning of a frozen LayerNorm's x~ (keep_frac).
    """

    quant_dense: bool = False
    quant_matmul_softmax: bool = False
    quant_gelu: bool = False
    prune_layernorm: bool = False
    keep_frac: float = 0.1
    dense_spec: FixedPointSpec = Q4_4
    matmul_softmax_spec: FixedPointSpec = Q4_4
    gelu_spec: FixedPointSpec = Q2_2
    prune_by_magnitude: bool = True

    @classmethod
    def all_on(cls, **overrides) -> "CompressionConfig":
        kw = dict(quant_dense=True, quant_matmul_softmax=True, quant_gelu=True,
                  prune_layernorm=True)
        kw.update(overrides)
        return cls(**kw)


# --------------------------------------------------------------------------- ledger

_serial = itertools.count()


class SavedValue:
    """One cached activation, raw tensor or CompressedActivation, tagged
    dynamic / static / semi_static (tensor.py:116-141)."""

    __slots__ = ("value", "kind", "name", "_nbytes", "serial", "transposed")

    def __init__(self, value, kind: str, name: str = "", transposed: bool = False):
        self.value = value
        self.kind = kind
        self.name = name
        self.transposed = transposed         # cached as the transpose of what get() returns
        self.serial = next(_serial)          # ledger identity (never reused, unlike id())
        if isinstance(value, CompressedActivation):
            self._nbytes = value.nbytes
        else:
            self._nbytes = int(value.numel() * value.element_size())

    def get(self, dtype=None) -> torch.Tensor:
        if isinstance(self.value, CompressedActivation):
            v = self.value.decompress(dtype or torch.float32)
            return v.transpose(-1, -2) if self.transposed else v
        return self.value

    @property
    def nbytes(self) -> int:
        return self._nbytes


class Tape:
    """Ledger of one recorded iteration (tensor.py:158-191).

    Holds (name, kind, nbytes) records only — never the tensors — so it does
    not extend any buffer's lifetime (a cache whose op will never run
    backward, e.g. a frozen LayerNorm fed only by frozen layers, is freed at
    once but still counted, as the reference's tape counts it).  Distinct
    SavedValue objects are counted separately (the q/k/v inputs count three
    times, as in the reference); one SavedValue registered twice (softmax
    probabilities shared with the context matmul) counts once.
    """

    def __init__(self, compression: CompressionConfig | None = None):
        self.compression = compression
        self._seen: set[int] = set()
        self.records: list[tuple[str, str, int]] = []

    def add_saved(self, sv: SavedValue):
        if sv.serial in self._seen:
            return
        self._seen.add(sv.serial)
        self.records.append((sv.name, sv.kind, sv.nbytes))

    def add_record(self, name: str, kind: str, nbytes: int):
        self.records.append((name, kind, int(nbytes)))

    def cached_bytes(self) -> dict:
        t = {"dynamic": 0, "static": 0, "semi_static": 0}
        for _, kind, b in self.records:
            t[kind] += b
        t["total"] = t["dynamic"] + t["static"] + t["semi_static"]
        return t

    def saved_records(self) -> list:
        return list(self.records)


class _EngineState(threading.local):
    def __init__(self):
        self.tape = None


_state = _EngineState()


class record:
    """Install a fresh Tape (and its CompressionConfig) for one iteration."""

    def __init__(self, compression: CompressionConfig | None = None):
        self.tape = Tape(compression)
        self._prev = None
        self._grad = None

    def __enter__(self) -> Tape:
        self._prev = _state.tape
        _state.tape = self.tape
        self._grad = torch.is_grad_enabled()
        torch.set_grad_enabled(True)
        return self.tape

    def __exit__(self, *exc):
        _state.tape = self._prev
        torch.set_grad_enabled(self._grad)
        return False


class no_grad:
    """Forward-only evaluation: no tape, no autograd graph, nothing cached."""

    def __enter__(self):
        self._prev = _state.tape
        _state.tape = None
        self._ctx = torch.no_grad()
        self._ctx.__enter__()
        return self

    def __exit__(self, *exc):
        _state.tape = self._prev
        self._ctx.__exit__(*exc)
        return False


def current_tape() -> Tape | None:
    return _state.tape


def _recording() -> bool:
    return _state.tape is not None and torch.is_grad_enabled()


def _cfg() -> CompressionConfig | None:
    return _state.tape.compression if _state.tape is not None else None


def _register(sv: SavedValue):
    if _state.tape is not None:
        _state.tape.add_saved(sv)
    return sv


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _save_maybe_quant8(t: torch.Tensor, on: bool, spec, kind: str, name: str) -> SavedValue:
    """tensor.py:280-283: 8-bit codes when the codec slot is on, else raw."""
    if on:
        ca = CompressedActivation.encode_async(lambda: CompressedActivation.quantized(t, spec), t)
        return _register(SavedValue(ca, kind, name))
    return _register(SavedValue(t, kind, name))


# --------------------------------------------------------------------------- linear

class ResidualLink:
    """The residual stream's gradient, handed from the residual LayerNorm's
    backward (`layernorm_residual`, which then returns no gradient for its
    `res` input) to the input-gradient product of the sublayer that reads the
    same tensor (`linear` / `self_attention` with the same link): that GEMM
    accumulates into it in its epilogue (beta = 1, TMA reduce-add) and hands
    the sum on, instead of autograd adding the two gradients in a separate
    pass over (B, T, H).  Autograd runs the LayerNorm's backward first: the
    sublayer's output feeds it."""

    __slots__ = ("g",)

    def __init__(self):
        self.g = None


class _Linear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, quant, spec, name, link=None):
        x2 = x.reshape(-1, x.shape[-1])
        y = G.mm(x2, weight, bias, fwd=True)
        ctx.enabled = weight.requires_grad
        ctx.sv = None
        if ctx.enabled and _state.tape is not None:
            ctx.sv = _save_maybe_quant8(x, quant, spec, "dynamic", f"{name}.input")
        ctx.weight = weight
        ctx.has_bias = bias is not None
        ctx.xshape = x.shape
        ctx.link = link
        return y.reshape(*x.shape[:-1], weight.shape[1])

    @staticmethod
    def backward(ctx, g):
        W = ctx.weight
        g2 = g.reshape(-1, g.shape[-1])
        dx = dW = db = None
        if ctx.needs_input_grad[0]:
            lk = ctx.link
            if lk is not None and lk.g is not None:     # + the residual gradient, in the epilogue
                dx, lk.g = lk.g, None
                G.mm(g2, W.t(), out=dx.view(-1, W.shape[0]), beta=1.0, grad_a=True)
            else:
                dx = G.mm(g2, W.t(), grad_a=True).reshape(ctx.xshape)
        ctx.link = None
        if ctx.sv is not None and (ctx.needs_input_grad[1] or ctx.needs_input_grad[2]):
            xv = ctx.sv.get().reshape(-1, W.shape[0])
            want_db = ctx.has_bias and ctx.needs_input_grad[2]
            if ctx.needs_input_grad[1]:
                dW, db = G.mm_wgrad_bias(xv, g2, want_db)     # db as the GEMM's extra output row
            elif want_db:
                db = g2.sum(dim=0)
        ctx.sv = None
        ctx.weight = None
        return dx, dW, db, None, None, None, None


def linear(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None, *,
           compress: str | None = None, save_name: str = "dense", link: ResidualLink | None = None) -> torch.Tensor:
    """y = x @ W + b; caches x (8-bit when compress="dense8" and the dense codec
    is on) only while W is trainable (tensor.py:337-379)."""
    if x.shape[-1] != weight.shape[0]:
        raise ShapeError(f"linear input width {tuple(x.shape)} vs weight {tuple(weight.shape)}")
    if not _recording():
        x2 = x.reshape(-1, x.shape[-1])
        y = G.mm(x2, weight, bias, fwd=True)
        return y.reshape(*x.shape[:-1], weight.shape[1])
    cfg = _cfg()
    quant = compress == "dense8" and cfg is not None and cfg.quant_dense
    spec = cfg.dense_spec if cfg is not None else None
    return _Linear.apply(x, weight, bias, quant, spec, save_name, link)


# --------------------------------------------------------------------------- attention heads

def _bias_grad(g: torch.Tensor, width: int) -> torch.Tensor:
    return g.reshape(-1, width).sum(dim=0)


class _SplitHeads(torch.autograd.Function):
    """(B, T, h*dh) [+ bias] -> contiguous (B, h, T, dh) in one pass (the
    reference's reshape/transpose after `x @ W + b`, model.py:202-238)."""

    @staticmethod
    def forward(ctx, y, bias, heads):
        B, Tn, H = y.shape
        dh = H // heads
        yc = y.contiguous()
        out = torch.empty((B, heads, Tn, dh), dtype=torch.float32, device=y.device)
        N.call("sf_split_heads", yc.data_ptr(), bias.data_ptr() if bias is not None else None,
               out.data_ptr(), None, B, Tn, heads, dh, 0, 0, _stream())
        ctx.dims = (B, Tn, heads, dh)
        ctx.has_bias = bias is not None
        return out

    @staticmethod
    def backward(ctx, g):
        B, Tn, heads, dh = ctx.dims
        gc = g.contiguous()
        gy = torch.empty((B, Tn, heads * dh), dtype=torch.float32, device=g.device)
        N.call("sf_merge_heads", gc.data_ptr(), gy.data_ptr(), B, Tn, heads, dh, _stream())
        db = _bias_grad(gy, heads * dh) if ctx.has_bias and ctx.needs_input_grad[1] else None
        return gy, db, None


class _MergeHeads(torch.autograd.Function):
    """(B, h, T, dh) -> (B, T, h*dh), the inverse move."""

    @staticmethod
    def forward(ctx, x):
        B, heads, Tn, dh = x.shape
        xc = x.contiguous()
        out = torch.empty((B, Tn, heads * dh), dtype=torch.float32, device=x.device)
        N.call("sf_merge_heads", xc.data_ptr(), out.data_ptr(), B, Tn, heads, dh, _stream())
        ctx.dims = (B, Tn, heads, dh)
        return out

    @staticmethod
    def backward(ctx, g):
        B, Tn, heads, dh = ctx.dims
        gc = g.contiguous()
        gx = torch.empty((B, heads, Tn, dh), dtype=torch.float32, device=g.device)
        N.call("sf_split_heads", gc.data_ptr(), None, gx.data_ptr(), None, B, Tn, heads, dh, 0, 0,
               _stream())
        return gx


def _stacked(ws):
    """(3, H_in, H_out) view over q/k/v weights that live back to back in one
    buffer (Model.build allocates them so), else None."""
    w0 = ws[0]
    step = w0.numel() * w0.element_size()
    if not all(w.is_contiguous() and w.shape == w0.shape and w.dtype == w0.dtype for w in ws):
        return None
    base = w0.untyped_storage().data_ptr()
    if any(w.untyped_storage().data_ptr() != base or w.data_ptr() != w0.data_ptr() + i * step
           for i, w in enumerate(ws)):
        return None       # separate allocations, even if they happen to be adjacent
    return torch.as_strided(w0.detach(), (len(ws), *w0.shape), (w0.numel(), *w0.stride()))


def _qkv_project(x2, ws):
    """(3, M, H) = x2 @ W_i for the three projections: one broadcast-batched
    GEMM over the stacked weights (x read once), else three GEMMs."""
    M, H = x2.shape
    st = _stacked(ws)
    if st is not None:
        return G.mm(x2.expand(len(ws), M, H), st, fwd=True)
    y3 = torch.empty((len(ws), M, ws[0].shape[1]), dtype=torch.float32, device=x2.device)
    for i, w in enumerate(ws):
        G.mm(x2, w, out=y3[i], fwd=True)
    return y3


class _QKV(torch.autograd.Function):
    """The three attention projections of one block with their head split
    (tensor.py:337-379 `linear` x3 + model.py:202-238 reshape/transpose).
    Each projection keeps the reference's caching rule: x is saved for it
    (a separate ledger entry per projection) only while that layer is
    enabled.  Backward merges the three head gradients side by side into one
    (M, 3H) operand: the input gradient is ONE K = 3H GEMM against the
    stacked transposed weights, the weight gradients read column slices of
    it, and the bias gradients are one column reduction."""

    @staticmethod
    def forward(ctx, x, wq, wk, wv, bq, bk, bv, heads, names):
        B, Tn, H = x.shape
        x2 = x.reshape(-1, H)
        ws, bs = (wq, wk, wv), (bq, bk, bv)
        Ho = wq.shape[1]
        dh = Ho // heads
        y3 = _qkv_project(x2, ws)
        outs = []
        for i in range(3):
            o = torch.empty((B, heads, Tn, dh), dtype=torch.float32, device=x.device)
            N.call("sf_split_heads", y3[i].data_ptr(), bs[i].data_ptr() if bs[i] is not None else None,
                   o.data_ptr(), None, B, Tn, heads, dh, 0, 0, _stream())
            outs.append(o)
        del y3
        ctx.enabled = [w.requires_grad for w in ws]
        ctx.sv = [None, None, None]
        if _state.tape is not None:
            ctx.sv = [_register(SavedValue(x, "dynamic", f"{n}.input")) if en else None
                      for en, n in zip(ctx.enabled, names)]
        ctx.ws = ws
        ctx.has_bias = [b is not None for b in bs]
        ctx.dims = (B, Tn, H, heads, dh)
        return tuple(outs)

    @staticmethod
    def backward(ctx, gq, gk, gv):
        B, Tn, H, heads, dh = ctx.dims
        Ho = heads * dh
        M = B * Tn
        dev = ctx.ws[0].device
        gcat = torch.empty((M, 3 * Ho), dtype=torch.float32, device=dev)
        for i, g in enumerate((gq, gk, gv)):
            if g is None:
                gcat[:, i * Ho:(i + 1) * Ho].zero_()
                continue
            gc = g.contiguous()
            N.call("sf_merge_heads_ld", gc.data_ptr(), gcat[:, i * Ho:].data_ptr(), B, Tn, heads, dh,
                   3 * Ho, _stream())
        ctx.sv_x = ctx.sv
        dx, dws, dbs = _qkv_input_grads(ctx, gcat, B, Tn, H, Ho)
        ctx.sv = ctx.sv_x = None
        ctx.ws = None
        return (dx, *dws, *dbs, None, None)


def _qkv_input_grads(ctx, gcat, B, Tn, H, Ho, link=None):
    """dx, dW_q/k/v, db_q/k/v of the three projections from the merged
    (M, 3Ho) head gradient (the shared tail of _QKV / _SelfAttention); with a
    ResidualLink holding the residual gradient, dx accumulates into it."""
    need = ctx.needs_input_grad
    dx = None
    if need[0]:
        st = _stacked(ctx.ws)
        wt = (st.transpose(1, 2).reshape(3 * Ho, H) if st is not None
              else torch.cat([w.detach().t() for w in ctx.ws], dim=0)).contiguous()
        if link is not None and link.g is not None:
            dx, link.g = link.g, None
            G.mm(gcat, wt, out=dx.view(-1, H), beta=1.0, grad_a=True)
        else:
            dx = G.mm(gcat, wt, grad_a=True).reshape(B, Tn, H)
    dws = [None, None, None]
    dbs = [None, None, None]
    if all(need[1 + i] and ctx.sv_x[i] is not None for i in range(3)):
        xs = [ctx.sv_x[i].get().reshape(-1, H) for i in range(3)]
        if xs[0].data_ptr() == xs[1].data_ptr() == xs[2].data_ptr():
            # one input buffer: [dW_q | dW_k | dW_v ; db_q | db_k | db_v] = [x^T; 1] gcat, ONE product
            want_db = all(need[4 + i] and ctx.has_bias[i] for i in range(3))
            dW, db = G.mm_wgrad_bias(xs[0], gcat, want_db)
            for i in range(3):
                dws[i] = dW[:, i * Ho:(i + 1) * Ho].contiguous()
                if want_db:
                    dbs[i] = db[i * Ho:(i + 1) * Ho]
            if want_db or not any(need[4 + i] and ctx.has_bias[i] for i in range(3)):
                return dx, dws, dbs
    for i in range(3):
        if dws[i] is None and need[1 + i] and ctx.sv_x[i] is not None:
            xv = ctx.sv_x[i].get().reshape(-1, H)
            dws[i] = G.mm(xv.t(), gcat[:, i * Ho:(i + 1) * Ho])
    if any(need[4 + i] and ctx.has_bias[i] for i in range(3)):
        colsum = gcat.sum(dim=0)
        for i in range(3):
            if need[4 + i] and ctx.has_bias[i]:
                dbs[i] = colsum[i * Ho:(i + 1) * Ho]
    return dx, dws, dbs


class _SelfAttention(torch.autograd.Function):
    """q/k/v projections + scores + softmax + context of one block with the
    matsoft8 caches (model.py:202-238; tensor.py:290-334, :337-379,
    :413-444): one batched GEMM, then ONE fused kernel per direction
    (csrc/attention.cu).  Caches and ledger entries are exactly the unfused
    ops' (the projection inputs per enabled layer; q, k^T, probs, v as 8-bit
    codes), so the memory accounting is unchanged."""

    @staticmethod
    def forward(ctx, x, wq, wk, wv, bq, bk, bv, heads, scale, spec, names, link=None, planes_only=False):
        B, Tn, H = x.shape
        ctx.link = link
        ws = (wq, wk, wv)
        Ho = wq.shape[1]
        dh = Ho // heads
        dev = x.device
        y3 = _qkv_project(x.reshape(-1, H), ws)
        out = torch.empty((B, Tn, Ho), dtype=torch.float32, device=dev)
        qc = torch.empty((B, heads, Tn, dh), dtype=spec.code_dtype, device=dev)
        kc = torch.empty_like(qc)
        vc = torch.empty_like(qc)
        pc = torch.empty((B, heads, Tn, Tn), dtype=spec.code_dtype, device=dev)
        # the output projection's A operand planes, from the tcgen05 forwards
        # (their context rows leave through shared memory as whole rows; the
        # mma.sync query-tiled kernels' fragment-ordered stores would scatter
        # them)
        tc5 = _ATTN_IMPL == "1" or (_ATTN_IMPL == "2" and Tn <= 128 and Tn % 4 == 0)
        pl = G.planes_target(out) if tc5 else None
        pf = G.fwd_format()
        # planes_only: the output projection is frozen and reads only the
        # context's planes (fp16-plane kernels, impl 1): no fp32 context
        skip = bool(planes_only and pl and _ATTN_IMPL == "1")
        N.call("sf_attention_fwd_pf", y3.data_ptr(), bq.data_ptr(), bk.data_ptr(), bv.data_ptr(), B, Tn, heads,
               dh, float(scale), spec.fb, None if skip else out.data_ptr(), qc.data_ptr(), kc.data_ptr(),
               vc.data_ptr(), pc.data_ptr(), pl, pf, _stream())
        if pl:
            G.planes_written(out, pf)
        if skip:
            G.mark_planes_only(out)
        del y3
        proj, scores, softmax_name, context = names
        ctx.enabled = [w.requires_grad for w in ws]
        ctx.sv_x = [SavedValue(x, "dynamic", f"{n}.input") if en else None for en, n in zip(ctx.enabled, proj)]
        sv_q = SavedValue(CompressedActivation("quant8", qc.shape, spec=spec, codes=qc), "static",
                          f"{scores}.lhs")
        sv_k = SavedValue(CompressedActivation("quant8", kc.shape, spec=spec, codes=kc), "static",
                          f"{scores}.rhs", transposed=True)
        sv_p = SavedValue(CompressedActivation("quant8", pc.shape, spec=spec, codes=pc), "static",
                          f"{softmax_name}.probs")
        sv_v = SavedValue(CompressedActivation("quant8", vc.shape, spec=spec, codes=vc), "static",
                          f"{context}.rhs")
        if _state.tape is not None:          # the unfused ops' registration order
            for sv in ctx.sv_x:
                if sv is not None:
                    _register(sv)
            for sv in (sv_q, sv_k, sv_p, sv_p, sv_v):
                _register(sv)
        ctx.codes = (qc, kc, vc, pc)
        ctx.ws = ws
        ctx.has_bias = [True, True, True]
        ctx.dims = (B, Tn, H, heads, dh, float(scale), spec.fb)
        return out

    @staticmethod
    def backward(ctx, g):
        B, Tn, H, heads, dh, scale, fb = ctx.dims
        Ho = heads * dh
        qc, kc, vc, pc = ctx.codes
        gc = g.contiguous()
        gcat = torch.empty((B * Tn, 3 * Ho), dtype=torch.float32, device=gc.device)
        nws = N.load().sf_attention_bwd_workspace_bytes(B, Tn, heads)
        ws = torch.empty(nws, dtype=torch.uint8, device=gc.device) if nws else None
        # no planes from the backward kernels: their fragment-ordered stores
        # would scatter them (measured slower than the product's own split)
        pl = None
        N.call("sf_attention_bwd_p", gc.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
               B, Tn, heads, dh, scale, fb, gcat.data_ptr(), ws.data_ptr() if ws is not None else None, pl,
               _stream())
        if pl:
            G.planes_written(gcat)
        dx, dws, dbs = _qkv_input_grads(ctx, gcat, B, Tn, H, Ho, ctx.link)
        ctx.codes = ctx.sv_x = ctx.ws = ctx.link = None
        return (dx, *dws, *dbs, None, None, None, None, None, None)


# one fused kernel per direction for the attention core (csrc/attention.cu);
# SLIMFIT_FUSED_ATTN=0 runs the unfused matmul / softmax / matmul ops
_FUSED_ATTN = os.environ.get("SLIMFIT_FUSED_ATTN", "1") != "0"


def fused_attention_ok(x: torch.Tensor, heads: int, width: int) -> bool:
    """The fused kernels' shape limits (csrc/attention.cu): head dim 64,
    T <= 384 (one CTA per head up to T = 128, query-tiled beyond); and the
    matsoft8 codec on (its caches are what the kernels write)."""
    cfg = _cfg()
    if not _FUSED_ATTN or not _recording() or cfg is None or not cfg.quant_matmul_softmax:
        return False
    spec = cfg.matmul_softmax_spec
    Tn = x.shape[1]
    return (x.dim() == 3 and width % heads == 0 and width // heads == 64 and Tn <= 384
            and spec.bits == 8 and spec.signed and x.is_cuda)


def self_attention(x: torch.Tensor, weights, biases, heads: int, scale: float, names,
                   link: ResidualLink | None = None, planes_only: bool = False) -> torch.Tensor:
    """Attention core of one block: returns the merged context (B, T, H)
    before the output projection.  `names` = (projection save names x3,
    scores, softmax, context save names)."""
    proj, scores, softmax_name, context = names
    spec = _cfg().matmul_softmax_spec
    return _SelfAttention.apply(x, *weights, *biases, heads, scale, spec,
                                (tuple(proj), scores, softmax_name, context), link, planes_only)


def qkv_heads(x: torch.Tensor, weights, biases, heads: int, save_names=("query", "key", "value")):
    """q, k, v = split_heads(linear(x, W_i), b_i) for the three projections,
    with the reference's per-projection caching (see _QKV)."""
    wq, wk, wv = weights
    bq, bk, bv = biases
    if x.dim() != 3 or any(w.shape[0] != x.shape[-1] for w in weights):
        raise ShapeError(f"qkv input {tuple(x.shape)} vs weights {[tuple(w.shape) for w in weights]}")
    Ho = wq.shape[1]
    if wk.shape[1] != Ho or wv.shape[1] != Ho or Ho % heads or (Ho // heads) % 4:
        raise ShapeError(f"cannot split projections of width {Ho} into {heads} heads")
    if not _recording():
        B, Tn, H = x.shape
        y3 = _qkv_project(x.reshape(-1, H), weights)
        return tuple(split_heads(y3[i].reshape(B, Tn, Ho), biases[i], heads) for i in range(3))
    return _QKV.apply(x, wq, wk, wv, bq, bk, bv, heads, tuple(save_names))


def split_heads(y: torch.Tensor, bias: torch.Tensor | None, heads: int) -> torch.Tensor:
    """(B, T, H) projection output (bias not yet added) -> (B, h, T, H/h)."""
    if y.dim() != 3 or y.shape[-1] % heads or (y.shape[-1] // heads) % 4:
        raise ShapeError(f"cannot split {tuple(y.shape)} into {heads} heads")
    if bias is not None and tuple(bias.shape) != (y.shape[-1],):
        raise ShapeError(f"bias {tuple(bias.shape)} vs width {y.shape[-1]}")
    return _SplitHeads.apply(y, bias, heads)


def merge_heads(x: torch.Tensor) -> torch.Tensor:
    """(B, h, T, dh) -> (B, T, h*dh)."""
    if x.dim() != 4 or x.shape[-1] % 4:
        raise ShapeError(f"cannot merge heads of {tuple(x.shape)}")
    return _MergeHeads.apply(x)


# --------------------------------------------------------------------------- matmul / softmax

class _Matmul(torch.autograd.Function):
    @staticmethod
    def forward(ctx, a, b, sv_a, sv_b):
        ctx.sv = (sv_a, sv_b)
        return G.mm(a, b)

    @staticmethod
    def backward(ctx, g):
        sv_a, sv_b = ctx.sv
        ga = gb = None
        if ctx.needs_input_grad[0]:
            ga = G.mm(g, sv_b.get().transpose(-1, -2))
        if ctx.needs_input_grad[1]:
            gb = G.mm(sv_a.get().transpose(-1, -2), g)
        ctx.sv = None
        return ga, gb, None, None


def matmul(a: torch.Tensor, b: torch.Tensor, *, compress: str | None = None,
           save_name: str = "matmul") -> torch.Tensor:
    """Batched a @ b caching both operands (8-bit with compress="matsoft8");
    an operand produced by `softmax` reuses the softmax's cached buffer
    instead of caching a second copy (tensor.py:290-334)."""
    if a.dim() < 1 or b.dim() < 1 or a.shape[-1] != b.shape[-2 if b.dim() > 1 else 0]:
        raise ShapeError(f"matmul inner dimensions disagree: {tuple(a.shape)} x {tuple(b.shape)}")
    cfg = _cfg()
    quant = compress == "matsoft8" and cfg is not None and cfg.quant_matmul_softmax
    spec = cfg.matmul_softmax_spec if cfg is not None else None

    def side(t, tag):
        shared = getattr(t, "_slimfit_shared", None)
        if shared is not None:
            _register(shared)
            return shared
        if quant and t.dim() >= 2 and not t.is_contiguous() and t.transpose(-1, -2).is_contiguous():
            # k^T of a head-split k: encode k itself (same codes, no transposing copy)
            tt = t.transpose(-1, -2)
            ca = CompressedActivation.encode_async(lambda: CompressedActivation.quantized(tt, spec), tt)
            return _register(SavedValue(ca, "static", f"{save_name}.{tag}", transposed=True))
        return _save_maybe_quant8(t, quant, spec, "static", f"{save_name}.{tag}")

    if not _recording():
        return G.mm(a, b)
    return _Matmul.apply(a, b, side(a, "lhs"), side(b, "rhs"))


class _Softmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, s, scale, quant, spec, name, box):
        rows, W = s.numel() // s.shape[-1], s.shape[-1]
        sc = s.contiguous()
        probs = torch.empty_like(sc)
        if quant:
            codes = torch.empty(sc.shape, dtype=spec.code_dtype, device=sc.device)
            N.call("sf_softmax_fwd_q8", sc.data_ptr(), probs.data_ptr(), codes.data_ptr(), rows, W,
                   float(scale), spec.fb, int(spec.signed), _stream())
            sv = SavedValue(CompressedActivation("quant8", sc.shape, spec=spec, codes=codes),
                            "static", f"{name}.probs")
        else:
            x = sc if scale == 1.0 else sc * torch.tensor(scale, dtype=sc.dtype, device=sc.device)
            torch.softmax(x, dim=-1, out=probs)
            sv = SavedValue(probs, "static", f"{name}.probs")
        ctx.sv = _register(sv) if _state.tape is not None else sv
        ctx.scale = scale
        ctx.quant = quant
        ctx.spec = spec
        box.append(ctx.sv)
        return probs

    @staticmethod
    def backward(ctx, g):
        sv = ctx.sv
        W = g.shape[-1]
        if ctx.quant:
            gc = g.contiguous()
            ds = torch.empty_like(gc)
            N.call("sf_softmax_bwd_q8", gc.data_ptr(), sv.value.codes.data_ptr(), ds.data_ptr(),
                   gc.numel() // W, W, ctx.spec.fb, int(ctx.spec.signed), float(ctx.scale), _stream())
        else:
            p = sv.get()
            ds = p * (g - (g * p).sum(dim=-1, keepdim=True))
            if ctx.scale != 1.0:
                ds = ds * torch.tensor(ctx.scale, dtype=ds.dtype, device=ds.device)
        ctx.sv = None
        return ds, None, None, None, None, None


def softmax(x: torch.Tensor, axis: int = -1, *, compress: str | None = None,
            save_name: str = "softmax", scale: float = 1.0) -> torch.Tensor:
    """Shift-by-max softmax over the last axis of (x * scale), caching its
    output (8-bit with compress="matsoft8"); a downstream `matmul` shares that
    cached buffer (tensor.py:413-444).  `scale` folds the reference's
    preceding scale op (tensor.py:583-593) into the same kernel."""
    if axis not in (-1, x.dim() - 1):
        raise ShapeError(f"softmax over axis {axis} of shape {tuple(x.shape)}: only the last axis")
    cfg = _cfg()
    quant = compress == "matsoft8" and cfg is not None and cfg.quant_matmul_softmax
    spec = cfg.matmul_softmax_spec if cfg is not None else None
    scale = float(torch.tensor(scale, dtype=torch.float32).item())    # f32(c), tensor.py:585
    if not _recording():
        xs = x if scale == 1.0 else x * scale
        return torch.softmax(xs, dim=-1)
    box = []
    out = _Softmax.apply(x, scale, quant, spec, save_name, box)
    out._slimfit_shared = box[0]
    return out


# --------------------------------------------------------------------------- GELU

def _pack4(xc, s, spec) -> CompressedActivation:
    """K4 with the prescale exponent already on the device."""
    n = xc.numel()
    out = torch.empty((n + 1) // 2, dtype=torch.uint8, device=xc.device)
    N.call("sf_quant4_pack", xc.data_ptr(), out.data_ptr(), n, s.data_ptr(), spec.fb, _stream())
    return CompressedActivation("packed4", xc.shape, spec=spec, packed=out, count=n, prescale_exp_dev=s)


class _Gelu(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, packed, spec, name, bias=None, planes_only=False, bwd_planes_only=False):
        ctx.has_bias = bias is not None
        ctx.bwd_planes_only = bwd_planes_only
        fuse = bias is not None and packed and x.numel() and x.is_contiguous()
        if bias is not None and not fuse:
            x = x + bias                          # unfused fallback: x @ W + b first
        xc = x.contiguous()
        y = torch.empty_like(xc)
        n = xc.numel()
        if fuse:
            # the GEMM output gets its bias in place during the same read that
            # computes GELU and the K3 histogram; K4 then packs x + b
            s = torch.zeros(1, dtype=torch.int32, device=xc.device)
            ws = torch.empty(N.load().sf_prescale_workspace_bytes(n), dtype=torch.uint8,
                             device=xc.device)
            pl = G.planes_target(y)               # the next projection's A operand planes
            pf = G.fwd_format()
            # planes_only: the next projection is frozen (caches nothing) and
            # reads only the planes, so the fp32 y is not written at all
            skip_y = bool(planes_only and pl)
            N.call("sf_gelu_fwd_prescale_bias_pf", xc.data_ptr(), bias.data_ptr(), xc.shape[-1],
                   None if skip_y else y.data_ptr(), n, Cz._quantile(99.9), float(spec.value_max), s.data_ptr(),
                   ws.data_ptr(), pl, pf, _stream())
            if pl:
                G.planes_written(y, pf)
            if skip_y:
                G.mark_planes_only(y)
            ca = CompressedActivation.encode_async(lambda: _pack4(xc, s, spec), xc, s)
            sv = SavedValue(ca, "static", f"{name}.input")
        elif packed and n:
            # one read of x: GELU forward + K3 histogram, then K4 packs x
            s = torch.zeros(1, dtype=torch.int32, device=xc.device)
            ws = torch.empty(N.load().sf_prescale_workspace_bytes(n), dtype=torch.uint8,
                             device=xc.device)
            N.call("sf_gelu_fwd_prescale", xc.data_ptr(), y.data_ptr(), n, Cz._quantile(99.9),
                   float(spec.value_max), s.data_ptr(), ws.data_ptr(), _stream())
            ca = CompressedActivation.encode_async(lambda: _pack4(xc, s, spec), xc, s)
            sv = SavedValue(ca, "static", f"{name}.input")
        elif packed:
            N.call("sf_gelu_fwd", xc.data_ptr(), y.data_ptr(), n, _stream())
            sv = SavedValue(CompressedActivation.packed(xc, spec), "static", f"{name}.input")
        else:
            N.call("sf_gelu_fwd", xc.data_ptr(), y.data_ptr(), n, _stream())
            sv = SavedValue(xc, "static", f"{name}.input")
        ctx.sv = _register(sv) if _state.tape is not None else sv
        return y

    @staticmethod
    def backward(ctx, g):
        sv = ctx.sv
        gc = g.contiguous()
        dx = torch.empty_like(gc)
        if isinstance(sv.value, CompressedActivation):
            ca = sv.value.wait()
            pl = G.planes_target(dx)              # the projection's input-gradient A operand
            pf = G.grad_format() if gc.shape[-1] <= 4096 else 0
            rsc = G.row_scale_target(dx) if pl and pf == 2 else None
            # the projection feeding this GELU is frozen (no weight or bias
            # gradient): its input-gradient product is dx's only reader
            skip_dx = bool(ctx.bwd_planes_only and pl and pf == 2 and not ctx.needs_input_grad[4])
            N.call("sf_gelu_bwd_packed4_pf", gc.data_ptr(), ca.packed_codes.data_ptr(),
                   ca.prescale_exp_dev.data_ptr(), ca.spec.fb, None if skip_dx else dx.data_ptr(), gc.numel(),
                   gc.shape[-1], pl, pf, rsc, _stream())
            if pl:
                G.planes_written(dx, pf)
            if skip_dx:
                G.mark_planes_only(dx)
        else:
            N.call("sf_gelu_bwd", gc.data_ptr(), sv.value.data_ptr(), dx.data_ptr(), gc.numel(),
                   _stream())
        ctx.sv = None
        db = _bias_grad(dx, dx.shape[-1]) if ctx.has_bias and ctx.needs_input_grad[4] else None
        return dx, None, None, None, db, None, None


def gelu(x: torch.Tensor, *, bias: torch.Tensor | None = None, save_name: str = "gelu",
         planes_only: bool = False, bwd_planes_only: bool = False) -> torch.Tensor:
    """tanh-form GELU of x (+ bias: the preceding projection's bias, fused
    here instead of in the GEMM) caching its input, 4-bit packed when the
    GELU codec is on (tensor.py:382-410).  planes_only: the caller's next
    use of the result is ONE frozen projection (no cache of its input), so
    on the fused path only that product's operand planes are written and the
    fp32 result is left unwritten (the product refuses it otherwise).
    bwd_planes_only: likewise for the input gradient, whose one reader is
    the input-gradient product of a frozen projection feeding x (no weight
    or bias gradient)."""
    cfg = _cfg()
    packed = cfg is not None and cfg.quant_gelu
    if bias is not None and tuple(bias.shape) != (x.shape[-1],):
        raise ShapeError(f"bias {tuple(bias.shape)} vs width {x.shape[-1]}")
    if not _recording():
        xb = (x + bias) if bias is not None else x
        xb = xb.contiguous()
        y = torch.empty_like(xb)
        N.call("sf_gelu_fwd", xb.data_ptr(), y.data_ptr(), xb.numel(), _stream())
        return y
    return _Gelu.apply(x, packed, cfg.gelu_spec if cfg is not None else None, save_name, bias, planes_only,
                       bwd_planes_only)


# --------------------------------------------------------------------------- LayerNorm

# per-site prune hints (frozen LayerNorm x~): the previous call's threshold
# at the same site brackets the next one (speed only, never the result)
_PRUNE_HINTS: dict = {}
_PRUNE_HINT_ON = os.environ.get("SLIMFIT_PRUNE_HINT", "1") != "0"


def _prune_hint(name, device):
    if not _PRUNE_HINT_ON:
        return None
    key = (name, str(device))
    h = _PRUNE_HINTS.get(key)
    if h is None:
        h = _PRUNE_HINTS[key] = Cz.new_prune_hint(device)
    return h


class _LayerNorm(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gamma, beta, eps, prune, keep_frac, by_mag, name, res=None, bias=None, link=None):
        H = x.shape[-1]
        xc = x.contiguous()
        rows = xc.numel() // H
        y = torch.empty_like(xc)
        rstd = torch.empty(xc.shape[:-1] + (1,), dtype=torch.float32, device=xc.device)
        xt = torch.empty_like(xc)
        ctx.fused = res is not None
        ctx.link = link
        enabled = gamma.requires_grad
        pruning = not enabled and prune
        pl = G.planes_target(y)                   # the next projection's A operand planes
        pf = G.fwd_format()
        if res is None:
            N.call("sf_layernorm_fwd_pf", xc.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
                   xt.data_ptr(), rstd.data_ptr(), rows, H, float(eps), pl, pf, _stream())
        else:                                     # LN(res + (x + bias)) in one pass
            rc = res.contiguous()
            N.call("sf_layernorm_fwd_residual_pf", rc.data_ptr(), xc.data_ptr(), bias.data_ptr(),
                   gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), None, xt.data_ptr(),
                   rstd.data_ptr(), rows, H, float(eps), pl, pf, _stream())
        if pl:
            G.planes_written(y, pf)
        if pruning:
            ca = CompressedActivation.encode_async(
                lambda: CompressedActivation("pruned", xt.shape, sparse=Cz.prune_topk(
                    xt, keep_frac, by_mag, row_pointers=True, hint=_prune_hint(name, xt.device))), xt)
            sv_xt = SavedValue(ca, "semi_static", f"{name}.xtilde")
            del xt
        else:
            sv_xt = SavedValue(xt, "semi_static", f"{name}.xtilde")
        return _LayerNorm._finish(ctx, y, sv_xt, rstd, gamma, enabled, name)

    @staticmethod
    def _finish(ctx, y, sv_xt, rstd, gamma, enabled, name):
        sv_r = SavedValue(rstd, "static", f"{name}.rstd")
        if _state.tape is not None:
            _register(sv_xt)
            _register(sv_r)
        ctx.sv = (sv_xt, sv_r)
        ctx.gamma = gamma
        ctx.enabled = enabled
        return y

    @staticmethod
    def backward(ctx, g):
        sv_xt, sv_r = ctx.sv
        gamma = ctx.gamma
        H = g.shape[-1]
        gc = g.contiguous()
        rows = gc.numel() // H
        dx = torch.empty_like(gc)
        want = ctx.enabled and (ctx.needs_input_grad[1] or ctx.needs_input_grad[2])
        dgamma = torch.empty_like(gamma) if want else None
        dbeta = torch.empty_like(gamma) if want else None
        ws = torch.empty(max(1, N.load().sf_layernorm_bwd_workspace_bytes(rows, H)),
                         dtype=torch.uint8, device=g.device)
        v = sv_xt.value
        pl = G.planes_target(dx)                  # the upstream projection's input-gradient A operand
        pf = G.grad_format()
        rsc = G.row_scale_target(dx) if pl and pf == 2 else None
        if isinstance(v, CompressedActivation):      # pruned x~, consumed sparse (fused K7)
            sp = v.wait().sparse
            N.call("sf_layernorm_bwd_pf", gc.data_ptr(), gamma.data_ptr(), None, sp.values.data_ptr(),
                   sp.indices.data_ptr(), sp.values.numel(),
                   sp.row_ptr.data_ptr() if sp.row_ptr is not None else None,
                   sv_r.value.data_ptr(), dx.data_ptr(),
                   None, None, rows, H, ws.data_ptr(), pl, pf, rsc, _stream())
        else:
            N.call("sf_layernorm_bwd_pf", gc.data_ptr(), gamma.data_ptr(), v.data_ptr(), None, None, 0,
                   None, sv_r.value.data_ptr(), dx.data_ptr(),
                   dgamma.data_ptr() if want else None, dbeta.data_ptr() if want else None,
                   rows, H, ws.data_ptr(), pl, pf, rsc, _stream())
        if pl:
            G.planes_written(dx, pf)
        ctx.sv = None
        ctx.gamma = None
        if not ctx.fused:
            return dx, dgamma, dbeta, None, None, None, None, None, None, None, None
        db = _bias_grad(dx, H) if ctx.needs_input_grad[9] else None
        dres = dx
        if ctx.link is not None and ctx.needs_input_grad[8]:
            # the sublayer reading `res` adds its input gradient into this one
            # (ResidualLink); its backward runs after this one
            ctx.link.g, dres = dx, None
        ctx.link = None
        return dx, dgamma, dbeta, None, None, None, None, None, dres, db, None


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5, *,
              save_name: str = "layernorm") -> torch.Tensor:
    """LayerNorm over the last axis caching x~ (semi-static: top-k pruned
    while the layer is frozen and the prune codec is on) and rstd
    (tensor.py:447-494)."""
    H = x.shape[-1]
    if tuple(gamma.shape) != (H,) or tuple(beta.shape) != (H,):
        raise ShapeError(f"layernorm affine shape {tuple(gamma.shape)} vs last axis {H}")
    cfg = _cfg()
    prune = cfg is not None and cfg.prune_layernorm
    keep = cfg.keep_frac if cfg is not None else 0.1
    mag = cfg.prune_by_magnitude if cfg is not None else True
    if not _recording():
        xc = x.contiguous()
        y = torch.empty_like(xc)
        rstd = torch.empty(xc.numel() // H, dtype=torch.float32, device=xc.device)
        N.call("sf_layernorm_fwd", xc.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(),
               None, rstd.data_ptr(), xc.numel() // H, H, float(eps), _stream())
        return y
    return _LayerNorm.apply(x, gamma, beta, eps, prune, keep, mag, save_name)


def layernorm_residual(res: torch.Tensor, x: torch.Tensor, bias: torch.Tensor, gamma: torch.Tensor,
                       beta: torch.Tensor, eps: float = 1e-5, *,
                       save_name: str = "layernorm", link: ResidualLink | None = None) -> torch.Tensor:
    """layernorm(res + (x + bias)): the post-norm residual add after a
    projection whose bias was left out of the GEMM, fused into the LayerNorm
    pass (same caches and ledger records as `layernorm` of the sum)."""
    H = x.shape[-1]
    if tuple(gamma.shape) != (H,) or tuple(beta.shape) != (H,) or tuple(bias.shape) != (H,):
        raise ShapeError(f"layernorm affine/bias shapes vs last axis {H}")
    if tuple(res.shape) != tuple(x.shape):
        raise ShapeError(f"residual {tuple(res.shape)} vs {tuple(x.shape)}")
    if not _recording():
        return layernorm(res + (x + bias), gamma, beta, eps, save_name=save_name)
    cfg = _cfg()
    prune = cfg is not None and cfg.prune_layernorm
    keep = cfg.keep_frac if cfg is not None else 0.1
    mag = cfg.prune_by_magnitude if cfg is not None else True
    return _LayerNorm.apply(x, gamma, beta, eps, prune, keep, mag, save_name, res, bias, link)


# --------------------------------------------------------------------------- embedding

class _Embedding(torch.autograd.Function):
    """Row lookup whose table gradient is accumulated in position order
    (np.add.at, tensor.py:497-520) by sf_embedding_bwd, without the host
    synchronisation torch's embedding backward needs to count unique ids."""

    @staticmethod
    def forward(ctx, table, ids):
        ctx.ids = ids
        ctx.shape = table.shape
        return F.embedding(ids, table)

    @staticmethod
    def backward(ctx, g):
        V, H = ctx.shape
        ids = ctx.ids.reshape(-1).long().contiguous()
        gc = g.reshape(-1, H).contiguous()
        n = ids.numel()
        ws = torch.empty(N.load().sf_embedding_grad_workspace_bytes(n, V), dtype=torch.uint8, device=g.device)
        dw = torch.empty((V, H), dtype=torch.float32, device=g.device)
        N.call("sf_embedding_grad", ids.data_ptr(), n, gc.data_ptr(), dw.data_ptr(), V, H, ws.data_ptr(),
               _stream())
        ctx.ids = None
        return dw, None


def embedding(table: torch.Tensor, ids: torch.Tensor, *, save_name: str = "embedding") -> torch.Tensor:
    """Row lookup; the ids are cached (int32, dynamic) only while the table
    is trainable (tensor.py:497-520)."""
    # range is validated on the host before upload (Model.forward); a device
    # tensor is trusted here to avoid a host sync per step
    if _recording() and table.requires_grad:
        _state.tape.add_record(f"{save_name}.ids", "dynamic", ids.numel() * 4)
        if table.shape[1] % 4 == 0 and table.shape[1] <= 1024 and table.is_cuda:
            return _Embedding.apply(table, ids)
    return F.embedding(ids, table)


def record_static(name: str, nbytes: int):
    """Ledger entry for a buffer cached by a native PyTorch op (tanh output,
    loss probabilities/labels: tensor.py:642, :665-666)."""
    if _recording():
        _state.tape.add_record(name, "static", nbytes)


def cross_entropy(logits: torch.Tensor, labels: torch.Tensor, *, save_name: str = "loss") -> torch.Tensor:
    """Mean cross-entropy (tensor.py:651-674)."""
    if logits.dim() != 2 or tuple(labels.shape) != (logits.shape[0],):
        raise ShapeError(f"cross_entropy logits {tuple(logits.shape)} vs labels {tuple(labels.shape)}")
    record_static(f"{save_name}.probs", logits.numel() * 4)
    record_static(f"{save_name}.labels", labels.numel() * 4)
    return F.cross_entropy(logits, labels.long())


def backward(loss: torch.Tensor):
    """Reverse sweep from a scalar loss (tensor.py:681-713)."""
    if loss.numel() != 1:
        raise SlimfitError(f"backward requires a scalar loss, got shape {tuple(loss.shape)}")
    if loss.grad_fn is None:
        return
    loss.backward()
