"""Dense fp32 GEMMs of the step through `sf_gemm_f32` (cuBLASLt, include/slimfit_b200.h).

The reference computes every product in float32 with numpy/OpenBLAS
(`linear` tensor.py:337-379: `x @ W + b`, `g @ W.T`, `x.T @ g`; `matmul`
tensor.py:290-334: batched `a @ b`).  On B200 these are the only
tensor-core-shaped work of the step.  Four arithmetic modes:

* ``"bf16x6"`` (default on sm_100): our tcgen05 kernel
  (`sf_gemm_split6`, csrc/gemm_tc.cu): each operand split exactly into
  three bf16 planes (`sf_split3_bf16`, transposing where the reduction
  runs along the stored rows), the six partial products that carry fp32
  accuracy in two TMEM accumulators, split-K for long reductions and small
  tile grids.  Error against an fp64 product is at strict SGEMM's level on
  every step shape (tests/test_gemm_gpu.py, tools/tc_gemm_probe.py);
  batched products and unaligned shapes go to cuBLASLt BF16x9;
* ``"bf16x9"`` (cuBLASLt >= 12.9): fp32 emulated on the tensor cores with
  three bf16 terms per operand and nine products;
* ``"fp32"``: strict SIMT SGEMM (CUBLAS_COMPUTE_32F);
* ``"tf32"``: one-pass TF32, opt-in only (not fp32-accurate).

In bf16x6 mode the forward products (`fwd=True`: activations times
weights, operands far below fp16's 65504) run as ``"f16x3"``
(`sf_gemm_f16x3`): two fp16 planes per operand, x = hi + 2^-11 lo (22
significant bits), and the three products hh + 2^-11 (hl + lh) -- half the
MMAs, error at strict SGEMM's level (tests/test_gemm_gpu.py).  The
input-gradient products (`grad_a=True`: g @ W^T) run f16x3 with g's planes
scaled per row (the row maximum in [2^14, 2^15), 2^-e per row applied in the
epilogue: gradients span far more than fp16's range, one row does not);
weight-gradient products keep bf16x6 (their B operand g would need a scale
per column over all tokens).  `SLIMFIT_GEMM_FWD=bf16x6` /
`SLIMFIT_GEMM_DGRAD=bf16x6` keep those products on bf16x6.

`SLIMFIT_GEMM=bf16x6|fp32|bf16x9|tf32` selects the mode process-wide; `set_mode`
changes it.  Operands may be transposed views (k^T of a head-split k,
`W.t()`, `x.t()`): the transpose is folded into the cuBLAS op, never copied.
"""

from __future__ import annotations

import os
import weakref

import torch

from . import _native as N
from .errors import ShapeError

MODES = {"fp32": 0, "bf16x9": 1, "tf32": 2, "bf16x6": 3}
WS_BYTES = 32 << 20

_mode: str | None = os.environ.get("SLIMFIT_GEMM") or None
_ws: dict = {}
_tc_ws: dict = {}          # (device, stream) -> grow-only [a planes, b planes, split-K partials, a row scales]
in_kernel_a_split = os.environ.get("SLIMFIT_GEMM_A32", "0") == "1"   # sf_gemm_split6_a32 for long-K, n <= 768
# batched products (attention at T > 128) on sf_gemm_split6_batched: exact, but
# measured no faster than cuBLASLt SGEMM in the ViT-B / BERT-large steps (the
# split of p and the per-entry epilogue outweigh K = dh = 64 of MMA work;
# profiles/r01_bench_v12_*.json), so opt-in
batched_tc = os.environ.get("SLIMFIT_GEMM_BATCHED", "0") == "1"
# forward products (activations x weights) as f16x3 in bf16x6 mode
fwd_f16 = os.environ.get("SLIMFIT_GEMM_FWD", "f16x3") != "bf16x6"
# input-gradient products (g @ W^T) as f16x3 with row-scaled g in bf16x6 mode
dgrad_f16 = os.environ.get("SLIMFIT_GEMM_DGRAD", "f16x3") != "bf16x6"


def available(mode: str) -> bool:
    if mode == "bf16x6":
        N.load()
        return torch.cuda.is_available() and torch.cuda.get_device_capability() == (10, 0)
    return bool(N.load().sf_gemm_available(MODES[mode]))


def get_mode() -> str:
    """The active arithmetic mode (resolved on first use: bf16x6 on sm_100,
    else bf16x9 if the toolkit cuBLASLt supports it, else strict fp32)."""
    global _mode
    if _mode is None:
        _mode = "bf16x6" if available("bf16x6") else ("bf16x9" if available("bf16x9") else "fp32")
    if _mode not in MODES:
        raise ValueError(f"SLIMFIT_GEMM={_mode!r}: expected one of {sorted(MODES)}")
    return _mode


def set_mode(mode: str) -> None:
    global _mode
    if mode not in MODES:
        raise ValueError(f"gemm mode {mode!r}: expected one of {sorted(MODES)}")
    _mode = mode


def _workspace(device) -> torch.Tensor:
    key = (device.index if device.index is not None else torch.cuda.current_device())
    ws = _ws.get(key)
    if ws is None:
        ws = _ws[key] = torch.empty(WS_BYTES, dtype=torch.uint8, device=device)
    return ws


def _batch_stride(t: torch.Tensor):
    """(count, stride) of the leading (batch) dims collapsed to one
    arithmetic progression, or None when they do not collapse."""
    lead = [(t.shape[i], t.stride(i)) for i in range(t.dim() - 2) if t.shape[i] != 1]
    if not lead:
        return 1, 0
    for (_, st0), (s1, st1) in zip(lead, lead[1:]):
        if st0 != st1 * s1:
            return None
    count = 1
    for s, _ in lead:
        count *= s
    # stride 0 = one matrix broadcast to every batch entry (cuBLAS reads it
    # once per entry; only operands, never the output, are broadcast)
    return count, lead[-1][1]


def _operand(t: torch.Tensor):
    """(tensor, ld, batch, batch_stride, transposed) describing t = op(stored)."""
    r, c = t.shape[-2], t.shape[-1]
    for _ in range(2):
        bs = _batch_stride(t)
        if bs is not None:
            sr, sc = t.stride(-2), t.stride(-1)
            if sc == 1 and (sr >= c or r == 1):
                return t, max(sr, c, 1), bs[0], bs[1], False
            if sr == 1 and (sc >= r or c == 1):
                return t, max(sc, r, 1), bs[0], bs[1], True
        t = t.contiguous()
    raise ShapeError(f"gemm operand with shape {tuple(t.shape)} / strides {t.stride()} is not addressable")


def mm(a: torch.Tensor, b: torch.Tensor, bias: torch.Tensor | None = None,
       out: torch.Tensor | None = None, beta: float = 0.0, mode: str | None = None,
       fwd: bool = False, grad_a: bool = False) -> torch.Tensor:
    """a @ b (+ bias) (+ beta * out) in float32 on the device; a (..., m, k),
    b (..., k, n) with equal (or broadcastable) batch dims.  Returns a new
    contiguous (..., m, n) tensor unless `out` is given; beta != 0 needs
    `out` and accumulates into it (one GEMM epilogue, no separate add).
    `fwd`: a forward product (activation x weight) -- f16x3 in bf16x6 mode;
    `grad_a`: an input-gradient product (gradient x weight^T) -- f16x3 with
    the gradient's planes scaled per row."""
    if a.dtype != torch.float32 or b.dtype != torch.float32:
        raise ShapeError(f"gemm needs float32 operands, got {a.dtype} x {b.dtype}")
    if a.dim() < 2 or b.dim() < 2 or a.shape[-1] != b.shape[-2]:
        raise ShapeError(f"gemm inner dimensions disagree: {tuple(a.shape)} x {tuple(b.shape)}")
    if a.shape[:-2] != b.shape[:-2]:
        try:
            lead = torch.broadcast_shapes(a.shape[:-2], b.shape[:-2])
        except RuntimeError:
            raise ShapeError(f"gemm batch dims disagree: {tuple(a.shape)} x {tuple(b.shape)}") from None
        a = a.expand(*lead, *a.shape[-2:])
        b = b.expand(*lead, *b.shape[-2:])
    _check_planes_only(a)
    m, k, n = a.shape[-2], a.shape[-1], b.shape[-1]
    if bias is not None and (bias.dim() != 1 or bias.shape[0] != n or not bias.is_contiguous()):
        raise ShapeError(f"gemm bias {tuple(bias.shape)} vs {n} columns")
    lead = a.shape[:-2]
    if beta != 0.0 and out is None:
        raise ShapeError("gemm accumulation (beta != 0) needs `out`")
    if out is None:
        out = torch.empty((*lead, m, n), dtype=torch.float32, device=a.device)
    elif tuple(out.shape) != (*lead, m, n) or not out.is_contiguous():
        raise ShapeError(f"gemm out {tuple(out.shape)} vs {(*lead, m, n)}")
    if out.numel() == 0:
        return out
    if k == 0:
        out.mul_(beta) if beta != 0.0 else out.zero_()
        return out if bias is None else out.add_(bias)
    ta_t, lda, batch, sa, ta = _operand(a)
    tb_t, ldb, _, sb, tb = _operand(b)
    mode = mode or get_mode()
    if mode == "bf16x6":
        if (batched_tc and batch > 1 and sa != 0 and sb != 0 and bias is None and beta == 0.0 and k % 8 == 0
                and out.is_contiguous()):
            if _mm_split6_batched(ta_t.data_ptr(), lda, sa, ta, tb_t.data_ptr(), ldb, sb, tb, m, n, k, batch, out):
                return out
        if k % 8 == 0 and n % 4 == 0 and lda % 4 == 0 and ldb % 4 == 0:
            fmt = 1 if (fwd and fwd_f16) else (2 if (grad_a and dgrad_f16 and not ta) else 0)
            if batch == 1:
                return _mm_split6(ta_t.data_ptr(), lda, ta, tb_t.data_ptr(), ldb, tb, m, n, k, bias, out, beta,
                                  fmt=fmt)
            if sa == 0 and out.is_contiguous():
                # one matrix against a batch (the stacked q/k/v weights):
                # split it once, one product per batch entry
                for i in range(batch):
                    _mm_split6(ta_t.data_ptr(), lda, ta, tb_t.data_ptr() + 4 * i * sb, ldb, tb, m, n, k, bias,
                               out.view(batch, m, n)[i], beta, split_a=i == 0, fmt=fmt)
                return out
        mode = "bf16x9"
    if batch > 1 and mode == "bf16x9" and m * n * k < (1 << 28):
        # measured on B200 (tools/gemm_mode_probe.py): cuBLASLt 12.9's
        # emulation runs the attention's small batched products (128x128x64)
        # ~20x slower than SGEMM, so small batched calls stay strict fp32
        mode = "fp32"
    ws = _workspace(a.device)
    N.call("sf_gemm_f32", int(ta), int(tb), m, n, k, ta_t.data_ptr(), lda, sa, tb_t.data_ptr(), ldb, sb,
           out.data_ptr(), n, m * n, batch, bias.data_ptr() if bias is not None else None, float(beta),
           MODES[mode], ws.data_ptr(), WS_BYTES, torch.cuda.current_stream(a.device).cuda_stream)
    return out


def _tc_buffers(device, stream: int, nbytes):
    key = (device.index if device.index is not None else torch.cuda.current_device(), stream)
    bufs = _tc_ws.setdefault(key, [None, None, None, None])
    if len(nbytes) < 4:
        nbytes = (*nbytes, 0)
    for i, nb in enumerate(nbytes):
        if nb and (bufs[i] is None or bufs[i].numel() < nb):
            if i in (0, 3):
                _pending.pop(key, None)      # planes / row scales written into the old buffer are gone
            bufs[i] = None
            bufs[i] = torch.empty(nb, dtype=torch.uint8, device=device)
    return bufs


def _split(ptr: int, ld: int, rows: int, cols: int, transpose: bool, buf: torch.Tensor, stream: int, fmt: int = 0):
    N.call("sf_split2_f16" if fmt else "sf_split3_bf16", ptr, rows, cols, ld, int(transpose), buf.data_ptr(), stream)


# operand plane bytes per element: three bf16 planes (bf16x6) / two fp16 planes
# (f16x3; 2: scaled per row)
_PLANE_BYTES = (6, 4, 4)


# ---- operand planes written by the producing kernel ------------------------
# The A-plane workspace of a (device, stream) can hold the planes of the
# tensor the next product will read as its A operand: the producer (LayerNorm,
# GELU, attention forward/backward, LayerNorm backward, GELU backward) writes
# them next to its fp32 output (the `_p` entry points), and `_mm_split6`
# skips the split pass when the pending planes are exactly its A operand
# (same data pointer and shape, tensor unchanged).  Anything else written
# into the workspace clears the claim, so a product in between only costs
# the split, never a wrong operand.
_pending: dict = {}        # (device index, stream) -> (data_ptr, rows, cols, weakref(tensor), version, fmt)
plane_hits = 0             # splits skipped (diagnostics)
# SLIMFIT_PRODUCER_PLANES=0: producers write no planes, every product splits its A operand
producer_planes = os.environ.get("SLIMFIT_PRODUCER_PLANES", "1") != "0"


def _key(device, stream: int):
    return (device.index if device.index is not None else torch.cuda.current_device(), stream)


def fwd_format() -> int:
    """Planes form a forward producer writes for the next (forward) product:
    1 = two fp16 planes (f16x3), 0 = three bf16 planes (bf16x6)."""
    return 1 if fwd_f16 else 0


def grad_format() -> int:
    """Planes form a backward producer writes for the input-gradient product:
    2 = two fp16 planes scaled per row (f16x3), 0 = three bf16 planes."""
    return 2 if dgrad_f16 else 0


def row_scale_target(t: torch.Tensor):
    """Device pointer for the per-row scales (rows floats) that go with the
    row-scaled planes a backward producer writes at `planes_target(t)`."""
    stream = torch.cuda.current_stream(t.device).cuda_stream
    _, _, _, rs = _tc_buffers(t.device, stream, (0, 0, 0, 4 * (t.numel() // t.shape[-1])))
    return rs.data_ptr()


def planes_target(t: torch.Tensor):
    """Device pointer the producer of `t` may write its A-operand planes to
    (the plane workspace of the current stream), or None when the next
    product would not read planes (not bf16x6, or a shape the tcgen05 path
    does not take).  `t` is (..., cols), contiguous.  The producer then
    writes the form the next product reads (`fwd_format()` for forward
    producers, bf16 planes otherwise) and reports it to `planes_written`."""
    if not producer_planes or not t.is_cuda or t.dim() < 2 or get_mode() != "bf16x6":
        return None
    cols = t.shape[-1]
    if cols % 8 or t.numel() == 0 or not t.is_contiguous():
        return None
    stream = torch.cuda.current_stream(t.device).cuda_stream
    pa = _tc_buffers(t.device, stream, (6 * t.numel(), 0, 0))[0]
    _pending.pop(_key(t.device, stream), None)          # the producer is about to overwrite it
    return pa.data_ptr()


_planes_only: dict = {}    # data_ptr -> weakref(tensor) whose fp32 values were never written


def mark_planes_only(t: torch.Tensor) -> None:
    """`t`'s fp32 values were never written, only its pending planes: the
    next product reading it (any view of it) must claim those planes -- mm
    raises otherwise -- and nothing else may read `t`."""
    _planes_only[t.data_ptr()] = weakref.ref(t)


def _check_planes_only(a: torch.Tensor) -> None:
    ref = _planes_only.pop(a.data_ptr(), None) if _planes_only else None
    if ref is None or ref() is None:
        return
    t = ref()
    stream = torch.cuda.current_stream(a.device).cuda_stream
    ent = _pending.get(_key(a.device, stream))
    ok = (ent is not None and ent[0] == a.data_ptr() and ent[3]() is t and ent[4] == t._version
          and a.dim() == 2 and ent[1] == a.shape[0] and ent[2] == a.shape[1] and a.is_contiguous())
    if not ok:
        raise N.KernelError("a planes-only operand (fp32 values never written) lost its planes before its product")


def planes_written(t: torch.Tensor, fmt: int = 0) -> None:
    """Record that the producer launched after `planes_target(t)` wrote t's
    planes (form `fmt`: 0 three bf16 planes, 1 two fp16 planes)."""
    stream = torch.cuda.current_stream(t.device).cuda_stream
    _pending[_key(t.device, stream)] = (t.data_ptr(), t.numel() // t.shape[-1], t.shape[-1], weakref.ref(t),
                                        t._version, fmt)


def _claim_planes(device, stream: int, at: int, lda: int, m: int, k: int, fmt: int = 0) -> bool:
    ent = _pending.pop(_key(device, stream), None)
    if ent is None:
        return False
    ptr, rows, cols, ref, ver, efmt = ent
    t = ref()
    return (t is not None and t._version == ver and ptr == at and rows == m and cols == k and lda == k
            and efmt == fmt)


_wplanes: dict = {}        # (ptr, ld, n, k, transposed, fmt) -> [weakref(param), version or None (stale), planes]
_wparams: dict = {}        # data_ptr -> weakref(param) of parameters whose planes may be kept


def keep_weight_planes(params) -> None:
    """Keep the bf16 planes of these parameters between products (the
    forward's W and the input gradient's W^T), re-split only after the
    parameter changes: torch in-place ops bump its version counter, and the
    optimizer (which writes through raw pointers) calls
    `weight_planes_changed` for the parameters it stepped."""
    for p in params:
        ptr = p.data_ptr()
        for key in [k for k in _wplanes if k[0] == ptr]:
            del _wplanes[key]
        _wparams[ptr] = weakref.ref(p)


def weight_planes_changed(params=None) -> None:
    """Mark the kept planes of `params` (all when None) stale; their buffers
    are reused by the next split (no allocation inside a step)."""
    ptrs = None if params is None else {p.data_ptr() for p in params}
    for key, ent in _wplanes.items():
        if ptrs is None or key[0] in ptrs:
            ent[1] = None


def _weight_planes(bt, ldb, n, k, tb, stream, fmt=0):
    """Planes [3][n][k] (bf16) / [2][n][k] (fp16, fmt 1) of a kept parameter operand, or None."""
    ref = _wparams.get(bt)
    p = ref() if ref is not None else None
    if p is None or p.data_ptr() != bt:
        return None
    key = (bt, ldb, n, k, tb, fmt)
    ent = _wplanes.get(key)
    if ent is None:
        ent = _wplanes[key] = [ref, None, torch.empty(_PLANE_BYTES[fmt] * n * k, dtype=torch.uint8,
                                                      device=p.device)]
    if ent[1] != p._version:
        if tb:
            _split(bt, ldb, n, k, False, ent[2], stream, fmt)
        else:
            _split(bt, ldb, k, n, True, ent[2], stream, fmt)
        ent[1] = p._version
    return ent[2]


def _mm_split6(at, lda, ta, bt, ldb, tb, m, n, k, bias, out, beta, split_a=True, fmt=0):
    """One `sf_gemm_split6` product: A planes [3][m][k], B planes [3][n][k]
    (both K-major), split from the stored operands (transposing split where
    the stored matrix has the reduction along its rows); fmt 1: the f16x3
    form (`sf_gemm_f16x3`, two fp16 planes per operand)."""
    lib = N.load()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    ws_bytes = lib.sf_gemm_split6_ws_bytes(m, n, k)
    pb_bytes = _PLANE_BYTES[fmt]
    pa, pb, ws, _ = _tc_buffers(out.device, stream, (pb_bytes * m * k, pb_bytes * n * k, ws_bytes))
    global plane_hits
    if fmt:
        rs = None
        if fmt == 2:
            _, _, _, rsb = _tc_buffers(out.device, stream, (0, 0, 0, 4 * m))
            rs = rsb.data_ptr()
        if split_a:
            if not ta and _claim_planes(out.device, stream, at, lda, m, k, fmt):
                plane_hits += 1
            elif fmt == 2:                   # not transposed (mm routes transposed gradients to bf16x6)
                N.call("sf_split2_f16_rows", at, m, k, lda, pa.data_ptr(), rs, stream)
            elif ta:
                _split(at, lda, k, m, True, pa, stream, 1)
            else:
                _split(at, lda, m, k, False, pa, stream, 1)
        wp = _weight_planes(bt, ldb, n, k, tb, stream, 1) if _wparams else None
        if wp is not None:
            pb = wp
        elif tb:
            _split(bt, ldb, n, k, False, pb, stream, 1)
        else:
            _split(bt, ldb, k, n, True, pb, stream, 1)
        N.call("sf_gemm_f16x3", m, n, k, pa.data_ptr(), rs, pb.data_ptr(), out.data_ptr(), n,
               bias.data_ptr() if bias is not None else None, float(beta),
               ws.data_ptr() if ws is not None else None, ws_bytes, stream)
        return out
    # a = op(stored): not transposed -> stored (m, k); transposed -> stored (k, m)
    if in_kernel_a_split and split_a and not ta and n <= 768 and k >= 2048 and lda % 4 == 0 and at % 16 == 0:
        # long reductions into few output tiles: the kernel splits the fp32 A
        # tiles itself (saves the separate pass over A, ~20 us per call on
        # these shapes; the conversion repeats for every N tile of the same A
        # rows).  Off by default: in the step the saving is within noise
        # (GEMM + split 28.4 vs 28.5 ms, profiles/r01_bench_v9.json)
        if tb:
            _split(bt, ldb, n, k, False, pb, stream)
        else:
            _split(bt, ldb, k, n, True, pb, stream)
        N.call("sf_gemm_split6_a32", m, n, k, at, lda, pb.data_ptr(), out.data_ptr(), n,
               bias.data_ptr() if bias is not None else None, float(beta),
               ws.data_ptr() if ws is not None else None, ws_bytes, stream)
        return out
    if split_a:
        if not ta and _claim_planes(out.device, stream, at, lda, m, k):
            plane_hits += 1                  # the producer wrote A's planes: no split pass
        elif ta:
            _split(at, lda, k, m, True, pa, stream)
        else:
            _split(at, lda, m, k, False, pa, stream)
    # b (k, n) = op(stored): transposed -> stored (n, k) as needed; else stored (k, n)
    wp = _weight_planes(bt, ldb, n, k, tb, stream) if _wparams else None
    if wp is not None:
        pb = wp
    elif tb:
        _split(bt, ldb, n, k, False, pb, stream)
    else:
        _split(bt, ldb, k, n, True, pb, stream)
    N.call("sf_gemm_split6", m, n, k, pa.data_ptr(), pb.data_ptr(), out.data_ptr(), n,
           bias.data_ptr() if bias is not None else None, float(beta),
           ws.data_ptr() if ws is not None else None, ws_bytes, stream)
    return out


def mm_wgrad_bias(x: torch.Tensor, g: torch.Tensor, want_db: bool = True):
    """(dW, db) = (x^T g, sum_rows g) of a linear layer (tensor.py:337-379;
    db = g.sum(0)) in ONE bf16x6 product: the A operand is [x^T; 1] -- the
    transposed split of x into planes with room for one more row, that row
    set to exactly 1 (hi = 1, mid = lo = 0) -- so the last output row is
    the column sum of g, and no separate reduction pass over g runs.
    x (tokens, n_in), g (tokens, n_out); other modes / shapes: mm + sum."""
    k, m = x.shape
    n = g.shape[1]
    if (not want_db or get_mode() != "bf16x6" or x.dim() != 2 or g.dim() != 2 or g.shape[0] != k
            or k % 8 or n % 4 or x.stride(1) != 1 or g.stride(1) != 1 or x.stride(0) % 4 or g.stride(0) % 4):
        dW = mm(x.t(), g)
        return dW, (g.sum(dim=0) if want_db else None)
    lib = N.load()
    stream = torch.cuda.current_stream(g.device).cuda_stream
    m1 = m + 1
    ws_bytes = lib.sf_gemm_split6_ws_bytes(m1, n, k)
    pa, pb, ws, _ = _tc_buffers(g.device, stream, (6 * m1 * k, 6 * n * k, ws_bytes))
    _pending.pop(_key(g.device, stream), None)
    N.call("sf_split3_bf16_ex", x.data_ptr(), k, m, x.stride(0), 1, pa.data_ptr(), m1 * k, stream)
    planes = pa[:6 * m1 * k].view(torch.bfloat16).view(3, m1, k)
    planes[0, m].fill_(1.0)
    planes[1:, m].zero_()
    _split(g.data_ptr(), g.stride(0), k, n, True, pb, stream)
    out = torch.empty(m1, n, dtype=torch.float32, device=g.device)
    N.call("sf_gemm_split6", m1, n, k, pa.data_ptr(), pb.data_ptr(), out.data_ptr(), n, None, 0.0,
           ws.data_ptr() if ws is not None else None, ws_bytes, stream)
    return out[:m], out[m]


def _mm_split6_batched(at, lda, sa, ta, bt, ldb, sb, tb, m, n, k, batch, out) -> bool:
    """Batched product (the attention's score / context products at T > 128,
    tensor.py:290-334) on the tcgen05 kernel: planes [3][batch][rows][k]
    (flat split of contiguous K-major entries, batched transposing split
    otherwise), one persistent launch over batch x tiles.  False when the
    layout is not supported (caller falls back to cuBLASLt)."""
    if batch > 65535:
        return False
    if (not ta and (lda != k or sa != m * k)) or (tb and (ldb != k or sb != n * k)):
        return False
    lib = N.load()
    stream = torch.cuda.current_stream(out.device).cuda_stream
    pa, pb, _, _ = _tc_buffers(out.device, stream, (6 * batch * m * k, 6 * batch * n * k, 0))
    _pending.pop(_key(out.device, stream), None)
    if not ta:
        _split(at, k, batch * m, k, False, pa, stream)
    else:      # stored per entry as (k, m)
        N.call("sf_split3_bf16_batched", at, batch, k, m, lda, sa, pa.data_ptr(), stream)
    if tb:     # stored per entry as (n, k)
        _split(bt, k, batch * n, k, False, pb, stream)
    else:
        N.call("sf_split3_bf16_batched", bt, batch, k, n, ldb, sb, pb.data_ptr(), stream)
    N.call("sf_gemm_split6_batched", m, n, k, batch, pa.data_ptr(), pb.data_ptr(), out.data_ptr(), m * n, stream)
    return True
