"""Activation codecs on device tensors — the drop-in for the reference's
compression module (compression.py:1-257 under /root/reference/pkg/src/slimfit).

Same names, same argument meaning, same errors (CodecError); the difference
is where the bytes live: inputs are moved to the current CUDA device if they
are not there already, payloads stay in HBM, and every transform is one of
the sm_100a kernels of libslimfit_b200.so.  There is no CPU path.

Bit-exactness contract (checked by tests/test_codecs_gpu.py against the
oracle and the reference's golden vectors): quantized codes, packed bytes,
prescale exponents, pruned indices and values are identical to the
reference's for identical float32 inputs.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import streams as S
from .errors import CodecError

PERCENTILE_Q = {}   # pct -> numpy's float64 quantile (np.true_divide(pct, 100))


# --------------------------------------------------------------------------- specs

@dataclass(frozen=True)
class FixedPointSpec:
    """Signed or unsigned fixed point with `ib` integer and `fb` fraction bits
    (reference compression.py:21-53); total width must be 4 or 8."""

    ib: int
    fb: int
    signed: bool = True

    def __post_init__(self):
        if self.ib + self.fb not in (4, 8):
            raise CodecError(f"total bit width must be 4 or 8, got {self.ib + self.fb}")
        if self.ib < 0 or self.fb < 0:
            raise CodecError("bit counts must be nonnegative")

    @property
    def bits(self) -> int:
        return self.ib + self.fb

    @property
    def code_min(self) -> int:
        return -(1 << (self.bits - 1)) if self.signed else 0

    @property
    def code_max(self) -> int:
        return (1 << (self.bits - 1)) - 1 if self.signed else (1 << self.bits) - 1

    @property
    def value_min(self) -> float:
        return self.code_min / (1 << self.fb)

    @property
    def value_max(self) -> float:
        return self.code_max / (1 << self.fb)

    @property
    def code_dtype(self):
        return torch.int8 if self.signed else torch.uint8


Q4_4 = FixedPointSpec(ib=4, fb=4)
Q2_2 = FixedPointSpec(ib=2, fb=2)
Q0_8_UNSIGNED = FixedPointSpec(ib=0, fb=8, signed=False)


# --------------------------------------------------------------------------- plumbing

def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def as_device_f32(x) -> torch.Tensor:
    """float32, contiguous, on the current CUDA device (copying if needed)."""
    if not torch.cuda.is_available():
        raise N.NativeUnavailable("a CUDA device is required (there is no CPU path)")
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.as_tensor(np.asarray(x))
    if not t.is_cuda:
        t = t.to(device="cuda", non_blocking=False)
    if t.dtype != torch.float32:
        t = t.to(torch.float32)
    return t.contiguous()


def as_device_f32_exact(x, what: str) -> torch.Tensor:
    """as_device_f32 for codecs whose reference math runs on the input's own
    float64 values (percentile, top-k keys): a float64 input is accepted
    only when every value is exactly a float32, so the results are the
    reference's; otherwise CodecError (no silent narrowing)."""
    src = x if isinstance(x, torch.Tensor) else np.asarray(x)
    if src.dtype in (torch.float64, np.float64):
        t64 = _as_device(src, torch.float64)
        t = t64.to(torch.float32)
        exact = torch.equal(t.to(torch.float64), t64) or bool(
            (torch.isnan(t64) | (t.to(torch.float64) == t64)).all())
        if not exact:
            raise CodecError(f"{what}: float64 values that are not exactly float32 are not supported "
                             "by the device codecs (activations are float32)")
        return t.contiguous()
    return as_device_f32(src)


def _as_device(x, dtype) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    if not t.is_cuda:
        t = t.to("cuda")
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _quantile(pct: float) -> float:
    q = PERCENTILE_Q.get(pct)
    if q is None:
        q = float(np.true_divide(pct, 100))
        PERCENTILE_Q[pct] = q
    return q


# --------------------------------------------------------------------------- K1 / K2

def quantize(x, spec: FixedPointSpec) -> torch.Tensor:
    """Saturating fixed-point codes, ties away from zero (compression.py:66-74),
    one int8 (signed spec) / uint8 code per element, same shape as x."""
    src = x if isinstance(x, torch.Tensor) else np.asarray(x)
    if src.dtype in (torch.float64, np.float64):
        # the reference scales and rounds in float64: keep float64 inputs
        # float64 (narrowing first can move a value across a half-code tie)
        t = _as_device(src, torch.float64)
        out = torch.empty(t.shape, dtype=spec.code_dtype, device=t.device)
        N.call("sf_quantize_f64", _ptr(t), _ptr(out), t.numel(), spec.bits, spec.fb, int(spec.signed),
               _stream())
        return out
    t = as_device_f32(src)
    out = torch.empty(t.shape, dtype=spec.code_dtype, device=t.device)
    N.call("sf_quantize", _ptr(t), _ptr(out), t.numel(), spec.bits, spec.fb, int(spec.signed),
           _stream())
    return out


def quantize_into(t: torch.Tensor, out: torch.Tensor, spec: FixedPointSpec):
    """K1 into a preallocated code buffer (no checks beyond the kernel's)."""
    N.call("sf_quantize", _ptr(t), _ptr(out), t.numel(), spec.bits, spec.fb, int(spec.signed),
           _stream())


def dequantize(codes, spec: FixedPointSpec, dtype=torch.float32) -> torch.Tensor:
    """code / 2^fb (compression.py:77-79), exact."""
    c = codes if isinstance(codes, torch.Tensor) else torch.as_tensor(np.asarray(codes))
    c = c.contiguous() if c.is_cuda else c.to("cuda").contiguous()
    if c.dtype not in (torch.int8, torch.uint8):
        # wider integer codes: narrow only when exact (the kernel decodes
        # bytes); codes no quantize() can produce are refused, not wrapped
        lo, hi = (-128, 127) if spec.signed else (0, 255)
        if c.is_floating_point() or (c.numel() and (int(c.min()) < lo or int(c.max()) > hi)):
            raise CodecError(f"codes must be integers in [{lo}, {hi}] for a {spec.bits}-bit "
                             f"{'signed' if spec.signed else 'unsigned'} spec")
        c = c.to(spec.code_dtype)
    y = torch.empty(c.shape, dtype=torch.float32, device=c.device)
    N.call("sf_dequant8", _ptr(c), _ptr(y), c.numel(), spec.fb, int(c.dtype == torch.int8),
           _stream())
    return y if dtype in (None, torch.float32, np.float32) else y.to(_torch_dtype(dtype))


def _torch_dtype(dtype):
    if isinstance(dtype, torch.dtype):
        return dtype
    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]


# --------------------------------------------------------------------------- K3 / K4 / K5

def pack4(codes) -> torch.Tensor:
    """Two 4-bit two's-complement codes per byte, even index in the low nibble,
    odd count padded with 0 (compression.py:82-95); returns uint8 on device."""
    c = codes if isinstance(codes, torch.Tensor) else torch.as_tensor(np.asarray(codes))
    c = c.reshape(-1)
    if not c.is_cuda:
        c = c.to("cuda")
    n = c.numel()
    # range check on the codes as given (compression.py:87-90 checks in
    # int64): narrowing first would let e.g. 248 wrap to -8 and pass
    if n and (float(c.min()) < -8 or float(c.max()) > 7):
        raise CodecError(f"4-bit codes must lie in [-8, 7], got range [{c.min().item()}, {c.max().item()}]")
    c = c.to(torch.int8).contiguous()
    out = torch.empty((n + 1) // 2, dtype=torch.uint8, device=c.device)
    if n:
        zero = torch.zeros(1, dtype=torch.int32, device=c.device)
        N.call("sf_quant4_pack", _ptr(c.to(torch.float32)), _ptr(out), n, _ptr(zero), 0, _stream())
    return out


def unpack4(data, count: int) -> torch.Tensor:
    """Inverse of pack4: `count` sign-extended codes as int8 (compression.py:98-108)."""
    p = _as_device(data, torch.uint8).reshape(-1)
    if count > 2 * p.numel():
        raise CodecError(f"cannot unpack {count} codes from {p.numel()} bytes")
    y = torch.empty(count, dtype=torch.float32, device=p.device)
    if count:
        zero = torch.zeros(1, dtype=torch.int32, device=p.device)
        N.call("sf_unpack4_dequant", _ptr(p), _ptr(y), count, _ptr(zero), 0, _stream())
    return y.to(torch.int8)


def prescale_exp_device(t: torch.Tensor, spec: FixedPointSpec, percentile: float = 99.9,
                        s_out: torch.Tensor | None = None) -> torch.Tensor:
    """K3: the prescale exponent left in device memory (int32[1]), no sync."""
    s = s_out if s_out is not None else torch.empty(1, dtype=torch.int32, device=t.device)
    ws = _ws(N.load().sf_prescale_workspace_bytes(t.numel()), t.device)
    N.call("sf_prescale_exp", _ptr(t), t.numel(), _quantile(percentile), float(spec.value_max),
           _ptr(s), None, _ptr(ws), _stream())
    return s


def choose_prescale_exp(x, spec: FixedPointSpec, percentile: float = 99.9) -> int:
    """s = max(0, ceil(log2(p / value_max))) with p numpy's linear-method
    percentile of |x| (compression.py:111-124).  Synchronises to return an int."""
    t = as_device_f32_exact(x, "choose_prescale_exp")
    if t.numel() == 0:
        return 0
    return int(prescale_exp_device(t, spec, percentile).item())


# --------------------------------------------------------------------------- K6 / K7

@dataclass
class PrunedSparse:
    """Top-k survivors (float32 values, strictly increasing int32 flat indices)
    of a dense tensor of `dense_size` elements and `shape` (compression.py:127-134)."""

    values: torch.Tensor
    indices: torch.Tensor
    dense_size: int
    shape: tuple
    row_ptr: torch.Tensor | None = None   # CSR over rows of shape[-1] (LayerNorm backward)


def keep_count(n: int, keep_frac: float) -> int:
    """k = ceil(keep_frac * n) in float64, as the reference forms it (compression.py:152)."""
    return math.ceil(keep_frac * n)


def new_prune_hint(device=None) -> torch.Tensor:
    """A per-call-site prune hint (4 uint32 on the device, zero = none yet):
    pass the same tensor to every `prune_topk` call at one site (e.g. one
    frozen LayerNorm); each call rewrites it with its threshold so the next
    call skips the sample and two grid barriers.  Results never depend on
    it (a stale hint falls back to the general path in the same launch)."""
    return torch.zeros(N.load().sf_prune_hint_bytes() // 4, dtype=torch.int32, device=device or "cuda")


def prune_topk(x, keep_frac: float = 0.1, by_magnitude: bool = True,
               row_pointers: bool = False, hint: torch.Tensor | None = None) -> PrunedSparse:
    """Keep the ceil(keep_frac * n) largest (|x| or x) over the whole tensor,
    ties toward the lower flat index, indices ascending (compression.py:137-162).
    row_pointers=True also returns the kept set's CSR row pointers over rows
    of the last dimension (written by the same pass).  `hint`: see
    `new_prune_hint` (speed only; identical output)."""
    t = as_device_f32_exact(x, "prune_topk")
    n = t.numel()
    if n == 0:
        raise CodecError("cannot prune an empty tensor")
    if not 0.0 < keep_frac <= 1.0:
        raise CodecError(f"keep_frac must be in (0, 1], got {keep_frac}")
    k = keep_count(n, keep_frac)
    vals = torch.empty(k, dtype=torch.float32, device=t.device)
    idx = torch.empty(k, dtype=torch.int32, device=t.device)
    ws = _ws(N.load().sf_prune_workspace_bytes(n), t.device)
    row_ptr = None
    if hint is not None:
        if not (hint.is_cuda and hint.numel() * hint.element_size() >= N.load().sf_prune_hint_bytes()
                and hint.data_ptr() % 16 == 0 and hint.is_contiguous()):
            raise CodecError("prune hint must be a contiguous 4-element 32-bit device tensor (new_prune_hint)")
        row_len = (t.shape[-1] if t.dim() else 1) if row_pointers else 0
        if row_pointers:
            row_ptr = torch.empty(n // row_len + 1, dtype=torch.int32, device=t.device)
        N.call("sf_prune_topk_hint", _ptr(t), n, k, int(by_magnitude), _ptr(vals), _ptr(idx), row_len,
               _ptr(row_ptr) if row_ptr is not None else None, _ptr(hint), _ptr(ws), _stream())
    elif row_pointers:
        row_len = t.shape[-1] if t.dim() else 1
        row_ptr = torch.empty(n // row_len + 1, dtype=torch.int32, device=t.device)
        N.call("sf_prune_topk_rows", _ptr(t), n, k, int(by_magnitude), _ptr(vals), _ptr(idx), row_len,
               _ptr(row_ptr), _ptr(ws), _stream())
    else:
        N.call("sf_prune_topk", _ptr(t), n, k, int(by_magnitude), _ptr(vals), _ptr(idx), _ptr(ws),
               _stream())
    return PrunedSparse(vals, idx, n, tuple(t.shape), row_ptr)


def restore(sparse: PrunedSparse, dtype=torch.float32) -> torch.Tensor:
    """Zero tensor of the original shape with the survivors scattered back
    (compression.py:165-169)."""
    dense = torch.empty(sparse.dense_size, dtype=torch.float32, device=sparse.values.device)
    rp = getattr(sparse, "row_ptr", None)
    H = sparse.shape[-1] if sparse.shape else 0
    if rp is not None and H and H % 4 == 0 and H <= 1536 and sparse.dense_size % H == 0:
        N.call("sf_restore_rows", _ptr(sparse.values), _ptr(sparse.indices), sparse.values.numel(), _ptr(rp), H,
               _ptr(dense), sparse.dense_size, _stream())
    else:
        N.call("sf_restore", _ptr(sparse.values), _ptr(sparse.indices), sparse.values.numel(),
               _ptr(dense), sparse.dense_size, _stream())
    out = dense.reshape(sparse.shape)
    return out if dtype in (None, torch.float32, np.float32) else out.to(_torch_dtype(dtype))


# --------------------------------------------------------------------------- container

class CompressedActivation:
    """Tagged encoded activation: "quant8", "packed4" or "pruned"
    (compression.py:172-257).  Payload tensors stay on the device; the
    packed4 prescale exponent stays on the device too (`prescale_exp_dev`)
    and is only fetched when `prescale_exp` is read."""

    __slots__ = ("tag", "shape", "spec", "codes", "packed_codes", "count", "prescale_exp_dev",
                 "sparse", "_s_host", "_ready")

    def __init__(self, tag, shape, spec=None, packed=None, codes=None, count=None,
                 prescale_exp_dev=None, sparse=None):
        self.tag = tag
        self.shape = tuple(shape)
        self.spec = spec
        self.codes = codes
        self.packed_codes = packed
        self.count = count
        self.prescale_exp_dev = prescale_exp_dev
        self.sparse = sparse
        self._s_host = None
        self._ready = None          # completion event when encoded on the codec side stream

    @classmethod
    def encode_async(cls, fn, *inputs) -> "CompressedActivation":
        """`fn()` (returning a CompressedActivation) on the codec side stream
        (streams.py); `inputs` are the tensors it reads."""
        ca, ev = S.run(fn, *inputs)
        ca._ready = ev
        return ca

    def wait(self) -> "CompressedActivation":
        """Order the current stream after the encoder (no-op when it ran inline)."""
        if self._ready is not None:
            ev, self._ready = self._ready, None
            sp = self.sparse
            S.consume(ev, [self.codes, self.packed_codes, self.prescale_exp_dev,
                           sp.values if sp else None, sp.indices if sp else None,
                           sp.row_ptr if sp else None])
        return self

    @classmethod
    def quantized(cls, x, spec: FixedPointSpec) -> "CompressedActivation":
        if spec.bits != 8:
            raise CodecError("quantized() stores one code per byte; use packed() for 4-bit")
        t = as_device_f32(x)
        return cls("quant8", t.shape, spec=spec, codes=quantize(t, spec))

    @classmethod
    def packed(cls, x, spec: FixedPointSpec, prescale_percentile: float = 99.9) -> "CompressedActivation":
        if spec.bits != 4:
            raise CodecError("packed() is for 4-bit specs")
        t = as_device_f32_exact(x, "packed")
        n = t.numel()
        s = torch.zeros(1, dtype=torch.int32, device=t.device)
        out = torch.empty((n + 1) // 2, dtype=torch.uint8, device=t.device)
        if n:
            prescale_exp_device(t, spec, prescale_percentile, s_out=s)
            N.call("sf_quant4_pack", _ptr(t), _ptr(out), n, _ptr(s), spec.fb, _stream())
        return cls("packed4", t.shape, spec=spec, packed=out, count=n, prescale_exp_dev=s)

    @classmethod
    def pruned(cls, x, keep_frac: float, by_magnitude: bool = True,
               row_pointers: bool = False) -> "CompressedActivation":
        t = as_device_f32_exact(x, "pruned")
        return cls("pruned", t.shape, sparse=prune_topk(t, keep_frac, by_magnitude, row_pointers))

    @property
    def prescale_exp(self) -> int:
        if self.tag != "packed4":
            return 0
        if self._s_host is None:
            self.wait()
            self._s_host = int(self.prescale_exp_dev.item())
        return self._s_host

    def decompress(self, dtype=torch.float32) -> torch.Tensor:
        self.wait()
        if self.tag == "quant8":
            return dequantize(self.codes, self.spec, dtype).reshape(self.shape)
        if self.tag == "packed4":
            y = torch.empty(self.count, dtype=torch.float32, device=self.packed_codes.device)
            if self.count:
                N.call("sf_unpack4_dequant", _ptr(self.packed_codes), _ptr(y), self.count,
                       _ptr(self.prescale_exp_dev), self.spec.fb, _stream())
            y = y.reshape(self.shape)
            return y if dtype in (None, torch.float32, np.float32) else y.to(_torch_dtype(dtype))
        if self.tag == "pruned":
            return restore(self.sparse, dtype)
        raise CodecError(f"unknown compression tag {self.tag!r}")

    @property
    def nbytes(self) -> int:
        if self.tag == "quant8":
            return int(self.codes.numel())
        if self.tag == "packed4":
            return int(self.packed_codes.numel())
        if self.tag == "pruned":
            return int(self.sparse.values.numel() * 8)
        raise CodecError(f"unknown compression tag {self.tag!r}")

    def dump(self) -> bytes:
        """JSON header line + little-endian payload, byte-compatible with the
        reference's container dump (compression.py:234-257)."""
        self.wait()
        header = {
            "tag": self.tag,
            "shape": list(self.shape),
            "spec": None if self.spec is None else
                    {"ib": self.spec.ib, "fb": self.spec.fb, "signed": self.spec.signed},
            "count": self.count if self.count is not None else
                     (int(self.sparse.values.numel()) if self.tag == "pruned" else
                      (int(self.codes.numel()) if self.tag == "quant8" else None)),
            "prescale_exp": self.prescale_exp,
        }
        head = json.dumps(header, sort_keys=True).encode() + b"\n"
        if self.tag == "quant8":
            body = self.codes.reshape(-1).cpu().numpy().astype("<i1").tobytes()
        elif self.tag == "packed4":
            body = self.packed_codes.cpu().numpy().tobytes()
        elif self.tag == "pruned":
            body = (self.sparse.values.cpu().numpy().astype("<f4").tobytes()
                    + self.sparse.indices.cpu().numpy().astype("<i4").tobytes())
        else:
            raise CodecError(f"unknown compression tag {self.tag!r}")
        return head + body
