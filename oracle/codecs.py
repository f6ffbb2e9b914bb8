"""Oracle codecs: fixed-point quantize, nibble packing, percentile prescale,
global top-k magnitude pruning (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Reference: compression.py (paths under /root/reference/pkg/src/slimfit/).
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np


class Fmt(NamedTuple):
    """Q(ib).(fb) code format — compression.py:21-53."""

    ib: int
    fb: int
    signed: bool = True

    @property
    def bits(self):
        return self.ib + self.fb

    @property
    def lo(self):
        return -(2 ** (self.bits - 1)) if self.signed else 0

    @property
    def hi(self):
        return 2 ** (self.bits - 1) - 1 if self.signed else 2 ** self.bits - 1

    @property
    def vmax(self):
        return self.hi / 2.0 ** self.fb


Q44 = Fmt(4, 4)            # compression.py:56
Q22 = Fmt(2, 2)            # compression.py:57
Q08U = Fmt(0, 8, False)    # compression.py:58


def quantize(x, fmt: Fmt) -> np.ndarray:
    """Saturating fixed point, ties away from zero — compression.py:61-74.

    Computed in float64 like the reference; NaN lands on code 0 and +-inf
    saturate (numpy's float->int cast of the clipped NaN gives 0 here).
    """
    v = np.asarray(x, dtype=np.float64) * float(2 ** fmt.fb)
    r = np.floor(np.abs(v) + 0.5)
    r = np.where(v < 0, -r, r)
    r = np.clip(r, fmt.lo, fmt.hi)
    with np.errstate(invalid="ignore"):
        out = r.astype(np.int8 if fmt.signed else np.uint8)
    return out


def dequantize(codes, fmt: Fmt) -> np.ndarray:
    """code / 2^fb in float64, then float32 — compression.py:77-79."""
    return (np.asarray(codes, dtype=np.float64) / float(2 ** fmt.fb)).astype(np.float32)


def pack4(codes) -> np.ndarray:
    """Two 4-bit two's-complement codes per byte, even index in the low nibble,
    odd count padded with a zero high nibble — compression.py:82-95."""
    c = np.asarray(codes).reshape(-1).astype(np.int64)
    if c.size and (c.min() < -8 or c.max() > 7):
        raise ValueError("4-bit code out of range")
    nib = (c & 0xF).astype(np.uint8)
    if nib.size & 1:
        nib = np.append(nib, np.uint8(0))
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8)


def unpack4(packed, count: int) -> np.ndarray:
    """Sign-extending nibble unpack — compression.py:98-108."""
    p = np.asarray(packed, dtype=np.uint8).reshape(-1)
    if count > 2 * p.size:
        raise ValueError("not enough packed bytes")
    both = np.stack([p & 0xF, p >> 4], axis=1).reshape(-1)[:count].astype(np.int16)
    both = np.where(both > 7, both - 16, both)
    return both.astype(np.int8)


def percentile_linear(mags: np.ndarray, pct: float) -> float:
    """numpy 2.3.5 `percentile(..., method='linear')` on a 1-D float64 array,
    restated step by step (numpy/lib/_function_base_impl.py `_quantile`,
    `_get_indexes`, `_lerp`) so the device kernel can mirror each rounding."""
    n = mags.size
    q = np.true_divide(pct, 100)
    vi = (n - 1) * q
    if np.isnan(mags).any():
        return float("nan")
    s = np.sort(mags)
    if vi >= n - 1:
        a = b = s[-1]
        lo = n - 1
    else:
        lo = int(math.floor(vi))
        a, b = s[lo], s[lo + 1]
    g = vi - float(lo) if vi < n - 1 else vi - math.floor(vi)
    diff = b - a
    p = a + diff * g
    if g >= 0.5:
        p = b - diff * (1.0 - g)
    return float(p)


def prescale_exp(x, fmt: Fmt, pct: float = 99.9) -> int:
    """Power-of-two prescale for the 4-bit GELU codec — compression.py:111-124."""
    mags = np.abs(np.asarray(x, dtype=np.float64)).reshape(-1)
    if mags.size == 0:
        return 0
    p = percentile_linear(mags, pct)
    if not math.isfinite(p) or p <= 0.0:
        return 0
    return max(0, math.ceil(math.log2(p / fmt.vmax)))


def pack_gelu(x, fmt: Fmt = Q22, pct: float = 99.9):
    """`CompressedActivation.packed` — compression.py:199-207.  Returns
    (packed bytes, prescale exponent, count)."""
    x = np.asarray(x)
    s = prescale_exp(x, fmt, pct)
    codes = quantize(x / (1 << s), fmt)
    return pack4(codes), s, int(x.size)


def unpack_gelu(packed, s: int, count: int, fmt: Fmt = Q22) -> np.ndarray:
    """packed4 branch of `decompress` — compression.py:216-219."""
    return dequantize(unpack4(packed, count), fmt) * np.float32(1 << s)


def keep_count(n: int, keep_frac: float) -> int:
    """k = ceil(keep_frac * n) in Python float64 — compression.py:152."""
    return math.ceil(keep_frac * n)


def prune_topk(x, keep_frac: float = 0.1, by_magnitude: bool = True):
    """Global top-k keep with ties toward the lower flat index; returns
    (values f32, indices int32 ascending) — compression.py:137-162."""
    flat = np.asarray(x).reshape(-1)
    n = flat.size
    if n == 0:
        raise ValueError("cannot prune an empty tensor")
    if not 0.0 < keep_frac <= 1.0:
        raise ValueError("keep_frac must be in (0, 1]")
    k = keep_count(n, keep_frac)
    key = np.abs(flat) if by_magnitude else flat
    # stable descending order == stable ascending order of the negated key;
    # NaN negates to NaN and therefore sorts last (below every number)
    order = np.argsort(-key, kind="stable")[:k]
    idx = np.sort(order).astype(np.int32)
    return flat[idx].astype(np.float32), idx


def restore(values, indices, n: int, shape=None) -> np.ndarray:
    """Zero-fill then scatter — compression.py:165-169."""
    dense = np.zeros(n, dtype=np.float32)
    dense[np.asarray(indices)] = np.asarray(values, dtype=np.float32)
    return dense if shape is None else dense.reshape(shape)


def payload_nbytes(tag: str, n: int, keep_frac: float = 0.1) -> int:
    """`CompressedActivation.nbytes` — compression.py:224-232."""
    if tag == "quant8":
        return n
    if tag == "packed4":
        return (n + 1) // 2
    if tag == "pruned":
        return keep_count(n, keep_frac) * 8
    raise ValueError(tag)
