"""Oracle for the inter-layer-scheduling (ILS) path: warm-start distances,
freeze selection, per-layer update distance, and the f32 AdamW step with
pause semantics (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

References: scheduler.py:19-21, :53-59, :71-89, :92-120;
trainer.py:27-76 (paths under /root/reference/pkg/src/slimfit/).
"""

from __future__ import annotations

import math

import numpy as np

WARM_LO, WARM_HI = 1.0e6, 2.0e6     # scheduler.py:19-20
DIV_GUARD = 1.0e-12                 # scheduler.py:21


def warm_distances(n: int, seed: int) -> np.ndarray:
    """default_rng(seed).uniform(1e6, 2e6, n) — scheduler.py:53-59."""
    if n < 1:
        raise ValueError("need at least one layer")
    return np.random.default_rng(seed).uniform(WARM_LO, WARM_HI, size=n)


def frozen_ids(d: np.ndarray, rate: float, pinned=()) -> list[int]:
    """The int(n*rate) smallest distances, ties to the lower id, pinned ids
    never chosen — scheduler.py:71-89."""
    if not 0.0 <= rate < 1.0:
        raise ValueError("freeze rate must lie in [0, 1)")
    d = np.array(d, dtype=np.float64)
    if pinned:
        d[list(pinned)] = np.inf
    k = int(d.size * rate)
    return sorted(int(i) for i in np.argsort(d, kind="stable")[:k])


def pairwise_sum(e: np.ndarray) -> float:
    """numpy's float64 add-reduce over a contiguous 1-D array, restated:
    8-way unrolled leaves of <= 128 elements, halving splits rounded down to
    a multiple of 8 (numpy/_core/src/umath/loops_utils.h.src pairwise_sum).

    Used by the tests to pin the exact summation order that the device
    distance kernel reproduces; `np.sum` itself is the arithmetic reference.
    """
    e = np.asarray(e, dtype=np.float64).reshape(-1)

    def rec(lo: int, n: int) -> float:
        if n < 8:
            acc = 0.0
            for i in range(n):
                acc = acc + float(e[lo + i])
            return acc
        if n <= 128:
            r = [float(v) for v in e[lo:lo + 8]]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] = r[j] + float(e[lo + i + j])
                i += 8
            acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                acc = acc + float(e[lo + i])
                i += 1
            return acc
        h = n // 2
        h -= h % 8
        return rec(lo, h) + rec(lo + h, n - h)

    return rec(0, e.size)


def rel_change(before, after) -> np.ndarray:
    """Elementwise |after - before| / (|before| + 1e-12) in float64 —
    scheduler.py:102-103."""
    b = np.asarray(before, dtype=np.float64).reshape(-1)
    a = np.asarray(after, dtype=np.float64).reshape(-1)
    return np.abs(a - b) / (np.abs(b) + DIV_GUARD)


def layer_distance(before_params, after_params) -> float:
    """Pooled mean relative change over a layer's params, summed with
    numpy's own add-reduce — scheduler.py:92-105."""
    total, count = 0.0, 0
    for b, a in zip(before_params, after_params):
        total += float(np.sum(rel_change(b, a)))
        count += np.asarray(b).size
    return total / count if count else 0.0


# ---------------------------------------------------------------------------
# AdamW, f32, per-layer step counts (trainer.py:27-76)

BETA1, BETA2, EPS, WD = 0.9, 0.999, 1e-8, 0.01


def adamw_constants(t: int, lr: float, beta1=BETA1, beta2=BETA2, eps=EPS, wd=WD):
    """The float32 constants numpy's weak-scalar promotion produces for step
    t (trainer.py:67-74): each Python float is rounded to f32 once."""
    f = np.float32
    return dict(b1=f(beta1), ob1=f(1 - beta1), b2=f(beta2), ob2=f(1 - beta2),
                bc1=f(1 - beta1 ** t), bc2=f(1 - beta2 ** t), eps=f(eps),
                wd=f(wd), lr=f(lr))


def adamw_param(p, g, m, v, t: int, lr: float, wd=WD):
    """One AdamW update of one f32 parameter; returns (p, m, v) new arrays.
    Operation order follows trainer.py:67-74 exactly (no fused multiply-add).
    """
    c = adamw_constants(t, lr, wd=wd)
    p = np.asarray(p, np.float32)
    g = np.asarray(g, np.float32)
    m = c["b1"] * m + c["ob1"] * g
    v = c["b2"] * v + (c["ob2"] * g) * g
    mh = m / c["bc1"]
    vh = v / c["bc2"]
    u = mh / (np.sqrt(vh) + c["eps"]) + c["wd"] * p
    return (p - c["lr"] * u).astype(np.float32), m, v


class AdamW:
    """Per-layer step counters; frozen layers are pauses — trainer.py:27-63."""

    def __init__(self, weight_decay=WD):
        self.wd = weight_decay
        self.moments = {}       # (layer_id, slot) -> (m, v)
        self.steps = {}         # layer_id -> t

    def step(self, layers: dict, grads: dict, lr: float, active):
        """layers: lid -> list of param arrays (replaced in place in the list);
        grads: lid -> list of grads or None."""
        for lid in active:
            gl = grads.get(lid)
            if gl is None or all(g is None for g in gl):
                continue
            self.steps[lid] = self.steps.get(lid, 0) + 1
            t = self.steps[lid]
            for slot, g in enumerate(gl):
                if g is None:
                    continue
                p = layers[lid][slot]
                key = (lid, slot)
                if key not in self.moments:
                    self.moments[key] = (np.zeros_like(p), np.zeros_like(p))
                m, v = self.moments[key]
                layers[lid][slot], m, v = adamw_param(p, g, m, v, t, lr, self.wd)
                self.moments[key] = (m, v)


class SGD:
    """p - f32(lr * g) per parameter with a gradient — trainer.py:63-65
    (numpy's weak-scalar promotion keeps the product in float32); per-layer
    step counters advance as AdamW's do (trainer.py:55-58)."""

    def __init__(self):
        self.steps = {}

    def step(self, layers: dict, grads: dict, lr: float, active):
        lr32 = np.float32(lr)
        for lid in active:
            gl = grads.get(lid)
            if gl is None or all(g is None for g in gl):
                continue
            self.steps[lid] = self.steps.get(lid, 0) + 1
            for slot, g in enumerate(gl):
                if g is not None:
                    p = np.asarray(layers[lid][slot], np.float32)
                    layers[lid][slot] = (p - lr32 * np.asarray(g, np.float32)).astype(np.float32)


def linear_lr(base: float, step: int, total: int, warmup_frac: float) -> float:
    """Linear warmup then linear decay — trainer.py:79-87."""
    w = int(warmup_frac * total)
    if w > 0 and step < w:
        return base * (step + 1) / w
    if total <= w:
        return base
    return base * max(0.0, 1.0 - (step - w) / max(1, total - w))


def keep_frac_k(n: int, frac: float) -> int:
    return math.ceil(frac * n)
