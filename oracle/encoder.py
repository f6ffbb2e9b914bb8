"""Oracle encoder: the reference's freezable transformer restated as explicit
per-layer forward/backward in numpy float32, with the reference's
freeze-aware, codec-aware activation caching and its cached-bytes ledger
(TEST INFRASTRUCTURE ONLY, see oracle/__init__).

References (under /root/reference/pkg/src/slimfit/):
  model.py:23-44 (config), :55-86 + :115-161 (registry and init),
  :202-295 (forward graph), tensor.py:290-674 (op semantics and what each
  op caches), tensor.py:168-179 (ledger), trainer.py:144-222 (loop).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import codecs as C
from . import ils

GELU_K = math.sqrt(2.0 / math.pi)   # tensor.py:27
GELU_CUBIC = 0.044715               # tensor.py:28
LN_EPS = 1e-5                       # tensor.py:447


@dataclass
class EncoderConfig:
    """model.py:23-44."""

    blocks: int = 3
    hidden: int = 32
    heads: int = 4
    max_seq: int = 16
    vocab: int = 64
    num_classes: int = 4
    pre_norm: bool = False
    type_vocab: int = 2

    @property
    def n_layers(self):
        return 4 + 8 * self.blocks + 2


@dataclass
class Codecs:
    """CompressionConfig — tensor.py:31-57."""

    quant_dense: bool = False
    quant_matmul_softmax: bool = False
    quant_gelu: bool = False
    prune_layernorm: bool = False
    keep_frac: float = 0.1
    dense_fmt: C.Fmt = C.Q44
    matsoft_fmt: C.Fmt = C.Q44
    gelu_fmt: C.Fmt = C.Q22
    prune_by_magnitude: bool = True

    @classmethod
    def all_on(cls, **kw):
        base = dict(quant_dense=True, quant_matmul_softmax=True, quant_gelu=True,
                    prune_layernorm=True)
        base.update(kw)
        return cls(**base)


BLOCK_SLOTS = ("attention.self.query", "attention.self.key", "attention.self.value",
               "attention.output.dense", "attention.output.LayerNorm",
               "intermediate.dense", "output.dense", "output.LayerNorm")


def layer_table(cfg: EncoderConfig):
    """(name, kind) per layer id, ids dense 0..n-1 — model.py:143-160."""
    t = [("embeddings.word_embeddings", "embedding"),
         ("embeddings.position_embeddings", "embedding"),
         ("embeddings.token_type_embeddings", "embedding"),
         ("embeddings.LayerNorm", "layernorm")]
    for i in range(cfg.blocks):
        for s in BLOCK_SLOTS:
            t.append((f"encoder.layer.{i}.{s}", "layernorm" if s.endswith("LayerNorm") else "dense"))
    t += [("pooler.dense", "dense"), ("classifier", "dense")]
    return t


def _tn(rng, shape, std=0.02):
    """Truncated normal by resampling beyond 2 sigma — model.py:96-103."""
    a = rng.normal(0.0, std, size=shape)
    out = np.abs(a) > 2 * std
    while out.any():
        a[out] = rng.normal(0.0, std, size=int(out.sum()))
        out = np.abs(a) > 2 * std
    return a.astype(np.float32)


def init_params(cfg: EncoderConfig, seed: int):
    """Per-layer parameter lists in registry order, drawing from one
    default_rng(seed) stream in construction order — model.py:115-161."""
    rng = np.random.default_rng(seed)
    H, I = cfg.hidden, 4 * cfg.hidden
    params = []
    for name, kind in layer_table(cfg):
        if kind == "embedding":
            rows = {"embeddings.word_embeddings": cfg.vocab,
                    "embeddings.position_embeddings": cfg.max_seq,
                    "embeddings.token_type_embeddings": cfg.type_vocab}[name]
            params.append([_tn(rng, (rows, H))])
        elif kind == "layernorm":
            params.append([np.ones(H, np.float32), np.zeros(H, np.float32)])
        else:
            if name.endswith("intermediate.dense"):
                fi, fo = H, I
            elif name.endswith("output.dense") and ".attention." not in name:
                fi, fo = I, H
            elif name == "classifier":
                fi, fo = H, cfg.num_classes
            else:
                fi, fo = H, H
            params.append([_tn(rng, (fi, fo)), np.zeros(fo, np.float32)])
    return params


# ---------------------------------------------------------------------------
# cached values: raw arrays or encoded payloads, with their ledger bytes


class Cache:
    """One cached activation (tensor.py:116-141): `get()` decodes."""

    def __init__(self, kind, name, raw=None, q8=None, p4=None, pr=None, shape=None):
        self.kind, self.name = kind, name
        self.raw, self.q8, self.p4, self.pr = raw, q8, p4, pr
        self.shape = shape if shape is not None else (raw.shape if raw is not None else None)

    def get(self):
        if self.raw is not None:
            return self.raw
        if self.q8 is not None:
            codes, fmt = self.q8
            return C.dequantize(codes, fmt).reshape(self.shape)
        if self.p4 is not None:
            packed, s, count, fmt = self.p4
            return C.unpack_gelu(packed, s, count, fmt).reshape(self.shape)
        vals, idx, n = self.pr
        return C.restore(vals, idx, n, self.shape)

    @property
    def nbytes(self):
        if self.raw is not None:
            return int(self.raw.nbytes)
        if self.q8 is not None:
            return int(self.q8[0].size)
        if self.p4 is not None:
            return int(self.p4[0].size)
        return int(self.pr[0].size) * 8


def _cache_q8(arr, on, fmt, kind, name):
    if on:
        return Cache(kind, name, q8=(C.quantize(arr, fmt), fmt), shape=arr.shape)
    return Cache(kind, name, raw=arr)


class Ledger:
    """Distinct cached buffers of one iteration — tensor.py:168-191."""

    def __init__(self):
        self.items = []
        self._seen = set()

    def add(self, c: Cache):
        if id(c) not in self._seen:
            self._seen.add(id(c))
            self.items.append(c)
        return c

    def totals(self):
        t = {"dynamic": 0, "static": 0, "semi_static": 0}
        for c in self.items:
            t[c.kind] += c.nbytes
        t["total"] = t["dynamic"] + t["static"] + t["semi_static"]
        return t


# ---------------------------------------------------------------------------
# one training step


def _ln_fwd(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xt = (x - mu) * rstd
    return xt * g + b, xt, rstd


def _gelu(x):
    return 0.5 * x * (1.0 + np.tanh(GELU_K * (x + GELU_CUBIC * x ** 3)))


def _gelu_grad(g, x):
    t = np.tanh(GELU_K * (x + GELU_CUBIC * x ** 3))
    du = GELU_K * (1.0 + 3.0 * GELU_CUBIC * x ** 2)
    return g * (0.5 * (1.0 + t) + 0.5 * x * (1.0 - t ** 2) * du)


class Step:
    """Forward + backward of one iteration on fixed params/freeze set.

    `params` is the per-layer list from `init_params`; `frozen` a set of layer
    ids; `codecs` a `Codecs` or None.  After `run()`: `loss`, `logits`,
    `grads` (lid -> list of arrays, only for enabled layers), `ledger`.
    """

    def __init__(self, cfg: EncoderConfig, params, frozen=(), codecs: Codecs | None = None):
        self.cfg, self.P, self.frozen, self.cx = cfg, params, set(frozen), codecs
        self.ledger = Ledger()
        self.grads = {}
        self.names = [n for n, _ in layer_table(cfg)]

    # -- helpers -----------------------------------------------------------
    def _on(self, lid):
        return lid not in self.frozen

    def _addg(self, lid, slot, g):
        gl = self.grads.setdefault(lid, [None] * len(self.P[lid]))
        gl[slot] = g if gl[slot] is None else gl[slot] + g

    def _dense_fwd(self, lid, x, compress8=False):
        W, b = self.P[lid]
        y = x @ W + b
        cache = None
        if self._on(lid):
            on = compress8 and self.cx is not None and self.cx.quant_dense
            fmt = self.cx.dense_fmt if self.cx is not None else None
            cache = self.ledger.add(_cache_q8(x, on, fmt, "dynamic", f"{self.names[lid]}.input"))
        return y, (lid, cache, x.shape)

    def _dense_bwd(self, st, g):
        lid, cache, xshape = st
        W, _ = self.P[lid]
        dx = (g @ W.T).reshape(xshape)
        if cache is not None:
            g2 = g.reshape(-1, g.shape[-1])
            xv = cache.get().reshape(-1, W.shape[0])
            self._addg(lid, 0, xv.T @ g2)
            self._addg(lid, 1, g2.sum(axis=0))
        return dx

    def _ln_fwd(self, lid, x):
        g, b = self.P[lid]
        y, xt, rstd = _ln_fwd(x, g, b)
        on = self._on(lid)
        name = self.names[lid]
        if not on and self.cx is not None and self.cx.prune_layernorm:
            vals, idx = C.prune_topk(xt, self.cx.keep_frac, self.cx.prune_by_magnitude)
            cx = Cache("semi_static", f"{name}.xtilde", pr=(vals, idx, xt.size), shape=xt.shape)
        else:
            cx = Cache("semi_static", f"{name}.xtilde", raw=xt)
        self.ledger.add(cx)
        cr = self.ledger.add(Cache("static", f"{name}.rstd", raw=rstd))
        return y, (lid, cx, cr, on)

    def _ln_bwd(self, st, g):
        lid, cx, cr, on = st
        gam = self.P[lid][0]
        H = gam.shape[0]
        xt = cx.get()
        rs = cr.get()
        gg = gam * g * rs / H
        dx = H * gg - gg.sum(axis=-1, keepdims=True) - xt * (gg * xt).sum(axis=-1, keepdims=True)
        if on:
            self._addg(lid, 0, (xt * g).reshape(-1, H).sum(axis=0))
            self._addg(lid, 1, g.reshape(-1, H).sum(axis=0))
        return dx

    # -- the step ----------------------------------------------------------
    def run(self, ids, labels):
        cfg, cx = self.cfg, self.cx
        ids = np.asarray(ids)
        labels = np.asarray(labels)
        B, T = ids.shape
        H, nh = cfg.hidden, cfg.heads
        dh = H // nh
        ms = cx is not None and cx.quant_matmul_softmax
        msf = cx.matsoft_fmt if cx is not None else None
        L = self.ledger

        word, pos, tok = self.P[0][0], self.P[1][0], self.P[2][0]
        if self._on(0):
            L.add(Cache("dynamic", "embeddings.word_embeddings.ids", raw=ids.astype(np.int32)))
        x = (word[ids] + pos[:T]) + tok[:1]
        x, st_eln = self._ln_fwd(3, x)

        blocks = []
        for i in range(cfg.blocks):
            base = 4 + 8 * i
            p = f"encoder.layer.{i}"
            rec = {}
            attn_in = x
            if cfg.pre_norm:
                attn_in, rec["ln1"] = self._ln_fwd(base + 4, x)
            q, rec["q"] = self._dense_fwd(base + 0, attn_in)
            k, rec["k"] = self._dense_fwd(base + 1, attn_in)
            v, rec["v"] = self._dense_fwd(base + 2, attn_in)
            qh = q.reshape(B, T, nh, dh).transpose(0, 2, 1, 3)
            kh = k.reshape(B, T, nh, dh).transpose(0, 2, 1, 3)
            vh = v.reshape(B, T, nh, dh).transpose(0, 2, 1, 3)
            kt = kh.transpose(0, 1, 3, 2)
            c_q = L.add(_cache_q8(qh, ms, msf, "static", f"{p}.attention.scores.lhs"))
            c_kt = L.add(_cache_q8(kt, ms, msf, "static", f"{p}.attention.scores.rhs"))
            scale = np.float32(1.0 / math.sqrt(dh))
            s = np.matmul(qh, kt) * scale
            s = s - s.max(axis=-1, keepdims=True)
            e = np.exp(s)
            probs = e / e.sum(axis=-1, keepdims=True)
            c_p = L.add(_cache_q8(probs, ms, msf, "static", f"{p}.attention.softmax.probs"))
            c_v = L.add(_cache_q8(vh, ms, msf, "static", f"{p}.attention.context.rhs"))
            ctx = np.matmul(probs, vh).transpose(0, 2, 1, 3).reshape(B, T, H)
            rec["attn"] = (c_q, c_kt, c_p, c_v, scale)
            a, rec["o"] = self._dense_fwd(base + 3, ctx)
            x = x + a
            if not cfg.pre_norm:
                x, rec["ln1"] = self._ln_fwd(base + 4, x)
            ffn_in = x
            if cfg.pre_norm:
                ffn_in, rec["ln2"] = self._ln_fwd(base + 7, x)
            hp, rec["i"] = self._dense_fwd(base + 5, ffn_in)
            if cx is not None and cx.quant_gelu:
                packed, sexp, cnt = C.pack_gelu(hp, cx.gelu_fmt)
                c_g = Cache("static", f"{p}.intermediate.gelu.input",
                            p4=(packed, sexp, cnt, cx.gelu_fmt), shape=hp.shape)
            else:
                c_g = Cache("static", f"{p}.intermediate.gelu.input", raw=hp)
            rec["gelu"] = L.add(c_g)
            h = _gelu(hp)
            o, rec["d"] = self._dense_fwd(base + 6, h, compress8=True)
            x = x + o
            if not cfg.pre_norm:
                x, rec["ln2"] = self._ln_fwd(base + 7, x)
            blocks.append(rec)

        n = cfg.n_layers
        cls = x[:, 0, :]
        pre, st_pool = self._dense_fwd(n - 2, cls)
        pooled = np.tanh(pre)
        c_tanh = L.add(Cache("static", "pooler.tanh.output", raw=pooled))
        logits, st_cls = self._dense_fwd(n - 1, pooled)

        z = logits - logits.max(axis=1, keepdims=True)
        ez = np.exp(z)
        pr = ez / ez.sum(axis=1, keepdims=True)
        nll = -(z[np.arange(B), labels] - np.log(ez.sum(axis=1)))
        self.loss = np.asarray(nll.mean(), dtype=logits.dtype)
        self.logits = logits
        L.add(Cache("static", "loss.probs", raw=pr))
        L.add(Cache("static", "loss.labels", raw=labels.astype(np.int32)))

        # -- backward (reverse order of the forward graph) --------------------
        one = np.ones_like(self.loss)
        dl = pr.copy()
        dl[np.arange(B), labels] -= 1.0
        dlogits = one * dl / B
        dpooled = self._dense_bwd(st_cls, dlogits)
        dpre = dpooled * (1.0 - c_tanh.get() ** 2)
        dcls = self._dense_bwd(st_pool, dpre)
        dx = np.zeros_like(x)
        dx[:, 0, :] = dcls

        for i in reversed(range(cfg.blocks)):
            rec = blocks[i]
            if not cfg.pre_norm:
                dx = self._ln_bwd(rec["ln2"], dx)
            dh_ = self._dense_bwd(rec["d"], dx)
            dhp = _gelu_grad(dh_, rec["gelu"].get())
            dffn = self._dense_bwd(rec["i"], dhp)
            if cfg.pre_norm:
                dffn = self._ln_bwd(rec["ln2"], dffn)
            dx = dx + dffn
            if not cfg.pre_norm:
                dx = self._ln_bwd(rec["ln1"], dx)
            dctx = self._dense_bwd(rec["o"], dx)
            c_q, c_kt, c_p, c_v, scale = rec["attn"]
            dctx = dctx.reshape(B, T, nh, dh).transpose(0, 2, 1, 3)
            pv = c_p.get()
            dprobs = np.matmul(dctx, np.swapaxes(c_v.get(), -1, -2))
            dvh = np.matmul(np.swapaxes(pv, -1, -2), dctx)
            ds = pv * (dprobs - (dprobs * pv).sum(axis=-1, keepdims=True))
            ds = ds * scale
            dqh = np.matmul(ds, np.swapaxes(c_kt.get(), -1, -2))
            dkt = np.matmul(np.swapaxes(c_q.get(), -1, -2), ds)
            dq = dqh.transpose(0, 2, 1, 3).reshape(B, T, H)
            dk = dkt.transpose(0, 1, 3, 2).transpose(0, 2, 1, 3).reshape(B, T, H)
            dv = dvh.transpose(0, 2, 1, 3).reshape(B, T, H)
            din = self._dense_bwd(rec["q"], dq)
            din = din + self._dense_bwd(rec["k"], dk)
            din = din + self._dense_bwd(rec["v"], dv)
            if cfg.pre_norm:
                din = self._ln_bwd(rec["ln1"], din)
            dx = dx + din

        dx = self._ln_bwd(st_eln, dx)
        if self._on(0):
            gw = np.zeros_like(word)
            np.add.at(gw, ids, dx)
            self._addg(0, 0, gw)
        if self._on(1):
            gp = np.zeros_like(pos)
            gp[:T] = dx.sum(axis=0)
            self._addg(1, 0, gp)
        if self._on(2):
            gt = np.zeros_like(tok)
            gt[:1] = dx.sum(axis=0).sum(axis=0, keepdims=True)
            self._addg(2, 0, gt)
        return self


# ---------------------------------------------------------------------------
# the fine-tuning loop (trainer.py:144-222)


def batch_stream(tokens, labels, batch_size, rng, shuffle=True):
    """Drop-tail shuffled minibatches — trainer.py:134-141."""
    n = len(labels)
    order = rng.permutation(n) if shuffle else np.arange(n)
    for s in range(0, n - batch_size + 1, batch_size):
        sel = order[s:s + batch_size]
        yield tokens[sel], labels[sel]


def fine_tune(cfg: EncoderConfig, params, tokens, labels, *, freeze_rate=0.0, epochs=1,
              batch_size=8, seed=0, lr=1e-3, warmup_frac=0.1, weight_decay=0.01,
              codecs: Codecs | None = None, scheduler="ils", pinned=(), max_iters=None,
              optimizer="adamw"):
    """ILS fine-tuning (scheduler kinds "ils" and "none"; optimizer "adamw"
    or "sgd"); returns a log dict with per-iteration loss, frozen ids,
    distances and ledger totals.  Every active layer's distance is refreshed
    after the step whatever the optimizer (trainer.py:194-200); a layer that
    did not move gets 0.0."""
    n = cfg.n_layers
    iters_per_epoch = len(labels) // batch_size
    total = iters_per_epoch * epochs
    d = ils.warm_distances(n, seed)
    opt = ils.AdamW(weight_decay) if optimizer == "adamw" else ils.SGD()
    data_rng = np.random.default_rng([seed, 0xDA7A])
    log = {"loss": [], "frozen": [], "d": [], "ledger": [], "lr": []}
    it = 0
    for _ in range(epochs):
        for tb, lb in batch_stream(tokens, labels, batch_size, data_rng):
            if max_iters is not None and it >= max_iters:
                return log
            fz = ils.frozen_ids(d, freeze_rate, pinned) if scheduler == "ils" else []
            st = Step(cfg, params, fz, codecs).run(tb, lb)
            lv = float(st.loss)
            if not math.isfinite(lv):
                raise FloatingPointError(f"non-finite loss {lv} at iteration {it}")
            active = [i for i in range(n) if i not in set(fz)]
            before = {i: [p.copy() for p in params[i]] for i in active}
            lr_t = ils.linear_lr(lr, it, total, warmup_frac)
            opt.step(params, st.grads, lr_t, active)
            for i in active:
                d[i] = ils.layer_distance(before[i], params[i])
            log["loss"].append(lv)
            log["frozen"].append(fz)
            log["d"].append(d.copy())
            log["ledger"].append(st.ledger.totals())
            log["lr"].append(lr_t)
            it += 1
    return log
