"""Closed-form cached-activation accounting — the drop-in for memory.py
(/root/reference/pkg/src/slimfit/memory.py).

Every buffer one forward pass caches is listed symbolically from the model
configuration with the op's ledger kind and codec slot, and priced with the
same byte formulas the codecs use, so `account_iteration` equals
`Tape.cached_bytes()` of a recorded device iteration exactly (the audit,
memory.py:271-284).  This is host arithmetic, not a kernel.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .model import ModelConfig, registry_size
from .scheduler import FreezeDecision, frozen_count
from .tensor import CompressionConfig

BYTES_F32 = 4
BYTES_I32 = 4
BYTES_ADAM_MOMENTS = 8


@dataclass(frozen=True)
class ActivationRecord:
    """One cached buffer: owner layer (None = unfreezable op), element count,
    ledger kind and codec slot (raw | dense8 | matsoft8 | gelu4 | ln_prune | int32)."""

    name: str
    kind: str
    count: int
    layer_id: int | None
    codec_slot: str = "raw"

    def bytes_under(self, codecs: CompressionConfig | None, frozen: bool) -> int:
        n = self.count
        if self.codec_slot == "int32":
            return n * BYTES_I32
        if codecs is not None:
            slot = self.codec_slot
            if slot == "dense8" and codecs.quant_dense:
                return n
            if slot == "matsoft8" and codecs.quant_matmul_softmax:
                return n if codecs.matmul_softmax_spec.bits == 8 else math.ceil(n / 2)
            if slot == "gelu4" and codecs.quant_gelu:
                return math.ceil(n / 2)
            if slot == "ln_prune" and codecs.prune_layernorm and frozen:
                return math.ceil(codecs.keep_frac * n) * (BYTES_F32 + BYTES_I32)
        return n * BYTES_F32


@dataclass
class MemoryReport:
    config: ModelConfig
    batch_size: int
    freeze_rate: float
    per_layer: list = field(default_factory=list)
    totals: dict = field(default_factory=dict)
    per_iteration_totals: list = field(default_factory=list)
    max_over_iterations: int = 0
    aside: dict = field(default_factory=dict)

    def to_dict(self) -> dict:
        c = self.config
        return {"model": {"blocks": c.blocks, "hidden": c.hidden, "heads": c.heads,
                          "max_seq": c.max_seq, "num_classes": c.num_classes},
                "batch_size": self.batch_size, "freeze_rate": self.freeze_rate,
                "records": [{"name": n, "kind": k, "bytes": b} for n, k, b in self.per_layer],
                "totals": dict(self.totals), "per_iteration_totals": list(self.per_iteration_totals),
                "max_over_iterations": self.max_over_iterations, "aside": dict(self.aside)}


def _block_records(i: int, B: int, Tn: int, H: int, heads: int) -> list[ActivationRecord]:
    p, base, BTH = f"encoder.layer.{i}", 4 + 8 * i, B * Tn * H
    R = ActivationRecord
    return [
        R(f"{p}.attention.self.query.input", "dynamic", BTH, base + 0),
        R(f"{p}.attention.self.key.input", "dynamic", BTH, base + 1),
        R(f"{p}.attention.self.value.input", "dynamic", BTH, base + 2),
        R(f"{p}.attention.scores.lhs", "static", BTH, None, "matsoft8"),
        R(f"{p}.attention.scores.rhs", "static", BTH, None, "matsoft8"),
        R(f"{p}.attention.softmax.probs", "static", B * heads * Tn * Tn, None, "matsoft8"),
        R(f"{p}.attention.context.rhs", "static", BTH, None, "matsoft8"),
        R(f"{p}.attention.output.dense.input", "dynamic", BTH, base + 3),
        R(f"{p}.attention.output.LayerNorm.xtilde", "semi_static", BTH, base + 4, "ln_prune"),
        R(f"{p}.attention.output.LayerNorm.rstd", "static", B * Tn, None),
        R(f"{p}.intermediate.dense.input", "dynamic", BTH, base + 5),
        R(f"{p}.intermediate.gelu.input", "static", 4 * BTH, None, "gelu4"),
        R(f"{p}.output.dense.input", "dynamic", 4 * BTH, base + 6, "dense8"),
        R(f"{p}.output.LayerNorm.xtilde", "semi_static", BTH, base + 7, "ln_prune"),
        R(f"{p}.output.LayerNorm.rstd", "static", B * Tn, None),
    ]


def enumerate_records(config: ModelConfig, batch_size: int) -> list[ActivationRecord]:
    """All buffers one forward caches, in forward order (memory.py:87-133)."""
    B, Tn, H, C = batch_size, config.max_seq, config.hidden, config.num_classes
    n = registry_size(config.blocks)
    R = ActivationRecord
    recs = [R("embeddings.word_embeddings.ids", "dynamic", B * Tn, 0, "int32"),
            R("embeddings.LayerNorm.xtilde", "semi_static", B * Tn * H, 3, "ln_prune"),
            R("embeddings.LayerNorm.rstd", "static", B * Tn, None)]
    for i in range(config.blocks):
        recs += _block_records(i, B, Tn, H, config.heads)
    recs += [R("pooler.dense.input", "dynamic", B * H, n - 2),
             R("pooler.tanh.output", "static", B * H, None),
             R("classifier.input", "dynamic", B * H, n - 1),
             R("loss.probs", "static", B * C, None),
             R("loss.labels", "static", B, None, "int32")]
    return recs


def block_trainable_counts(config: ModelConfig, batch_size: int) -> list[tuple[str, int]]:
    """Input element counts of one block's eight trainable layers."""
    BTH = batch_size * config.max_seq * config.hidden
    return [("attention.self.query", BTH), ("attention.self.key", BTH), ("attention.self.value", BTH),
            ("attention.output.dense", BTH), ("attention.output.LayerNorm", BTH),
            ("intermediate.dense", BTH), ("output.dense", 4 * BTH), ("output.LayerNorm", BTH)]


def imbalance_ratio(config: ModelConfig) -> float:
    c = [n for _, n in block_trainable_counts(config, 1)]
    return max(c) / min(c)


def imbalance_byte_ratio(config: ModelConfig, codecs: CompressionConfig) -> float:
    BTH = config.max_seq * config.hidden
    wide = ActivationRecord("output.dense.input", "dynamic", 4 * BTH, 0, "dense8")
    narrow = ActivationRecord("intermediate.dense.input", "dynamic", BTH, 0)
    return wide.bytes_under(codecs, False) / narrow.bytes_under(codecs, False)


def parameter_aside(config: ModelConfig) -> dict:
    """Weight / gradient / moment bytes, reported beside the activations."""
    H, I, V = config.hidden, config.intermediate, config.vocab
    block = 4 * (H * H + H) + 2 * (2 * H) + (H * I + I) + (I * H + H)
    emb = V * H + config.max_seq * H + config.type_vocab * H + 2 * H
    head = (H * H + H) + (H * config.num_classes + config.num_classes)
    n = emb + config.blocks * block + head
    return {"parameter_bytes": n * BYTES_F32, "gradient_bytes": n * BYTES_F32,
            "optimizer_moment_bytes": n * BYTES_ADAM_MOMENTS}


def account_iteration(config: ModelConfig, batch_size: int, decision: FreezeDecision,
                      codecs: CompressionConfig | None = None) -> MemoryReport:
    """Bytes cached in one iteration under a freeze decision (memory.py:166-191)."""
    frozen = decision.frozen_ids
    totals = {"dynamic": 0, "static": 0, "semi_static": 0}
    per = []
    for r in enumerate_records(config, batch_size):
        fz = r.layer_id is not None and r.layer_id in frozen
        if r.kind == "dynamic" and fz:
            continue
        b = r.bytes_under(codecs, fz)
        per.append((r.name, r.kind, b))
        totals[r.kind] += b
    totals["activations_total"] = totals["dynamic"] + totals["static"] + totals["semi_static"]
    n = registry_size(config.blocks)
    return MemoryReport(config, batch_size, len(frozen) / max(1, n), per, totals,
                        [totals["activations_total"]], totals["activations_total"],
                        parameter_aside(config))


def budget_decision(config: ModelConfig, freeze_rate: float) -> FreezeDecision:
    """Worst case at a rate: the cheapest layers freeze first (memory.py:212-231)."""
    n = registry_size(config.blocks)
    cost = np.zeros(n)
    for r in enumerate_records(config, 1):
        if r.layer_id is None:
            continue
        if r.kind == "dynamic":
            cost[r.layer_id] += r.count * BYTES_F32
        elif r.kind == "semi_static":
            cost[r.layer_id] += r.count * BYTES_F32 * 0.8
    fz = frozenset(int(i) for i in np.argsort(cost, kind="stable")[:frozen_count(n, freeze_rate)])
    return FreezeDecision(0, fz, frozenset(range(n)) - fz)


def account_budget(config: ModelConfig, batch_size: int, freeze_rate: float,
                   codecs: CompressionConfig | None = None) -> MemoryReport:
    rep = account_iteration(config, batch_size, budget_decision(config, freeze_rate), codecs)
    rep.freeze_rate = freeze_rate
    return rep


def account_schedule(config: ModelConfig, batch_size: int, decisions,
                     codecs: CompressionConfig | None = None) -> MemoryReport:
    decisions = list(decisions)
    if not decisions:
        raise ValueError("account_schedule needs at least one decision")
    reps = [account_iteration(config, batch_size, d, codecs) for d in decisions]
    tot = [r.totals["activations_total"] for r in reps]
    worst = reps[int(np.argmax(tot))]
    worst.per_iteration_totals = tot
    worst.max_over_iterations = max(tot)
    return worst


@dataclass
class AuditResult:
    analytic: dict
    instrumented: dict
    relative_difference: float

    @property
    def within(self) -> float:
        return self.relative_difference


def audit_runtime(config: ModelConfig, batch_size: int, decision: FreezeDecision,
                  codecs: CompressionConfig | None, tape) -> AuditResult:
    """Analytic bytes vs a recorded tape's ledger (memory.py:271-284)."""
    a = account_iteration(config, batch_size, decision, codecs).totals
    m = tape.cached_bytes()
    inst = {"dynamic": m["dynamic"], "static": m["static"], "semi_static": m["semi_static"],
            "activations_total": m["total"]}
    rel = abs(a["activations_total"] - inst["activations_total"]) / max(1, inst["activations_total"])
    return AuditResult(a, inst, rel)
