"""Analytic activation accounting vs the reference's (golden memory.npz) and
vs the recorded ledger of the oracle step (reference tests/test_memory.py
pins: BERT-base b32 ~3.2 GB baseline, ~0.5 GB at F=0.95 with codecs, exact
linearity in B, imbalance 4.0, analytic == instrumented)."""

import numpy as np
import pytest

from paper_2305_18513_b200 import memory as M
from paper_2305_18513_b200.model import ModelConfig
from paper_2305_18513_b200.scheduler import FreezeDecision
from paper_2305_18513_b200.tensor import CompressionConfig

CASES = {
    "bert_base_b32": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522, num_classes=2), 32),
    "bert_base_b128": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522, num_classes=2), 128),
    "vit_b_b128": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=197, vocab=1000, num_classes=100,
                               pre_norm=True), 128),
    "bert_large_b16": (ModelConfig(blocks=24, hidden=1024, heads=16, max_seq=384, vocab=30522, num_classes=2), 16),
    "tiny": (ModelConfig(blocks=2, hidden=128, heads=2, max_seq=128, vocab=30522, num_classes=2), 8),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_account_budget_matches_reference(golden, name):
    g = golden("memory.npz")
    cfg, B = CASES[name]
    for F in (0.0, 0.5, 0.75, 0.95):
        for tag, cx in (("none", None), ("all", CompressionConfig.all_on())):
            t = M.account_budget(cfg, B, F, cx).totals
            got = [t["dynamic"], t["static"], t["semi_static"], t["activations_total"]]
            assert got == g[f"{name}_{F}_{tag}"].tolist(), (name, F, tag)
    assert list(M.parameter_aside(cfg).values()) == g[f"{name}_aside"].tolist()
    assert M.imbalance_ratio(cfg) == float(g[f"{name}_imb"])


def test_paper_table_pins():
    cfg, _ = CASES["bert_base_b32"]
    base = M.account_budget(cfg, 32, 0.0).totals["activations_total"]
    slim = M.account_budget(cfg, 32, 0.95, CompressionConfig.all_on()).totals["activations_total"]
    assert abs(base / 1e9 - 3.2) <= 0.25 * 3.2
    assert abs(slim / 1e9 - 0.5) <= 0.30 * 0.5
    a = M.account_budget(cfg, 16, 0.5).totals["activations_total"]
    b = M.account_budget(cfg, 32, 0.5).totals["activations_total"]
    assert 2 * a == b
    assert M.imbalance_ratio(cfg) == 4.0


@pytest.mark.parametrize("tag", ["plain", "frozen_codecs", "codecs"])
def test_analytic_equals_recorded_ledger(golden, tag):
    g = golden("step.npz")
    cfg = ModelConfig(blocks=2, hidden=32, heads=4, max_seq=16, vocab=64, num_classes=4)
    fz = frozenset(int(i) for i in g[f"{tag}_frozen"])
    n = 4 + 8 * 2 + 2
    dec = FreezeDecision(0, fz, frozenset(range(n)) - fz)
    cx = None if tag == "plain" else CompressionConfig.all_on()
    t = M.account_iteration(cfg, 4, dec, cx).totals
    assert [t["dynamic"], t["static"], t["semi_static"], t["activations_total"]] == g[f"{tag}_ledger"].tolist()


def test_schedule_takes_the_max():
    cfg, B = CASES["tiny"]
    n = 4 + 8 * 2 + 2
    decs = [FreezeDecision(i, frozenset(range(i)), frozenset(range(i, n))) for i in (0, 5, 10)]
    rep = M.account_schedule(cfg, B, decs, CompressionConfig.all_on())
    assert rep.max_over_iterations == max(rep.per_iteration_totals) == rep.per_iteration_totals[0]
