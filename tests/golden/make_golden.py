"""Generate the golden fixtures that pin the oracle (and, through it, the
device kernels) to the reference package.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports `slimfit` read-only, calls the reference's own public functions on
seeded inputs, and writes small `.npz` files next to this script.  Nothing on
the GPU box reads /root/reference; only these committed outputs travel.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True          # never write __pycache__ into the reference tree
sys.path.insert(0, "/root/reference/pkg/src")

import slimfit  # noqa: E402
from slimfit import compression as RC  # noqa: E402
from slimfit import scheduler as RS  # noqa: E402
from slimfit import tensor as RT  # noqa: E402
from slimfit.model import Batch, ModelConfig, build_model  # noqa: E402
from slimfit.trainer import OptimizerState, RunConfig, fine_tune  # noqa: E402


def adversarial_f32(rng, n=4096):
    """Half ties at k/32 and k/8, saturating values, +-0, +-inf, NaN, values at
    and around 1.75*2^k, subnormals, plus normal draws."""
    ties = np.arange(-300, 301, dtype=np.float64) / 32.0
    ties4 = np.arange(-80, 81, dtype=np.float64) / 8.0
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e30, -1e30, 8.0, -8.0,
                        7.96875, -8.03125, 0.49999997, -0.49999997, 1e-40, -1e-45])
    pw = np.array([1.75 * 2.0 ** k for k in range(-4, 12)])
    near = np.concatenate([pw, np.nextafter(pw.astype(np.float32), np.float32(np.inf)),
                           np.nextafter(pw.astype(np.float32), np.float32(0))])
    body = rng.standard_normal(n) * 3
    x = np.concatenate([ties, -ties[::-1], ties4, special, near, -near, body])
    return x.astype(np.float32)


def codec_fixtures(rng):
    out = {}
    x = adversarial_f32(rng)
    out["q_x"] = x
    out["q44"] = RC.quantize(x, RC.Q4_4)
    out["q08u"] = RC.quantize(x, RC.Q0_8_UNSIGNED)
    out["q22_direct"] = RC.quantize(np.nan_to_num(x, nan=0.0) / 4.0, RC.Q2_2)
    codes8 = np.arange(-128, 128, dtype=np.int8)
    out["dq_codes"] = codes8
    out["dq44"] = RC.dequantize(codes8, RC.Q4_4)
    ucodes = np.arange(0, 256, dtype=np.uint8)
    out["dq08u"] = RC.dequantize(ucodes, RC.Q0_8_UNSIGNED)
    c4 = rng.integers(-8, 8, size=1001).astype(np.int8)
    out["p4_codes"] = c4
    out["p4_packed"] = np.frombuffer(RC.pack4(c4), dtype=np.uint8)

    # packed4 (prescale + pack) on a family of inputs
    cases = {
        "n01": rng.standard_normal(10007).astype(np.float32),
        "n03": (rng.standard_normal(20011) * 3).astype(np.float32),
        "big": (rng.standard_normal(5000) * 300).astype(np.float32),
        "small": (rng.standard_normal(777) * 0.1).astype(np.float32),
        "const14": np.full(1000, 14.0, np.float32),
        "zeros": np.zeros(64, np.float32),
        "with_nan": np.concatenate([rng.standard_normal(99), [np.nan]]).astype(np.float32),
        "with_inf": np.concatenate([rng.standard_normal(5000), [np.inf]]).astype(np.float32),
        "one": np.array([3.5], np.float32),
        "odd9": np.linspace(-1, 1, 9, dtype=np.float32),
        "edge175": np.full(2000, 1.75, np.float32),
        "edge35": np.concatenate([np.full(1000, 3.5), np.full(1000, 3.5000002)]).astype(np.float32),
        "adv": x[np.isfinite(x)],
    }
    for name, arr in cases.items():
        ca = RC.CompressedActivation.packed(arr, RC.Q2_2)
        out[f"pk_{name}_x"] = arr
        out[f"pk_{name}_s"] = np.int64(ca.prescale_exp)
        out[f"pk_{name}_packed"] = np.frombuffer(ca.packed_codes, dtype=np.uint8)
        out[f"pk_{name}_dec"] = ca.decompress()

    # prune
    pcases = {
        "spec": (np.array([0.1, -5, 0.2, 3, 0, 0.05, 0.3, -0.4, 0.01, 2], np.float32), 0.1, True),
        "ties": (np.full(10, 2.5, np.float32), 0.3, True),
        "signed": (np.array([-5.0, 4.0, 1.0, 0.0], np.float32), 0.25, False),
        "rand": (rng.standard_normal(50000).astype(np.float32), 0.1, True),
        "rand_signed": (rng.standard_normal(30001).astype(np.float32), 0.1, False),
        "quantized_ties": (np.round(rng.standard_normal(20000) * 4).astype(np.float32) / 4, 0.1, True),
        "zeros_pm": (np.where(rng.random(1000) < 0.5, 0.0, -0.0).astype(np.float32), 0.2, True),
        "nan_inf": (np.concatenate([[np.nan, np.inf, -np.inf, np.nan], rng.standard_normal(96)]).astype(np.float32), 0.5, True),
        "nan_signed": (np.concatenate([[np.nan, -np.inf, 1.0], rng.standard_normal(97)]).astype(np.float32), 0.99, False),
        "keep_all": (np.linspace(-1, 1, 12, dtype=np.float32), 1.0, True),
        "one": (np.array([7.0], np.float32), 0.1, True),
        "ln_rows": (None, 0.1, True),
    }
    xt = rng.standard_normal((16, 64)).astype(np.float32)
    xt = (xt - xt.mean(axis=-1, keepdims=True)) / xt.std(axis=-1, keepdims=True)
    pcases["ln_rows"] = (xt.astype(np.float32), 0.1, True)
    for name, (arr, keep, mag) in pcases.items():
        sp = RC.prune_topk(arr, keep, mag)
        out[f"pr_{name}_x"] = arr
        out[f"pr_{name}_keep"] = np.float64(keep)
        out[f"pr_{name}_mag"] = np.bool_(mag)
        out[f"pr_{name}_vals"] = sp.values
        out[f"pr_{name}_idx"] = sp.indices
        out[f"pr_{name}_dense"] = RC.restore(sp)
    return out


def ils_fixtures(rng):
    out = {}
    for seed in (0, 1, 123):
        for n in (4, 22, 102, 198):
            out[f"init_{seed}_{n}"] = RS.init_distances(n, seed).d
    sel = []
    for t in range(40):
        n = int(rng.integers(1, 60))
        d = rng.choice([1.0, 2.0, 3.0, 0.5], size=n) if t % 3 == 0 else rng.random(n) * 10
        f = float(rng.choice([0.0, 0.25, 0.5, 0.55, 0.75, 0.95]))
        pinned = tuple(int(i) for i in rng.choice(n, size=min(2, n), replace=False)) if t % 4 == 0 else ()
        dv = RS.DistanceVector(d.astype(np.float64), np.ones(n, bool))
        dec = RS.select_frozen(dv, f, pinned_active=pinned)
        mask = np.zeros(n, bool)
        mask[list(dec.frozen_ids)] = True
        out[f"sel_{t}_d"] = d.astype(np.float64)
        out[f"sel_{t}_f"] = np.float64(f)
        out[f"sel_{t}_pinned"] = np.array(pinned, np.int64)
        out[f"sel_{t}_mask"] = mask
    # layer distances over BERT-ish and odd shapes, zero-init biases included
    dshapes = [[(37,), (5,)], [(128, 512), (512,)], [(768,), (768,)], [(1000, 3)], [(300, 129), (129,)],
               [(4099,)], [(64, 64), (64,)]]
    for t, shapes in enumerate(dshapes):
        before, after = [], []
        for j, shp in enumerate(shapes):
            if j == 1 and len(shp) == 1:
                b = np.zeros(shp, np.float32)
                b[::3] = rng.standard_normal(b[::3].shape).astype(np.float32) * 0.02
            else:
                b = (rng.standard_normal(shp) * 0.02).astype(np.float32)
            a = (b - 1e-4 * np.sign(rng.standard_normal(shp))).astype(np.float32)
            a[..., ::7] = b[..., ::7]
            before.append(b)
            after.append(a)
            out[f"dist_{t}_b{j}"] = b
            out[f"dist_{t}_a{j}"] = a
        out[f"dist_{t}_np"] = np.int64(len(shapes))
        out[f"dist_{t}_d"] = np.float64(RS.layer_distance(before, after))
    return out


def adamw_fixture(rng):
    """Reference OptimizerState.step on a tiny model with synthetic grads,
    three steps with a pause for layer 1 at step 2."""
    cfg = ModelConfig(blocks=1, hidden=8, heads=2, max_seq=4, vocab=10, num_classes=3)
    m = build_model(cfg, seed=11)
    opt = OptimizerState(kind="adamw")
    out = {}
    n = len(m.registry)
    sched = [list(range(n)), [i for i in range(n) if i != 1], list(range(n))]
    for s, active in enumerate(sched):
        for e in m.registry:
            for j, p in enumerate(e.params):
                if e.layer_id in active:
                    g = (rng.standard_normal(p.data.shape) * 0.1).astype(np.float32)
                    p.grad = g
                    out[f"g_{s}_{e.layer_id}_{j}"] = g
                else:
                    p.grad = None
        for e in m.registry:
            for j, p in enumerate(e.params):
                out[f"p_{s}_{e.layer_id}_{j}"] = p.data.copy()
        opt.step(m, [1e-3, 5e-4, 2e-3][s], active)
    for e in m.registry:
        for j, p in enumerate(e.params):
            out[f"p_final_{e.layer_id}_{j}"] = p.data.copy()
    out["lrs"] = np.array([1e-3, 5e-4, 2e-3])
    out["n_layers"] = np.int64(n)
    return out


def optim_fixture(rng):
    """Reference OptimizerState.step followed by the reference's distance
    refresh (trainer.py:194-200: clone_layer_data, step, update_distances)
    for both optimizers, three steps on a tiny model.  The active set
    includes a layer whose parameters have no gradient at all (it does not
    move: d = 0.0) and a layer with one gradient-less parameter (counted,
    contributes 0); a frozen layer keeps its distance."""
    cfg = ModelConfig(blocks=1, hidden=8, heads=2, max_seq=4, vocab=10, num_classes=3)
    out = {}
    for kind, lrs in (("sgd", [1e-2, 5e-3, 2e-2]), ("adamw", [1e-3, 5e-4, 2e-3])):
        m = build_model(cfg, seed=13)
        n = len(m.registry)
        opt = OptimizerState(kind=kind)
        dv = RS.init_distances(n, 5)
        out[f"{kind}_d_init"] = dv.d.copy()
        # step s: active = all but `frozen[s]`; `nograd[s]` active without grads;
        # `halfgrad[s]` active with its second parameter gradient-less
        frozen, nograd, halfgrad = [2, 7, 2], [5, 3, 9], [4, 10, 6]
        for s in range(3):
            active = [i for i in range(n) if i != frozen[s]]
            for e in m.registry:
                for j, p in enumerate(e.params):
                    if e.layer_id in active and e.layer_id != nograd[s] and not (
                            e.layer_id == halfgrad[s] and j == 1):
                        g = (rng.standard_normal(p.data.shape) * 0.1).astype(np.float32)
                        p.grad = g
                        out[f"{kind}_g_{s}_{e.layer_id}_{j}"] = g
                    else:
                        p.grad = None
            before = m.clone_layer_data(active)
            opt.step(m, lrs[s], active)
            after = {lid: [p.data for p in m.registry.by_id(lid).params] for lid in active}
            RS.update_distances(dv, before, after, active)
            out[f"{kind}_active_{s}"] = np.array(active, np.int64)
            out[f"{kind}_d_{s}"] = dv.d.copy()
            out[f"{kind}_mask_{s}"] = dv.initialized_mask.copy()
            out[f"{kind}_steps_{s}"] = np.array([opt.layer_steps.get(i, 0) for i in range(n)], np.int64)
        for e in m.registry:
            for j, p in enumerate(e.params):
                out[f"{kind}_p_final_{e.layer_id}_{j}"] = p.data.copy()
        out[f"{kind}_lrs"] = np.array(lrs)
    return out


def _grad_digest(g: np.ndarray, rng) -> dict:
    """A large gradient as a few exact statistics plus sampled entries: the
    full tensors of a 768/1024-wide model would be tens of MB."""
    flat = g.reshape(-1)
    idx = np.sort(rng.choice(flat.size, size=min(flat.size, 256), replace=False)).astype(np.int64)
    return {"sum": np.float64(np.sum(flat, dtype=np.float64)),
            "abs": np.float64(np.sum(np.abs(flat), dtype=np.float64)),
            "max": np.float64(np.abs(flat).max()),
            "idx": idx, "val": flat[idx].copy()}


def wide_step_fixture(name, blocks, hidden, heads, seq, vocab, classes, batch, pre_norm, frozen, seed):
    """One recorded forward/backward with every codec on at a BASELINE
    config's real width and sequence length (few blocks, small batch):
    T = 197 pre-norm (ViT-B/16-shaped) or T = 384 (BERT-large-shaped).
    Loss, logits, ledger and per-gradient digests."""
    cfg = ModelConfig(blocks=blocks, hidden=hidden, heads=heads, max_seq=seq, vocab=vocab,
                      num_classes=classes, pre_norm=pre_norm)
    rng = np.random.default_rng(seed + 77)
    ids = rng.integers(0, vocab, size=(batch, seq))
    labels = rng.integers(0, classes, size=batch)
    m = build_model(cfg, seed=seed)
    m.freeze_set(frozen)
    with RT.record(RT.CompressionConfig.all_on()) as tape:
        logits = m.forward(Batch(ids, labels))
        loss = RT.cross_entropy(logits, labels)
        RT.backward(loss)
    cb = tape.cached_bytes()
    out = {"cfg": np.array([blocks, hidden, heads, seq, vocab, classes, batch, seed, int(pre_norm)]),
           "ids": ids, "labels": labels, "frozen": np.array(frozen, np.int64),
           "loss": np.float32(loss.data), "logits": logits.data,
           "ledger": np.array([cb["dynamic"], cb["static"], cb["semi_static"], cb["total"]])}
    drng = np.random.default_rng(seed + 78)
    for e in m.registry:
        for j, p in enumerate(e.params):
            if p.grad is not None:
                for k, v in _grad_digest(p.grad, drng).items():
                    out[f"g_{e.layer_id}_{j}_{k}"] = v
    return out


def step_fixture():
    """One recorded forward/backward of a small model: loss, logits, every
    surviving grad, and the ledger, for a frozen set with all codecs on."""
    cfg = ModelConfig(blocks=2, hidden=32, heads=4, max_seq=16, vocab=64, num_classes=4)
    rng = np.random.default_rng(7)
    ids = rng.integers(0, 64, size=(4, 16))
    labels = rng.integers(0, 4, size=4)
    out = {"ids": ids, "labels": labels}
    for tag, frozen, codecs in [("plain", [], None),
                                ("frozen_codecs", [1, 5, 8, 9, 12, 14, 17, 19], RT.CompressionConfig.all_on()),
                                ("codecs", [], RT.CompressionConfig.all_on())]:
        m = build_model(cfg, seed=3)
        m.freeze_set(frozen)
        with RT.record(codecs) as tape:
            logits = m.forward(Batch(ids, labels))
            loss = RT.cross_entropy(logits, labels)
            RT.backward(loss)
        out[f"{tag}_frozen"] = np.array(frozen, np.int64)
        out[f"{tag}_loss"] = np.float32(loss.data)
        out[f"{tag}_logits"] = logits.data
        cb = tape.cached_bytes()
        out[f"{tag}_ledger"] = np.array([cb["dynamic"], cb["static"], cb["semi_static"], cb["total"]])
        for e in m.registry:
            for j, p in enumerate(e.params):
                if p.grad is not None:
                    out[f"{tag}_g_{e.layer_id}_{j}"] = p.grad
    return out


def finetune_fixture(blocks, hidden, heads, seq, vocab, classes, batch, iters, freeze, codecs, seed,
                     pre_norm=False, lr=1e-3, optimizer="adamw"):
    cfg = ModelConfig(blocks=blocks, hidden=hidden, heads=heads, max_seq=seq, vocab=vocab,
                      num_classes=classes, pre_norm=pre_norm)
    rng = np.random.default_rng(1000 + seed)
    tokens = rng.integers(0, vocab, size=(batch * iters, seq))
    labels = rng.integers(0, classes, size=batch * iters)
    m = build_model(cfg, seed=seed)
    rc = RunConfig(scheduler="ils", freeze_rate=freeze, epochs=1, batch_size=batch, seed=seed,
                   lr=lr, warmup_frac=0.0, compression=codecs, track_memory=True, optimizer=optimizer)
    log = fine_tune(m, (tokens, labels), rc)
    n = len(m.registry)
    out = {"cfg": np.array([blocks, hidden, heads, seq, vocab, classes, batch, iters, seed, int(pre_norm)]),
           "freeze": np.float64(freeze), "lr": np.float64(lr), "optimizer": np.str_(optimizer),
           "codecs": np.bool_(codecs is not None),
           "tokens": tokens.astype(np.int32), "labels": labels.astype(np.int32),
           "loss": np.array([mm[1] for mm in log.metrics]),
           "d": log.distance_matrix(),
           "memory": np.array(log.memory, dtype=np.int64)}
    fm = np.zeros((len(log.decisions), n), bool)
    for i, dec in enumerate(log.decisions):
        fm[i, list(dec.frozen_ids)] = True
    out["frozen"] = fm
    out["param_sums"] = np.array([float(np.sum(p.data, dtype=np.float64)) for p in m.parameters()])
    return out


def memory_fixture():
    """Reference analytic accounting (memory.py) at the BASELINE shapes."""
    from slimfit import memory as RM
    out = {}
    cases = {
        "bert_base_b32": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522,
                                      num_classes=2), 32),
        "bert_base_b128": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522,
                                       num_classes=2), 128),
        "vit_b_b128": (ModelConfig(blocks=12, hidden=768, heads=12, max_seq=197, vocab=1000,
                                   num_classes=100, pre_norm=True), 128),
        "bert_large_b16": (ModelConfig(blocks=24, hidden=1024, heads=16, max_seq=384, vocab=30522,
                                       num_classes=2), 16),
        "tiny": (ModelConfig(blocks=2, hidden=128, heads=2, max_seq=128, vocab=30522, num_classes=2), 8),
    }
    for name, (cfg, B) in cases.items():
        for F in (0.0, 0.5, 0.75, 0.95):
            for tag, cx in (("none", None), ("all", RT.CompressionConfig.all_on())):
                rep = RM.account_budget(cfg, B, F, cx)
                t = rep.totals
                out[f"{name}_{F}_{tag}"] = np.array([t["dynamic"], t["static"], t["semi_static"],
                                                    t["activations_total"]], dtype=np.int64)
        out[f"{name}_aside"] = np.array(list(RM.parameter_aside(cfg).values()), dtype=np.int64)
        out[f"{name}_imb"] = np.float64(RM.imbalance_ratio(cfg))
    return out


def main(only=()):
    """Write every fixture, or only the named ones (`make_golden.py optim
    finetune_sgd`).  Fixtures added after round 1 draw from their own
    generators, so generating a subset reproduces the same bytes."""
    rng = np.random.default_rng(2305_18513)
    meta = {"numpy": np.__version__, "slimfit": slimfit.__version__}
    print("reference", meta)
    on = RT.CompressionConfig.all_on
    jobs = [
        ("memory", lambda: memory_fixture()),
        ("codecs", lambda: codec_fixtures(rng)),
        ("ils", lambda: ils_fixtures(rng)),
        ("adamw", lambda: adamw_fixture(rng)),
        ("step", lambda: step_fixture()),
        # BASELINE configs[0]: tiny BERT L2 H128 (2 heads) on 8x128 token batches, all codecs, F = 0.5
        ("finetune_tiny", lambda: finetune_fixture(2, 128, 2, 128, 30522, 2, 8, 6, 0.5, on(), seed=0)),
        # a small pre-norm (ViT-like) run without codecs, F = 0.25
        ("finetune_prenorm", lambda: finetune_fixture(2, 32, 4, 16, 64, 4, 8, 6, 0.25, None, seed=4,
                                                      pre_norm=True)),
        # optimizer step + distance refresh for SGD and AdamW, incl. gradient-less active layers
        ("optim", lambda: optim_fixture(np.random.default_rng(2305_18513 + 1))),
        # ILS with SGD: configs[0] shape, all codecs (the distance refresh runs for every optimizer)
        ("finetune_sgd", lambda: finetune_fixture(2, 128, 2, 128, 30522, 2, 8, 6, 0.5, on(), seed=2,
                                                  lr=5e-2, optimizer="sgd")),
        # BASELINE configs[2]/[4]-shaped: ViT (pre-norm, T = 197, 1000-entry
        # patch vocab, 100 classes) at full width H = 768, 2 blocks, batch 2
        ("step_vit_b", lambda: wide_step_fixture("vit_b", 2, 768, 12, 197, 1000, 100, 2, True,
                                                 [1, 5, 8, 12, 14, 17, 19], seed=21)),
        # BASELINE configs[3]-shaped: BERT-large width H = 1024, 16 heads, T = 384
        ("step_bert_large", lambda: wide_step_fixture("bert_large", 2, 1024, 16, 384, 30522, 2, 2, False,
                                                      [0, 2, 3, 6, 9, 11, 13, 15, 20], seed=22)),
        ("finetune_vit_b", lambda: finetune_fixture(2, 768, 12, 197, 1000, 100, 2, 5, 0.75, on(), seed=23,
                                                    pre_norm=True, lr=5e-5)),
        ("finetune_vit_b_sgd", lambda: finetune_fixture(2, 768, 12, 197, 1000, 100, 2, 5, 0.75, on(), seed=25,
                                                        pre_norm=True, lr=1e-2, optimizer="sgd")),
        ("finetune_bert_large", lambda: finetune_fixture(2, 1024, 16, 384, 30522, 2, 2, 5, 0.75, on(), seed=30,
                                                         lr=5e-5)),
    ]
    for name, make in jobs:
        if only and name not in only:
            if name in ("codecs", "ils", "adamw"):
                make()                       # keep the shared generator's sequence
            continue
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **make(), numpy_version=np.__version__)
        print("wrote", name)
    print("done")


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))
