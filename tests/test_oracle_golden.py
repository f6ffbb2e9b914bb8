"""Pin the CPU oracle to the reference: every golden fixture produced by the
real `slimfit` package (tests/golden/make_golden.py) must be reproduced by the
oracle restatement — bit-exact for codes, indices, decisions and distances,
within float32 round-off for the encoder step (reference test pins:
tests/test_compression.py, test_scheduler.py, test_tensor_ops.py,
test_trainer.py under /root/reference/pkg/)."""

import math

import numpy as np
import pytest

from oracle import codecs as C
from oracle import ils
from oracle import encoder as E


# --------------------------------------------------------------------- codecs

def test_quantize_golden(golden):
    g = golden("codecs.npz")
    x = g["q_x"]
    assert np.array_equal(C.quantize(x, C.Q44), g["q44"])
    assert np.array_equal(C.quantize(x, C.Q08U), g["q08u"])
    assert np.array_equal(C.quantize(np.nan_to_num(x, nan=0.0) / 4.0, C.Q22), g["q22_direct"])
    assert np.array_equal(C.dequantize(g["dq_codes"], C.Q44), g["dq44"])
    assert np.array_equal(C.dequantize(np.arange(256, dtype=np.uint8), C.Q08U), g["dq08u"])


def test_pack4_golden(golden):
    g = golden("codecs.npz")
    assert np.array_equal(C.pack4(g["p4_codes"]), g["p4_packed"])
    assert np.array_equal(C.unpack4(g["p4_packed"], g["p4_codes"].size), g["p4_codes"])


@pytest.mark.parametrize("name", ["n01", "n03", "big", "small", "const14", "zeros", "with_nan",
                                  "with_inf", "one", "odd9", "edge175", "edge35", "adv"])
def test_packed4_golden(golden, name):
    g = golden("codecs.npz")
    x = g[f"pk_{name}_x"]
    packed, s, cnt = C.pack_gelu(x)
    assert s == int(g[f"pk_{name}_s"])
    assert np.array_equal(packed, g[f"pk_{name}_packed"])
    dec = C.unpack_gelu(packed, s, cnt)
    assert np.array_equal(dec, g[f"pk_{name}_dec"])


@pytest.mark.parametrize("name", ["spec", "ties", "signed", "rand", "rand_signed", "quantized_ties",
                                  "zeros_pm", "nan_inf", "nan_signed", "keep_all", "one", "ln_rows"])
def test_prune_golden(golden, name):
    g = golden("codecs.npz")
    x = g[f"pr_{name}_x"]
    vals, idx = C.prune_topk(x, float(g[f"pr_{name}_keep"]), bool(g[f"pr_{name}_mag"]))
    assert np.array_equal(idx, g[f"pr_{name}_idx"])
    assert np.array_equal(vals, g[f"pr_{name}_vals"], equal_nan=True)
    dense = C.restore(vals, idx, x.size, x.shape)
    assert np.array_equal(dense, g[f"pr_{name}_dense"], equal_nan=True)


def test_reference_known_answers():
    # tests/test_compression.py:31-48, :64-71, :86-99, :132-157
    assert C.quantize(np.array([0.5]), C.Q44)[0] == 8
    assert C.quantize(np.array([10.0]), C.Q44)[0] == 127
    assert C.quantize(np.array([0.03125, -0.03125]), C.Q44).tolist() == [1, -1]
    assert C.dequantize(np.array([127], np.int8), C.Q44)[0] == 7.9375
    assert C.pack4(np.array([3, -2])).tolist() == [0xE3]
    assert C.pack4(np.array([7])).tolist() == [0x07]
    assert C.pack4(np.array([], np.int8)).size == 0
    v, i = C.prune_topk(np.array([0.1, -5, 0.2, 3, 0, 0.05, 0.3, -0.4, 0.01, 2], np.float32), 0.1)
    assert v.tolist() == [-5.0] and i.tolist() == [1]
    assert C.prune_topk(np.full(10, 2.5, np.float32), 0.3)[1].tolist() == [0, 1, 2]
    assert C.payload_nbytes("packed4", 9) == 5
    assert C.payload_nbytes("pruned", 20) == 16
    assert C.prescale_exp(np.array([0.5, -0.25], np.float32), C.Q22) == 0
    s = C.prescale_exp(np.full(1000, 14.0, np.float32), C.Q22)
    assert 14.0 / (1 << s) <= C.Q22.vmax
    # k inherits float64 rounding: 0.1 * 12582912 = 1258291.2000000002
    assert C.keep_count(12_582_912, 0.1) == 1_258_292


def test_percentile_matches_numpy():
    rng = np.random.default_rng(5)
    for n in [1, 2, 3, 10, 999, 1000, 1001, 12345]:
        m = np.abs(rng.standard_normal(n))
        assert C.percentile_linear(m, 99.9) == float(np.percentile(m, 99.9))


# ------------------------------------------------------------------------ ILS

def test_init_distances_golden(golden):
    g = golden("ils.npz")
    for seed in (0, 1, 123):
        for n in (4, 22, 102, 198):
            assert np.array_equal(ils.warm_distances(n, seed), g[f"init_{seed}_{n}"])


def test_select_frozen_golden(golden):
    g = golden("ils.npz")
    for t in range(40):
        d = g[f"sel_{t}_d"]
        fz = ils.frozen_ids(d, float(g[f"sel_{t}_f"]), tuple(g[f"sel_{t}_pinned"].tolist()))
        mask = np.zeros(d.size, bool)
        mask[fz] = True
        assert np.array_equal(mask, g[f"sel_{t}_mask"]), t


def test_layer_distance_golden(golden):
    g = golden("ils.npz")
    t = 0
    while f"dist_{t}_d" in g:
        k = int(g[f"dist_{t}_np"])
        before = [g[f"dist_{t}_b{j}"] for j in range(k)]
        after = [g[f"dist_{t}_a{j}"] for j in range(k)]
        assert ils.layer_distance(before, after) == float(g[f"dist_{t}_d"])
        # the restated pairwise tree reproduces numpy's sum bit for bit
        tot = 0.0
        for b, a in zip(before, after):
            tot += ils.pairwise_sum(ils.rel_change(b, a))
        assert tot / sum(b.size for b in before) == float(g[f"dist_{t}_d"])
        t += 1


def test_reference_scheduler_known_answers():
    # tests/test_scheduler.py:42-46, :56-58, :67-69, :79-101
    assert ils.frozen_ids(np.array([5.0, 1.0, 3.0, 2.0]), 0.5) == [1, 3]
    assert len(ils.frozen_ids(ils.warm_distances(10, 0), 0.55)) == 5
    assert ils.frozen_ids(np.array([2.0] * 4), 0.5) == [0, 1]
    assert 0 not in ils.frozen_ids(np.array([0.1, 0.2, 0.3, 0.4]), 0.5, pinned=(0,))
    assert ils.layer_distance([np.array([1.0, 2.0])], [np.array([1.1, 2.2])]) == pytest.approx(0.1, rel=1e-9)
    assert ils.layer_distance([np.ones(2), np.ones(1)], [np.ones(2) * 1.1, np.ones(1) * 1.3]) == \
        pytest.approx(0.5 / 3, rel=1e-9)


def test_adamw_golden(golden):
    g = golden("adamw.npz")
    n = int(g["n_layers"])
    lrs = g["lrs"]
    layers = {}
    lid = 0
    while f"p_0_{lid}_0" in g:
        j = 0
        layers[lid] = []
        while f"p_0_{lid}_{j}" in g:
            layers[lid].append(g[f"p_0_{lid}_{j}"].copy())
            j += 1
        lid += 1
    opt = ils.AdamW()
    for s in range(3):
        grads, active = {}, []
        for lid in layers:
            gl = [g[f"g_{s}_{lid}_{j}"] if f"g_{s}_{lid}_{j}" in g else None
                  for j in range(len(layers[lid]))]
            if any(x is not None for x in gl):
                grads[lid] = gl
                active.append(lid)
            for j in range(len(layers[lid])):
                assert np.array_equal(layers[lid][j], g[f"p_{s}_{lid}_{j}"])
        opt.step(layers, grads, float(lrs[s]), active)
    for lid in layers:
        for j in range(len(layers[lid])):
            assert np.array_equal(layers[lid][j], g[f"p_final_{lid}_{j}"]), (lid, j)
    assert n == len(layers)


# -------------------------------------------------------------------- encoder

STEP_CFG = E.EncoderConfig(blocks=2, hidden=32, heads=4, max_seq=16, vocab=64, num_classes=4)


@pytest.mark.parametrize("tag,codecs", [("plain", None), ("frozen_codecs", E.Codecs.all_on()),
                                        ("codecs", E.Codecs.all_on())])
def test_encoder_step_golden(golden, tag, codecs):
    g = golden("step.npz")
    params = E.init_params(STEP_CFG, seed=3)
    st = E.Step(STEP_CFG, params, g[f"{tag}_frozen"].tolist(), codecs).run(g["ids"], g["labels"])
    np.testing.assert_allclose(st.logits, g[f"{tag}_logits"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(float(st.loss), float(g[f"{tag}_loss"]), rtol=1e-6)
    t = st.ledger.totals()
    assert [t["dynamic"], t["static"], t["semi_static"], t["total"]] == g[f"{tag}_ledger"].tolist()
    seen = set()
    for lid, gl in st.grads.items():
        for j, gr in enumerate(gl):
            key = f"{tag}_g_{lid}_{j}"
            assert key in g, key
            seen.add(key)
            np.testing.assert_allclose(gr, g[key], rtol=2e-4, atol=1e-6, err_msg=key)
    assert seen == {k for k in g.files if k.startswith(f"{tag}_g_")}


def _optimizer(g) -> str:
    return str(g["optimizer"]) if "optimizer" in g.files else "adamw"


@pytest.mark.parametrize("kind", ["sgd", "adamw"])
def test_optimizer_distance_refresh_golden(golden, kind):
    """Reference step + update_distances (trainer.py:194-200) for both
    optimizers: an active layer without gradients gets d = 0.0, a
    gradient-less parameter still counts, frozen entries keep their value;
    bit-exact."""
    g = golden("optim.npz")
    cfg = E.EncoderConfig(blocks=1, hidden=8, heads=2, max_seq=4, vocab=10, num_classes=3)
    params = E.init_params(cfg, seed=13)
    n = cfg.n_layers
    opt = ils.AdamW() if kind == "adamw" else ils.SGD()
    d = g[f"{kind}_d_init"].copy()
    for s in range(3):
        active = g[f"{kind}_active_{s}"].tolist()
        grads = {lid: [g[f"{kind}_g_{s}_{lid}_{j}"] if f"{kind}_g_{s}_{lid}_{j}" in g else None
                       for j in range(len(params[lid]))] for lid in active}
        before = {lid: [p.copy() for p in params[lid]] for lid in active}
        opt.step(params, grads, float(g[f"{kind}_lrs"][s]), active)
        for lid in active:
            d[lid] = ils.layer_distance(before[lid], params[lid])
        assert np.array_equal(d, g[f"{kind}_d_{s}"]), s
        assert [opt.steps.get(i, 0) for i in range(n)] == g[f"{kind}_steps_{s}"].tolist()
    for lid in range(n):
        for j, p in enumerate(params[lid]):
            assert np.array_equal(p, g[f"{kind}_p_final_{lid}_{j}"]), (lid, j)


def _digest_close(gr, g, prefix, rtol):
    """A gradient against its golden digest: exact sample positions within
    rtol of the tensor's scale, sum / sum|.| / max|.| within rtol."""
    flat = np.asarray(gr, np.float64).reshape(-1)
    scale = float(g[prefix + "max"])
    idx = g[prefix + "idx"]
    np.testing.assert_allclose(flat[idx], g[prefix + "val"], rtol=0, atol=rtol * scale + 1e-9,
                               err_msg=prefix)
    np.testing.assert_allclose(np.abs(flat).max(), scale, rtol=rtol, atol=1e-9, err_msg=prefix)
    np.testing.assert_allclose(np.abs(flat).sum(), float(g[prefix + "abs"]), rtol=rtol, atol=1e-9,
                               err_msg=prefix)


@pytest.mark.parametrize("fixture", ["step_vit_b.npz", "step_bert_large.npz"])
def test_wide_step_golden(golden, fixture):
    """The encoder step at the BASELINE configs' width and sequence length
    (T = 197 pre-norm ViT-B/16-shaped, T = 384 BERT-large-shaped): logits,
    loss, ledger and every surviving gradient's digest."""
    g = golden(fixture)
    L, H, nh, T, V, Cn, B, seed, pre = g["cfg"].tolist()
    cfg = E.EncoderConfig(blocks=L, hidden=H, heads=nh, max_seq=T, vocab=V, num_classes=Cn, pre_norm=bool(pre))
    params = E.init_params(cfg, seed)
    st = E.Step(cfg, params, g["frozen"].tolist(), E.Codecs.all_on()).run(g["ids"], g["labels"])
    np.testing.assert_allclose(st.logits, g["logits"], rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(float(st.loss), float(g["loss"]), rtol=1e-5)
    t = st.ledger.totals()
    assert [t["dynamic"], t["static"], t["semi_static"], t["total"]] == g["ledger"].tolist()
    seen = set()
    for lid, gl in st.grads.items():
        for j, gr in enumerate(gl):
            if gr is None:
                continue
            seen.add((lid, j))
            _digest_close(gr, g, f"g_{lid}_{j}_", 2e-3)
    assert seen == {(int(k.split("_")[1]), int(k.split("_")[2])) for k in g.files if k.endswith("_sum")}


FINETUNE_FIXTURES = ["finetune_tiny.npz", "finetune_prenorm.npz", "finetune_sgd.npz", "finetune_vit_b.npz",
                     "finetune_vit_b_sgd.npz", "finetune_bert_large.npz"]


@pytest.mark.parametrize("fixture", FINETUNE_FIXTURES)
def test_finetune_golden(golden, fixture):
    g = golden(fixture)
    L, H, nh, T, V, Cn, B, iters, seed, pre = g["cfg"].tolist()
    cfg = E.EncoderConfig(blocks=L, hidden=H, heads=nh, max_seq=T, vocab=V, num_classes=Cn,
                          pre_norm=bool(pre))
    params = E.init_params(cfg, seed)
    log = E.fine_tune(cfg, params, g["tokens"], g["labels"], freeze_rate=float(g["freeze"]),
                      epochs=1, batch_size=B, seed=seed, lr=float(g["lr"]), warmup_frac=0.0,
                      codecs=E.Codecs.all_on() if bool(g["codecs"]) else None, optimizer=_optimizer(g))
    fm = np.zeros_like(g["frozen"])
    for i, fz in enumerate(log["frozen"]):
        fm[i, fz] = True
    assert np.array_equal(fm, g["frozen"])                      # schedule bit-exact
    np.testing.assert_allclose(log["loss"], g["loss"], rtol=1e-5)
    np.testing.assert_allclose(np.array(log["d"]), g["d"], rtol=1e-3)
    mem = np.array([[i, t["dynamic"], t["static"] + t["semi_static"], t["total"]]
                    for i, t in enumerate(log["ledger"])])
    assert np.array_equal(mem, g["memory"])
    sums = np.array([float(np.sum(p, dtype=np.float64)) for lp in params for p in lp])
    np.testing.assert_allclose(sums, g["param_sums"], rtol=1e-4, atol=1e-6)
