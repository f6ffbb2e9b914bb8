"""BASELINE configs[2]-[4] code paths at their real width and sequence
length: ViT-B/16-shaped (pre-norm, T = 197, 1000-entry vocab, 100 classes,
H = 768) and BERT-large-shaped (H = 1024, 16 heads, T = 384), two blocks,
batch 2 — against the reference's own step (tests/golden/step_*.npz), and
every codec payload those steps write checked bit for bit against the
oracle codecs on the very tensors the step encoded.

Bars: logits / loss / gradient digests within float32 tolerance (2e-3 of
each tensor's scale: cuBLAS-class vs OpenBLAS accumulation order); ledger
byte-identical; codes, packed bytes, prescale exponents, pruned (index,
value) pairs bit-exact.
"""

import numpy as np
import pytest
import torch

from conftest import cuda_ok
from oracle import codecs as C

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

GRAD_RTOL = 2e-3


@pytest.fixture(scope="module")
def sf():
    torch.backends.cuda.matmul.allow_tf32 = False
    import paper_2305_18513_b200 as sf
    return sf


def _digest_close(gr, g, prefix, rtol):
    flat = np.asarray(gr, np.float64).reshape(-1)
    scale = float(g[prefix + "max"])
    idx = g[prefix + "idx"]
    err = np.abs(flat[idx] - g[prefix + "val"]).max()
    assert err <= rtol * scale + 1e-9, (prefix, err, scale)
    assert abs(np.abs(flat).max() - scale) <= rtol * scale + 1e-9, prefix
    assert abs(np.abs(flat).sum() - float(g[prefix + "abs"])) <= rtol * float(g[prefix + "abs"]) + 1e-9, prefix


class Capture:
    """Records (input, payload) of every codec the step runs: all encoders
    go through CompressedActivation.encode_async, the fused softmax codes
    through tensor._Softmax.forward."""

    def __init__(self, sf, monkeypatch):
        from paper_2305_18513_b200 import compression as Cz
        from paper_2305_18513_b200 import tensor as T_
        self.items = []
        orig_enc = Cz.CompressedActivation.encode_async.__func__
        items = self.items

        def enc(cls, fn, *inputs):
            x = inputs[0].detach().clone()
            ca = orig_enc(cls, fn, *inputs)
            items.append(("enc", x, ca))
            return ca

        monkeypatch.setattr(Cz.CompressedActivation, "encode_async", classmethod(enc))
        orig_sm = T_._Softmax.forward

        def sm(ctx, s, scale, quant, spec, name, box):
            probs = orig_sm(ctx, s, scale, quant, spec, name, box)
            if quant:
                items.append(("softmax", s.detach().clone(), (probs.detach().clone(), ctx.sv.value.codes.clone(),
                                                              scale)))
            return probs

        monkeypatch.setattr(T_._Softmax, "forward", staticmethod(sm))

    def check(self):
        seen = {"quant8": 0, "packed4": 0, "pruned": 0, "softmax": 0}
        for kind, x, payload in self.items:
            xn = x.cpu().numpy()
            if kind == "softmax":
                probs, codes, scale = payload
                p = probs.cpu().numpy()
                assert np.array_equal(codes.cpu().numpy(), C.quantize(p, C.Q44))   # codes of its own probs
                z = xn * np.float32(scale)
                e = np.exp(z - z.max(-1, keepdims=True))
                want = e / e.sum(-1, keepdims=True)
                assert np.abs(p - want).max() <= 1e-5 * np.abs(want).max() + 1e-7
                seen["softmax"] += 1
                continue
            ca = payload.wait()
            torch.cuda.synchronize()
            if ca.tag == "quant8":
                fmt = C.Q44
                assert np.array_equal(ca.codes.cpu().numpy().reshape(-1), C.quantize(xn, fmt).reshape(-1))
            elif ca.tag == "packed4":
                packed, s, _ = C.pack_gelu(xn.reshape(-1))
                assert int(ca.prescale_exp_dev.item()) == s
                assert np.array_equal(ca.packed_codes.cpu().numpy(), packed)
            elif ca.tag == "pruned":
                vals, idx = C.prune_topk(xn, 0.1, True)
                assert np.array_equal(ca.sparse.indices.cpu().numpy(), idx)
                assert np.array_equal(ca.sparse.values.cpu().numpy(), vals)
            seen[ca.tag] += 1
        return seen


@pytest.mark.parametrize("fixture", ["step_vit_b.npz", "step_bert_large.npz"])
def test_wide_step_vs_golden_and_codecs(golden, sf, monkeypatch, fixture):
    g = golden(fixture)
    L, H, nh, T, V, Cn, B, seed, pre = g["cfg"].tolist()
    cfg = sf.ModelConfig(blocks=L, hidden=H, heads=nh, max_seq=T, vocab=V, num_classes=Cn, pre_norm=bool(pre))
    m = sf.build_model(cfg, seed=seed)
    frozen = g["frozen"].tolist()
    m.freeze_set(frozen)
    cap = Capture(sf, monkeypatch)
    labels = torch.as_tensor(g["labels"]).cuda()
    with sf.tensor.record(sf.CompressionConfig.all_on()) as tape:
        logits = m.forward(sf.Batch(g["ids"], g["labels"]))
        loss = sf.tensor.cross_entropy(logits, labels)
        sf.tensor.backward(loss)
    torch.cuda.synchronize()
    lg = logits.detach().cpu().numpy()
    assert np.abs(lg - g["logits"]).max() <= 1e-3 * np.abs(g["logits"]).max() + 1e-5
    assert abs(float(loss) - float(g["loss"])) <= 1e-4 * abs(float(g["loss"]))
    cb = tape.cached_bytes()
    assert [cb["dynamic"], cb["static"], cb["semi_static"], cb["total"]] == g["ledger"].tolist()
    want_keys = {(int(k.split("_")[1]), int(k.split("_")[2])) for k in g.files if k.endswith("_sum")}
    got_keys = set()
    for e in m.registry:
        for j, p in enumerate(e.params):
            if p.grad is None:
                continue
            got_keys.add((e.layer_id, j))
            _digest_close(p.grad.cpu().numpy(), g, f"g_{e.layer_id}_{j}_", GRAD_RTOL)
    assert got_keys == want_keys
    for lid in frozen:
        assert all(p.grad is None for p in m.registry.by_id(lid).params)
    seen = cap.check()
    # every codec family ran at this shape: dense8 / matsoft8 codes, the
    # W = T softmax codes, 4-bit GELU, pruned frozen-LayerNorm x~
    assert seen["quant8"] > 0 and seen["packed4"] == L and seen["pruned"] > 0
    assert seen["softmax"] in (0, L)      # 0 when the fused attention kernel writes the probability codes
