"""Host-side logic that needs no GPU: the distance plan (chunking of numpy's
pairwise tree), the ILS decisions, the AdamW constants and the registry."""

import numpy as np
import pytest

from oracle import ils

from paper_2305_18513_b200 import scheduler as S


def simulate_plan(e: np.ndarray) -> float:
    """Evaluate np.sum(e) the way the device does: each chunk with numpy's
    pairwise order, then the level-ordered tree above the chunks."""
    chunks, tree, levels = S.pairwise_plan(e.size)
    partial = [ils.pairwise_sum(e[o:o + n]) for o, n in chunks]
    nc = len(partial)
    node = [0.0] * tree.shape[0]

    def val(i):
        return partial[i] if i < nc else node[i - nc]

    for lv in range(len(levels) - 1):
        for k in range(levels[lv], levels[lv + 1]):
            node[k] = val(int(tree[k, 0])) + val(int(tree[k, 1]))
    return node[-1] if tree.shape[0] else partial[0]


@pytest.mark.parametrize("n", [1, 7, 128, 129, 4096, 4097, 8192, 8193, 100_003, 768 * 3072 + 5])
def test_pairwise_plan_reproduces_numpy_sum(n):
    rng = np.random.default_rng(n)
    e = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
    assert simulate_plan(e) == float(np.sum(e))


def eval_program(e: np.ndarray) -> float:
    """Evaluate one chunk through its device program (leaves then levels)."""
    prog = S.chunk_program(e.size)
    nl, nn, nlev = int(prog[0]), int(prog[1]), int(prog[2])
    leaves = prog[4:4 + 2 * nl].reshape(-1, 2)
    nodes = prog[4 + 2 * nl:4 + 2 * nl + 2 * nn].reshape(-1, 2)
    levels = prog[4 + 2 * nl + 2 * nn:]
    assert len(levels) == (nlev + 1 if nn else 1)
    val = [ils.pairwise_sum(e[o:o + m]) for o, m in leaves] + [0.0] * nn
    for lv in range(nlev):
        for i in range(levels[lv], levels[lv + 1]):
            val[nl + i] = val[int(nodes[i, 0])] + val[int(nodes[i, 1])]
    assert nl <= 64 and leaves[:, 1].max() <= 128
    return val[nl + nn - 1] if nn else val[0]


@pytest.mark.parametrize("n", [1, 5, 8, 100, 128, 129, 300, 1000, 2049, 4095, 4096])
def test_chunk_program_reproduces_pairwise(n):
    rng = np.random.default_rng(n + 7)
    e = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
    assert eval_program(e) == float(np.sum(e))


def test_plan_levels_are_topological():
    chunks, tree, levels = S.pairwise_plan(23_440_896)
    nc = chunks.shape[0]
    done = set(range(nc))
    for lv in range(len(levels) - 1):
        new = []
        for k in range(levels[lv], levels[lv + 1]):
            assert int(tree[k, 0]) in done and int(tree[k, 1]) in done
            new.append(nc + k)
        done.update(new)
    assert chunks[:, 1].max() <= 4096 and chunks[:, 1].sum() == 23_440_896


def test_decisions_match_oracle():
    rng = np.random.default_rng(0)
    for t in range(50):
        n = int(rng.integers(1, 200))
        d = rng.choice([0.5, 1.0, 2.0], size=n) if t % 2 else rng.random(n)
        f = float(rng.choice([0.0, 0.5, 0.75, 0.95]))
        dv = S.DistanceVector(d.copy(), np.ones(n, bool))
        assert sorted(S.select_frozen(dv, f).frozen_ids) == ils.frozen_ids(d, f)
    assert np.array_equal(S.init_distances(102, 7).d, ils.warm_distances(102, 7))


def test_scheduler_errors():
    from paper_2305_18513_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        S.init_distances(0, 0)
    with pytest.raises(ConfigError):
        S.select_frozen(S.init_distances(4, 0), 1.0)
    with pytest.raises(ConfigError):
        S.Scheduler("bogus", 4, 0.5, 0)


def test_adamw_constants_match_numpy_promotion():
    from paper_2305_18513_b200.trainer import OptimizerState
    opt = OptimizerState()
    for t in (1, 2, 10, 1000):
        a = opt._consts(t, 5e-5)
        b = ils.adamw_constants(t, 5e-5)
        for k in ("bc1", "bc2", "ob1", "ob2", "lr", "eps", "wd"):
            assert a[k] == b[k] and a[k].dtype == np.float32


def test_slot_packing_roundtrip():
    v = S._pack(np.float32(0.9), np.float32(-0.1))
    u = np.int64(v).view(np.uint64)
    assert np.uint32(u & 0xFFFFFFFF).view(np.float32) == np.float32(0.9)
    assert np.uint32(u >> 32).view(np.float32) == np.float32(-0.1)


def test_qkv_weights_are_stacked_views_with_reference_init():
    """Model.build keeps the reference's init draws but places each block's
    q/k/v weights back to back (one batched GEMM over them)."""
    import numpy as np
    import paper_2305_18513_b200 as sf
    from oracle import encoder as E
    from paper_2305_18513_b200 import tensor as T
    cfg = sf.ModelConfig(blocks=2, hidden=32, heads=4, max_seq=16, vocab=64, num_classes=4)
    m = sf.build_model(cfg, 3, device="cpu")
    ref = E.init_params(E.EncoderConfig(blocks=2, hidden=32, heads=4, max_seq=16, vocab=64, num_classes=4), seed=3)
    assert all(np.array_equal(a, b) for la, lb in zip(m.to_numpy(), ref) for a, b in zip(la, lb))
    for i in range(2):
        ws = [m.registry.by_name(f"encoder.layer.{i}.attention.self.{n}").params[0] for n in ("query", "key", "value")]
        assert all(w.is_contiguous() for w in ws)
        assert T._stacked(ws) is not None
