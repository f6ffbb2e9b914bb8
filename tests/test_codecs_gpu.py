"""Device codecs vs the oracle and the reference's golden vectors.

Bar: bit-exact codes / packed bytes / prescale exponents / pruned indices and
values (reference tests/test_compression.py pins ported as device tests,
plus seeded fuzzing at BERT-base sizes and the adversarial sets).
"""

import math

import numpy as np
import pytest
import torch

from oracle import codecs as C
from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def sf():
    import paper_2305_18513_b200 as sf
    return sf


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


# ----------------------------------------------------------------- quant8

def test_quantize_golden(golden, sf):
    g = golden("codecs.npz")
    x = g["q_x"]
    assert np.array_equal(host(sf.quantize(dev(x), sf.Q4_4)), g["q44"])
    assert np.array_equal(host(sf.quantize(dev(x), sf.Q0_8_UNSIGNED)), g["q08u"])
    assert np.array_equal(host(sf.quantize(dev(np.nan_to_num(x, nan=0.0) / 4.0), sf.Q2_2)),
                          g["q22_direct"])
    assert np.array_equal(host(sf.dequantize(dev(g["dq_codes"]), sf.Q4_4)), g["dq44"])
    assert np.array_equal(host(sf.dequantize(dev(np.arange(256, dtype=np.uint8)),
                                             sf.Q0_8_UNSIGNED)), g["dq08u"])


@pytest.mark.parametrize("n", [1, 15, 16, 17, 1000, 4099, 1 << 20, 50_331_648])
def test_quantize_fuzz_sizes(sf, n):
    rng = np.random.default_rng(n)
    x = (rng.standard_normal(n) * 4).astype(np.float32)
    x[:: max(1, n // 97)] = (rng.integers(-300, 300, size=x[:: max(1, n // 97)].size) / 32.0)
    t = dev(x)
    for spec, fmt in [(sf.Q4_4, C.Q44), (sf.Q0_8_UNSIGNED, C.Q08U)]:
        codes = sf.quantize(t, spec)
        assert np.array_equal(host(codes), C.quantize(x, fmt))
        assert np.array_equal(host(sf.dequantize(codes, spec)), C.dequantize(C.quantize(x, fmt), fmt))


def test_quantize_misaligned_view(sf):
    x = (np.random.default_rng(0).standard_normal(10_003) * 3).astype(np.float32)
    t = dev(x)[3:]                          # not 16-byte aligned, tail path
    assert np.array_equal(host(sf.quantize(t, sf.Q4_4)), C.quantize(x[3:], C.Q44))


def test_round_half_away_near_ties(sf):
    # values one ulp either side of k + 0.5 after scaling (the fp32 floor(|v|+0.5) trap)
    base = (np.arange(-40, 40) + 0.5) / 16.0
    x = np.concatenate([base, np.nextafter(base.astype(np.float32), np.float32(np.inf)),
                        np.nextafter(base.astype(np.float32), np.float32(-np.inf)),
                        np.float32([0.49999997 / 16, -0.49999997 / 16])]).astype(np.float32)
    assert np.array_equal(host(sf.quantize(dev(x), sf.Q4_4)), C.quantize(x, C.Q44))


def test_reference_known_answers(sf):
    # tests/test_compression.py:31-48
    assert host(sf.quantize(dev(np.float32([0.5, 10.0, 0.0, 0.03125, -0.03125])), sf.Q4_4)).tolist() == \
        [8, 127, 0, 1, -1]
    ca = sf.CompressedActivation.quantized(dev(np.float32([[0.5, -1.25], [7.9375, 100.0]])), sf.Q4_4)
    assert ca.nbytes == 4
    out = host(ca.decompress())
    assert out[0, 0] == 0.5 and out[1, 1] == 7.9375
    blob = sf.CompressedActivation.quantized(dev(np.float32([0.5, -0.5])), sf.Q4_4).dump()
    head, _, body = blob.partition(b"\n")
    assert b'"tag": "quant8"' in head and body == np.array([8, -8], np.int8).tobytes()


# ----------------------------------------------------------------- pack4 / prescale

def test_pack4_golden_and_bijection(golden, sf):
    g = golden("codecs.npz")
    assert np.array_equal(host(sf.pack4(dev(g["p4_codes"]))), g["p4_packed"])
    assert np.array_equal(host(sf.unpack4(dev(g["p4_packed"]), g["p4_codes"].size)), g["p4_codes"])
    assert host(sf.pack4(dev(np.int8([3, -2])))).tolist() == [0xE3]
    assert host(sf.pack4(dev(np.int8([7])))).tolist() == [0x07]
    with pytest.raises(sf.CodecError):
        sf.pack4(dev(np.int8([8])))
    with pytest.raises(sf.CodecError):
        sf.unpack4(dev(np.uint8([1])), 3)


PK_CASES = ["n01", "n03", "big", "small", "const14", "zeros", "with_nan", "with_inf", "one", "odd9",
            "edge175", "edge35", "adv"]


@pytest.mark.parametrize("name", PK_CASES)
def test_packed4_golden(golden, sf, name):
    g = golden("codecs.npz")
    x = g[f"pk_{name}_x"]
    ca = sf.CompressedActivation.packed(dev(x), sf.Q2_2)
    assert ca.prescale_exp == int(g[f"pk_{name}_s"])
    assert np.array_equal(host(ca.packed_codes), g[f"pk_{name}_packed"])
    assert np.array_equal(host(ca.decompress()), g[f"pk_{name}_dec"])
    assert ca.nbytes == (x.size + 1) // 2


def _straddle(lo_val, hi_val, n, n_hi):
    x = np.full(n, lo_val, np.float32)
    x[-n_hi:] = hi_val
    return np.random.default_rng(n).permutation(x)


@pytest.mark.parametrize("x", [
    _straddle(3.5, 3.6, 2000, 2),            # a = 3.5 (edge), b = 3.6 -> refine pass
    _straddle(1.75, 1.7500001, 5000, 5),
    _straddle(0.2, 7.0, 1001, 1),
    _straddle(6.9999995, 7.0, 100_000, 100),
    _straddle(224.0, 300.0, 10_000, 10),
], ids=["3.5|3.6", "1.75|up", "0.2|7", "7-|7", "224|300"])
def test_prescale_straddle_refine(sf, x):
    s = sf.choose_prescale_exp(dev(x), sf.Q2_2)
    assert s == C.prescale_exp(x, C.Q22)


@pytest.mark.parametrize("sigma,n", [(1.0, 50_331_648), (3.0, 9_682_944), (0.05, 1_000_003),
                                     (40.0, 777_777), (1e4, 100_000)])
def test_packed4_fuzz(sf, sigma, n):
    rng = np.random.default_rng(int(sigma * 100) + n)
    x = (rng.standard_normal(n) * sigma).astype(np.float32)
    ca = sf.CompressedActivation.packed(dev(x), sf.Q2_2)
    s = C.prescale_exp(x, C.Q22)
    assert ca.prescale_exp == s
    codes = C.quantize(x / np.float32(1 << s), C.Q22)
    assert np.array_equal(host(ca.packed_codes), C.pack4(codes))
    assert np.array_equal(host(ca.decompress()), C.unpack_gelu(C.pack4(codes), s, n))


# ----------------------------------------------------------------- prune / restore

PR_CASES = ["spec", "ties", "signed", "rand", "rand_signed", "quantized_ties", "zeros_pm", "nan_inf",
            "nan_signed", "keep_all", "one", "ln_rows"]


@pytest.mark.parametrize("name", PR_CASES)
def test_prune_golden(golden, sf, name):
    g = golden("codecs.npz")
    x = g[f"pr_{name}_x"]
    sp = sf.prune_topk(dev(x), float(g[f"pr_{name}_keep"]), bool(g[f"pr_{name}_mag"]))
    assert np.array_equal(host(sp.indices), g[f"pr_{name}_idx"])
    assert np.array_equal(host(sp.values), g[f"pr_{name}_vals"], equal_nan=True)
    assert np.array_equal(host(sf.restore(sp)), g[f"pr_{name}_dense"], equal_nan=True)


@pytest.mark.parametrize("n,layout", [
    (5_000_000, "head"), (5_000_000, "tail"), (5_000_000, "two_ends"), (5_000_000, "uniform"),
    (8192 * 300, "every_other_tile"), (8192 * 7 + 3, "all"), (100_003, "single"), (64, "none"),
])
def test_restore_layouts(sf, n, layout):
    """restore assembles each output tile in shared memory from the tile's
    slice of the index list: skewed, empty, full and ragged index sets must
    scatter exactly (compression.py:165-169)."""
    rng = np.random.default_rng(n)
    pos = np.arange(n, dtype=np.int64)
    if layout == "head":
        idx = pos[: n // 10]
    elif layout == "tail":
        idx = pos[-(n // 10):]
    elif layout == "two_ends":
        idx = np.concatenate([pos[:100_000], pos[-100_000:]])
    elif layout == "uniform":
        idx = np.sort(rng.choice(n, n // 10, replace=False))
    elif layout == "every_other_tile":
        idx = pos[(pos // 8192) % 2 == 0][::3]
    elif layout == "all":
        idx = pos
    elif layout == "single":
        idx = np.array([n - 1])
    else:
        idx = pos[:0]
    idx = idx.astype(np.int32)
    vals = rng.standard_normal(idx.size).astype(np.float32)
    sp = sf.PrunedSparse(dev(vals), dev(idx), n, (n,))
    want = np.zeros(n, np.float32)
    want[idx] = vals
    assert np.array_equal(host(sf.restore(sp)), want)


@pytest.mark.parametrize("n,keep,mag,kind", [
    (12_582_912, 0.1, True, "ln"), (2_420_736, 0.1, True, "ln"), (1_000_001, 0.1, False, "normal"),
    (300_000, 0.37, True, "quantized"), (65_536, 0.1, True, "constant"), (4096 * 3 + 5, 0.5, True, "normal"),
    # tie-heavy inputs force the exact single-CTA slow path (candidates > buffer)
    (200_000, 0.1, True, "constant"), (500_000, 0.25, False, "quantized"),
    # a sorted ramp: the sampled bracket sits in a smooth, dense region
    (1_048_576, 0.1, True, "ramp"),
    # ~4000 copies per level: the threshold bin holds more candidates than the
    # finish kernel ranks in shared memory -> its radix-select path
    (2_000_000, 0.1, True, "levels500"), (2_000_000, 0.3, False, "levels500"),
    # ~100K copies per level: more candidates than the buffer -> slow path
    (2_000_000, 0.1, True, "levels20"),
])
def test_prune_fuzz(sf, n, keep, mag, kind):
    rng = np.random.default_rng(n)
    if kind == "ln":
        x = rng.standard_normal((n // 768, 768)).astype(np.float32)
        x = ((x - x.mean(-1, keepdims=True)) / x.std(-1, keepdims=True)).astype(np.float32)
    elif kind == "quantized":
        x = (np.round(rng.standard_normal(n) * 8) / 8).astype(np.float32)
    elif kind == "constant":
        x = np.full(n, -1.5, np.float32)
    elif kind == "ramp":
        x = np.linspace(-3, 3, n, dtype=np.float32)
    elif kind.startswith("levels"):
        lv = int(kind[6:])
        x = (rng.integers(-lv // 2, lv // 2, n) / 16).astype(np.float32)
    else:
        x = rng.standard_normal(n).astype(np.float32)
    vals, idx = C.prune_topk(x, keep, mag)
    sp = sf.prune_topk(dev(x), keep, mag)
    assert np.array_equal(host(sp.indices), idx)
    assert np.array_equal(host(sp.values), vals)
    dense = host(sf.restore(sp))
    assert np.array_equal(dense, C.restore(vals, idx, x.size, x.shape))


@pytest.mark.parametrize("n,row_len,keep,kind", [
    # staged path (keep <= ~0.13): row starts before the first / after the last
    # staged key of a tile, rows spanning tiles, ragged last tile
    (768 * 853, 768, 0.1, "normal"), (768 * 69, 768, 0.05, "normal"),
    (1024 * 4000, 1024, 0.12, "sparse_rows"), (768 * 37, 768, 0.1, "normal"), (300 * 7, 7, 0.1, "normal"),
    # x path (the staging list overflows) and the slow path (heavy ties)
    (768 * 2000, 768, 0.4, "normal"), (768 * 3000, 768, 0.1, "levels4"),
])
def test_prune_row_pointers(sf, n, row_len, keep, kind):
    """CSR row pointers of the kept set, written by the emit pass from the
    staged lists (or from x): row_ptr[r] = #kept with index < r * row_len,
    row_ptr[rows] = k -- equal to a searchsorted over the oracle's indices."""
    rng = np.random.default_rng(n + row_len)
    if kind == "levels4":
        x = (rng.integers(-2, 2, n) / 4).astype(np.float32)
    else:
        x = rng.standard_normal(n).astype(np.float32)
    if kind == "sparse_rows":               # most rows hold no survivor at all
        x[(np.arange(n) // row_len) % 5 != 0] *= np.float32(1e-3)
    vals, idx = C.prune_topk(x, keep, True)
    sp = sf.prune_topk(dev(x.reshape(-1, row_len)), keep, True, row_pointers=True)
    assert np.array_equal(host(sp.indices), idx)
    assert np.array_equal(host(sp.values), vals)
    want = np.searchsorted(idx, np.arange(n // row_len + 1, dtype=np.int64) * row_len).astype(np.int32)
    assert np.array_equal(host(sp.row_ptr), want)
    # K7 through the row pointers (sf_restore_rows) equals the oracle's restore
    if row_len % 4 == 0:
        dense = sf.restore(sp)
        assert np.array_equal(host(dense).reshape(-1), C.restore(vals, idx, n))


@pytest.mark.parametrize("keep", [0.01, 0.05, 0.1, 0.125, 0.13, 0.2, 0.5, 0.9, 1.0])
def test_prune_keep_fractions(sf, keep):
    """Every keep fraction is exact whichever path it takes (staged lists up
    to ~0.13, x re-read above)."""
    n = 16384 * 50 + 123
    rng = np.random.default_rng(int(keep * 1000))
    x = rng.standard_normal(n).astype(np.float32)
    for mag in (True, False):
        vals, idx = C.prune_topk(x, keep, mag)
        sp = sf.prune_topk(dev(x), keep, mag)
        assert np.array_equal(host(sp.indices), idx)
        assert np.array_equal(host(sp.values), vals)


def test_prune_many_tiles_properties(sf):
    """> 4096 tiles of 16384 (the finish kernel's general scan path) at a size
    the oracle's full argsort would take long on: checked by the defining
    properties -- k kept, ascending unique indices, every kept |x| >= every
    dropped |x|, and ties at the threshold kept in index order."""
    n = 70_000_000
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.randint(-2000, 2000, (n,), generator=g, device="cuda").float() / 64)
    sp = sf.prune_topk(x, 0.1)
    k = sf.compression.keep_count(n, 0.1)
    idx = sp.indices.long()
    assert idx.numel() == k
    assert bool((idx[1:] > idx[:-1]).all())
    assert torch.equal(sp.values, x[idx])
    kept = torch.zeros(n, dtype=torch.bool, device="cuda")
    kept[idx] = True
    a = x.abs()
    t = a[idx].min()
    assert float(a[~kept].max()) <= float(t)
    tie_kept = torch.nonzero(kept & (a == t)).flatten()
    tie_drop = torch.nonzero(~kept & (a == t)).flatten()
    assert tie_kept.numel() > 0
    if tie_drop.numel():
        assert int(tie_kept.max()) < int(tie_drop.min())
    assert int((a > t).sum()) + tie_kept.numel() == k


def test_prune_errors(sf):
    with pytest.raises(sf.CodecError):
        sf.prune_topk(dev(np.zeros(0, np.float32)), 0.1)
    with pytest.raises(sf.CodecError):
        sf.prune_topk(dev(np.ones(4, np.float32)), 1.5)
    assert sf.compression.keep_count(12_582_912, 0.1) == 1_258_292
    ca = sf.CompressedActivation.pruned(dev(np.arange(20, dtype=np.float32)), keep_frac=0.1)
    assert ca.nbytes == 16


def test_determinism(sf):
    x = dev(np.random.default_rng(3).standard_normal(3_000_000).astype(np.float32))
    a = sf.prune_topk(x, 0.1)
    b = sf.prune_topk(x, 0.1)
    assert torch.equal(a.indices, b.indices) and torch.equal(a.values, b.values)
    p = sf.CompressedActivation.packed(x, sf.Q2_2)
    q = sf.CompressedActivation.packed(x, sf.Q2_2)
    assert torch.equal(p.packed_codes, q.packed_codes)


def _hint_case(kind, n, rng):
    if kind == "ln":
        x = rng.standard_normal((n // 768, 768)).astype(np.float32)
        return ((x - x.mean(-1, keepdims=True)) / x.std(-1, keepdims=True)).astype(np.float32)
    if kind == "levels4":
        return (rng.integers(-2, 2, n) / 4).astype(np.float32)
    if kind == "constant":
        return np.full(n, 0.75, np.float32)
    if kind == "nan_inf":
        x = rng.standard_normal(n).astype(np.float32)
        x[rng.integers(0, n, n // 50)] = np.nan
        x[rng.integers(0, n, 7)] = np.inf
        return x
    return rng.standard_normal(n).astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("seq", [
    ("ln", "ln", "ln", "ln"),                        # same site, fresh batches: the hinted path
    ("ln", "scaled", "ln", "scaled"),                 # the threshold moves 3x: a miss, then re-hinted
    ("normal", "levels4", "constant", "normal"),     # ties and a bracket full of equal keys
    ("nan_inf", "nan_inf", "normal", "nan_inf"),
])
def test_prune_hint_sequences(sf, seq):
    """A per-site hint changes nothing but the path: every call of a sequence
    at one site (hint rewritten each time) equals the oracle bit for bit,
    values, indices and CSR row pointers alike -- hits, misses (threshold
    moved, ties filling the bracket) and the first call without a hint."""
    rng = np.random.default_rng(len("".join(seq)))
    hint = sf.compression.new_prune_hint()
    row_len = 768
    for i, kind in enumerate(seq):
        n = row_len * (700 + 37 * i)
        x = _hint_case("normal" if kind == "scaled" else kind, n, rng)
        if kind == "scaled":
            x = (x * 3).astype(np.float32)
        for keep in (0.1, 0.03):
            vals, idx = C.prune_topk(x, keep, True)
            sp = sf.prune_topk(dev(x.reshape(-1, row_len)), keep, True, row_pointers=True, hint=hint)
            assert np.array_equal(host(sp.indices), idx), (i, kind, keep)
            assert np.array_equal(host(sp.values), vals, equal_nan=True), (i, kind, keep)
            want_rp = np.searchsorted(idx, np.arange(0, n + 1, row_len), side="left")
            want_rp[-1] = idx.size
            assert np.array_equal(host(sp.row_ptr), want_rp.astype(np.int32)), (i, kind, keep)
            h = host(hint).view(np.uint32)
            assert h[0] == 1 and h[2] >= (1 << 14)
            assert not h[4:(h.size * 4 - 80) // 4].any()    # the grid state left zeroed (t[10] excepted)


@pytest.mark.gpu
def test_prune_hint_large_and_unhinted_equal(sf):
    """At the BERT-base size: the hinted call (second call at the site) is
    identical to the unhinted one; a signed-key call ignores the hint."""
    n = 128 * 128 * 768
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n // 768, 768, generator=g, device="cuda")
    x = (x - x.mean(-1, keepdim=True)) / x.std(-1, keepdim=True, unbiased=False)
    hint = sf.compression.new_prune_hint()
    ref = sf.prune_topk(x, 0.1, True, row_pointers=True)
    for _ in range(3):
        sp = sf.prune_topk(x, 0.1, True, row_pointers=True, hint=hint)
        assert torch.equal(sp.indices, ref.indices) and torch.equal(sp.values, ref.values)
        assert torch.equal(sp.row_ptr, ref.row_ptr)
    x2 = x + 0.01 * torch.randn(x.shape, generator=g, device="cuda")
    ref2 = sf.prune_topk(x2, 0.1, True)
    sp2 = sf.prune_topk(x2, 0.1, True, hint=hint)
    assert torch.equal(sp2.indices, ref2.indices) and torch.equal(sp2.values, ref2.values)
    refs = sf.prune_topk(x2, 0.1, False)
    sps = sf.prune_topk(x2, 0.1, False, hint=hint)
    assert torch.equal(sps.indices, refs.indices) and torch.equal(sps.values, refs.values)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 100, 4097, 148 * 32 * 16 + 5])
def test_prune_hint_small_and_ragged(sf, n):
    """Tiny and ragged sizes (most warps own no elements) at one hinted site,
    keep fractions up to 1.0, all-zero and all-NaN tensors (whose thresholds
    give no usable hint) -- every call equal to the oracle."""
    rng = np.random.default_rng(n)
    hint = sf.compression.new_prune_hint()
    cases = [rng.standard_normal(n).astype(np.float32) for _ in range(3)]
    cases += [np.zeros(n, np.float32), np.full(n, np.nan, np.float32), rng.standard_normal(n).astype(np.float32)]
    for x in cases:
        for keep in (0.1, 0.5, 1.0):
            vals, idx = C.prune_topk(x, keep, True)
            sp = sf.prune_topk(dev(x), keep, True, hint=hint)
            assert np.array_equal(host(sp.indices), idx)
            assert np.array_equal(host(sp.values), vals, equal_nan=True)
