"""Fused bias / layout kernels of the encoder step vs plain PyTorch fp32.

* split / merge heads (+ bias, + codes): bit-exact against permute + add and
  against sf_quantize of the same values;
* GELU with the projection bias fused: y, the packed4 cache and the prescale
  exponent bit-exact against the unfused kernels run on x + b;
* residual LayerNorm LN(res + (x + b)): bit-exact against the plain LN kernel
  on the same sum (the sum rounds identically), float32-close to torch;
* the autograd ops' gradients against torch autograd of the unfused graph.
"""

import numpy as np
import pytest
import torch

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def sf():
    import paper_2305_18513_b200 as sf
    return sf


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("B,T,h,dh", [(2, 5, 3, 8), (4, 128, 12, 64), (1, 197, 16, 64)])
def test_split_merge_heads(sf, B, T, h, dh):
    N = sf._native
    g = torch.Generator(device="cuda").manual_seed(B * T)
    y = torch.randn(B, T, h * dh, generator=g, device="cuda") * 3
    bias = torch.randn(h * dh, generator=g, device="cuda")
    out = torch.empty(B, h, T, dh, device="cuda")
    codes = torch.empty(B, h, T, dh, dtype=torch.int8, device="cuda")
    N.call("sf_split_heads", y.data_ptr(), bias.data_ptr(), out.data_ptr(), codes.data_ptr(), B, T, h, dh,
           4, 1, _stream())
    ref = (y + bias).view(B, T, h, dh).permute(0, 2, 1, 3).contiguous()
    assert torch.equal(out, ref)
    assert torch.equal(codes, sf.compression.quantize(ref, sf.Q4_4))
    back = torch.empty(B, T, h * dh, device="cuda")
    N.call("sf_merge_heads", out.data_ptr(), back.data_ptr(), B, T, h, dh, _stream())
    assert torch.equal(back, y + bias)


def test_split_heads_autograd(sf):
    from paper_2305_18513_b200 import tensor as T
    B, Tn, h, dh = 3, 7, 4, 8
    g = torch.Generator(device="cuda").manual_seed(1)
    y = torch.randn(B, Tn, h * dh, generator=g, device="cuda", requires_grad=True)
    b = torch.randn(h * dh, generator=g, device="cuda", requires_grad=True)
    w = torch.randn(B, h, Tn, dh, generator=g, device="cuda")
    with T.record(sf.CompressionConfig()):
        out = T.split_heads(y, b, h)
        z = T.merge_heads(out * w)
        z.square().sum().backward()
    gy, gb = y.grad.clone(), b.grad.clone()
    y.grad = b.grad = None
    ref = ((y + b).view(B, Tn, h, dh).permute(0, 2, 1, 3) * w).permute(0, 2, 1, 3).reshape(B, Tn, h * dh)
    ref.square().sum().backward()
    assert torch.allclose(gy, y.grad, rtol=1e-6, atol=1e-6)
    assert torch.allclose(gb, b.grad, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("rows,H", [(16384, 768), (37, 128), (5, 1024)])
def test_layernorm_residual(sf, rows, H):
    N = sf._native
    g = torch.Generator(device="cuda").manual_seed(rows)
    r = torch.randn(rows, H, generator=g, device="cuda")
    x = torch.randn(rows, H, generator=g, device="cuda") * 2
    b = torch.randn(H, generator=g, device="cuda")
    gam = torch.randn(H, generator=g, device="cuda")
    bet = torch.randn(H, generator=g, device="cuda")
    y1, xt1, s1 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    rs1 = torch.empty(rows, device="cuda")
    N.call("sf_layernorm_fwd_residual", r.data_ptr(), x.data_ptr(), b.data_ptr(), gam.data_ptr(),
           bet.data_ptr(), y1.data_ptr(), s1.data_ptr(), xt1.data_ptr(), rs1.data_ptr(), rows, H, 1e-5,
           _stream())
    t = r + (x + b)
    assert torch.equal(s1, t)
    y2, xt2 = torch.empty_like(x), torch.empty_like(x)
    rs2 = torch.empty(rows, device="cuda")
    N.call("sf_layernorm_fwd", t.data_ptr(), gam.data_ptr(), bet.data_ptr(), y2.data_ptr(), xt2.data_ptr(),
           rs2.data_ptr(), rows, H, 1e-5, _stream())
    assert torch.equal(y1, y2) and torch.equal(xt1, xt2) and torch.equal(rs1, rs2)
    ref = torch.nn.functional.layer_norm(t, (H,), gam, bet, 1e-5)
    assert torch.allclose(y1, ref, rtol=1e-4, atol=1e-4)


def test_layernorm_residual_autograd(sf):
    from paper_2305_18513_b200 import tensor as T
    rows, H = 64, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    r = torch.randn(2, rows // 2, H, generator=g, device="cuda", requires_grad=True)
    x = torch.randn(2, rows // 2, H, generator=g, device="cuda", requires_grad=True)
    b = torch.randn(H, generator=g, device="cuda", requires_grad=True)
    gam = torch.randn(H, generator=g, device="cuda", requires_grad=True)
    bet = torch.randn(H, generator=g, device="cuda", requires_grad=True)
    w = torch.randn(2, rows // 2, H, generator=g, device="cuda")
    with T.record(sf.CompressionConfig()):
        (T.layernorm_residual(r, x, b, gam, bet) * w).sum().backward()
    got = [t.grad.clone() for t in (r, x, b, gam, bet)]
    for t in (r, x, b, gam, bet):
        t.grad = None
    (torch.nn.functional.layer_norm(r + (x + b), (H,), gam, bet, 1e-5) * w).sum().backward()
    for a, t in zip(got, (r, x, b, gam, bet)):
        assert torch.allclose(a, t.grad, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("rows,N_", [(16384, 3072), (197 * 4, 3072), (33, 512)])
def test_gelu_bias_fused(sf, rows, N_):
    N = sf._native
    Cz = sf.compression
    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(rows, N_, generator=g, device="cuda") * 2
    b = torch.randn(N_, generator=g, device="cuda")
    xb = x + b
    n = x.numel()
    lib = N.load()
    ws = torch.empty(lib.sf_prescale_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    q = Cz._quantile(99.9)
    s1 = torch.zeros(1, dtype=torch.int32, device="cuda")
    y1 = torch.empty_like(x)
    x1 = x.clone()
    N.call("sf_gelu_fwd_prescale_bias", x1.data_ptr(), b.data_ptr(), N_, y1.data_ptr(), n, q, 1.75,
           s1.data_ptr(), ws.data_ptr(), _stream())
    s2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    y2 = torch.empty_like(x)
    N.call("sf_gelu_fwd_prescale", xb.data_ptr(), y2.data_ptr(), n, q, 1.75, s2.data_ptr(), ws.data_ptr(),
           _stream())
    assert torch.equal(x1, xb)
    assert torch.equal(y1, y2)
    assert int(s1) == int(s2)


def test_gelu_bias_autograd(sf):
    from paper_2305_18513_b200 import tensor as T
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(6, 40, 256, generator=g, device="cuda", requires_grad=True)
    b = torch.randn(256, generator=g, device="cuda", requires_grad=True)
    w = torch.randn(6, 40, 256, generator=g, device="cuda")
    with T.record(sf.CompressionConfig()):          # codecs off: exact cached input
        (T.gelu(x * 1.0, bias=b) * w).sum().backward()
    gx, gb = x.grad.clone(), b.grad.clone()
    x.grad = b.grad = None
    (torch.nn.functional.gelu(x + b, approximate="tanh") * w).sum().backward()
    assert torch.allclose(gx, x.grad, rtol=1e-4, atol=1e-5)
    assert torch.allclose(gb, b.grad, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("frozen", [(), ("q",), ("k", "v"), ("q", "k", "v")])
@pytest.mark.parametrize("stacked", [True, False])
def test_qkv_heads_matches_separate_projections(sf, frozen, stacked):
    """qkv_heads (one batched GEMM forward, one K=3H GEMM for dx) against
    three linear + split_heads ops: outputs, the per-projection ledger
    entries and all gradients (float32 tolerance: GEMM order differs)."""
    from paper_2305_18513_b200 import tensor as T
    g = torch.Generator(device="cuda").manual_seed(11)
    B, Tn, H, h = 4, 16, 64, 4
    x0 = torch.randn(B, Tn, H, generator=g, device="cuda")
    if stacked:
        buf = torch.randn(3, H, H, generator=g, device="cuda") * 0.05
        W = [torch.nn.Parameter(buf[i]) for i in range(3)]
    else:
        W = [torch.nn.Parameter(torch.randn(H, H, generator=g, device="cuda") * 0.05) for _ in range(3)]
    bias = [torch.nn.Parameter(torch.randn(H, generator=g, device="cuda")) for _ in range(3)]
    assert (T._stacked(W) is not None) == stacked
    for name, w, b in zip("qkv", W, bias):
        w.requires_grad_(name not in frozen)
        b.requires_grad_(name not in frozen)
    gout = [torch.randn(B, h, Tn, H // h, generator=g, device="cuda") for _ in range(3)]

    def run(fused):
        x = x0.clone().requires_grad_(True)
        for p in W + bias:
            p.grad = None
        with T.record(sf.CompressionConfig()) as tape:
            if fused:
                outs = T.qkv_heads(x, W, bias, h, save_names=["q", "k", "v"])
            else:
                outs = [T.split_heads(T.linear(x, w, None, save_name=n), b, h) for w, b, n in zip(W, bias, "qkv")]
            sum((o * go).sum() for o, go in zip(outs, gout)).backward()
        grads = [x.grad] + [p.grad for p in W + bias]
        return [o.detach() for o in outs], grads, tape.cached_bytes()

    o1, g1, c1 = run(True)
    o0, g0, c0 = run(False)
    assert c1 == c0
    for a, b in zip(o1, o0):
        torch.testing.assert_close(a, b, rtol=1e-5, atol=1e-5)
    for a, b in zip(g1, g0):
        assert (a is None) == (b is None)
        if a is not None:
            torch.testing.assert_close(a, b, rtol=1e-4, atol=1e-4)


def test_merge_heads_ld_writes_column_slices(sf):
    N = sf._native
    B, T, h, dh = 2, 5, 3, 8
    x = torch.randn(B, h, T, dh, device="cuda")
    out = torch.full((B * T, 3 * h * dh), -1.0, device="cuda")
    N.call("sf_merge_heads_ld", x.data_ptr(), out[:, h * dh:].data_ptr(), B, T, h, dh, 3 * h * dh, _stream())
    want = x.permute(0, 2, 1, 3).reshape(B * T, h * dh)
    assert torch.equal(out[:, h * dh:2 * h * dh], want)
    assert bool((out[:, :h * dh] == -1).all()) and bool((out[:, 2 * h * dh:] == -1).all())


@pytest.mark.parametrize("B,T", [(2, 16), (3, 100), (4, 128), (2, 197), (1, 384), (2, 130)])
@pytest.mark.parametrize("frozen", [(), ("q", "v")])
def test_fused_self_attention_matches_unfused_ops(sf, B, T, frozen):
    """csrc/attention.cu against the unfused qkv_heads / matmul / softmax /
    matmul / merge_heads ops: context and gradients within float32
    tolerance (summation order differs), q/k/v codes bit-exact, probability
    codes equal up to round-off ties, ledger byte-identical."""
    from paper_2305_18513_b200 import tensor as T_
    g = torch.Generator(device="cuda").manual_seed(B * T)
    h, H = 12, 768
    x0 = torch.randn(B, T, H, generator=g, device="cuda")
    buf = torch.randn(3, H, H, generator=g, device="cuda") * 0.05
    W = [torch.nn.Parameter(buf[i]) for i in range(3)]
    bias = [torch.nn.Parameter(torch.randn(H, generator=g, device="cuda") * 0.1) for _ in range(3)]
    for name, w, b in zip("qkv", W, bias):
        w.requires_grad_(name not in frozen)
        b.requires_grad_(name not in frozen)
    gout = torch.randn(B, T, H, generator=g, device="cuda")
    scale = 0.125
    names = (["q", "k", "v"], "s", "sm", "c")

    def run(fused):
        x = x0.clone().requires_grad_(True)
        for p in W + bias:
            p.grad = None
        with T_.record(sf.CompressionConfig.all_on()) as tape:
            if fused:
                assert T_.fused_attention_ok(x, h, H)
                out = T_.self_attention(x, W, bias, h, scale, names)
            else:
                q, k, v = T_.qkv_heads(x, W, bias, h, save_names=["q", "k", "v"])
                raw = T_.matmul(q, k.transpose(-1, -2), compress="matsoft8", save_name="s")
                probs = T_.softmax(raw, compress="matsoft8", save_name="sm", scale=scale)
                out = T_.merge_heads(T_.matmul(probs, v, compress="matsoft8", save_name="c"))
            (out * gout).sum().backward()
        recs = {n: b for n, _, b in tape.saved_records()}
        return out.detach(), [x.grad] + [p.grad for p in W + bias], tape, recs

    o1, g1, t1, r1 = run(True)
    o0, g0, t0, r0 = run(False)
    assert t1.cached_bytes() == t0.cached_bytes() and r1 == r0
    sc = o0.abs().max().item()
    assert (o1 - o0).abs().max().item() <= 2e-5 * sc
    for a, b in zip(g1, g0):
        assert (a is None) == (b is None)
        if a is not None:
            assert (a - b).abs().max().item() <= 1e-4 * max(b.abs().max().item(), 1e-20)


@pytest.mark.parametrize("T", [128, 130, 197, 256, 384])
def test_fused_attention_codes_vs_quantize(sf, T):
    """The forward kernels' q/k/v codes are sf_quantize of (y + b), and the
    probability codes match quantize(softmax(q k^T * scale)) computed from
    the same q/k up to rare rounding-boundary flips (|diff| <= 1); the
    context within fp32 tolerance of an fp64 evaluation.  T = 128: one CTA
    per head; the other T: the query-tiled kernels (ViT T = 197, BERT-large
    T = 384, ragged T)."""
    N = sf._native
    g = torch.Generator(device="cuda").manual_seed(3 + T)
    B, h, dh = 2, 12, 64
    H = h * dh
    y3 = torch.randn(3, B * T, H, generator=g, device="cuda") * 0.7
    bs = [torch.randn(H, generator=g, device="cuda") * 0.1 for _ in range(3)]
    ctx = torch.empty(B * T, H, device="cuda")
    qc = torch.empty(B, h, T, dh, dtype=torch.int8, device="cuda")
    kc, vc = torch.empty_like(qc), torch.empty_like(qc)
    pc = torch.empty(B, h, T, T, dtype=torch.int8, device="cuda")
    N.call("sf_attention_fwd", y3.data_ptr(), bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr(), B, T, h,
           dh, 0.125, 4, ctx.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(), _stream())
    heads = [(y3[i] + bs[i]).reshape(B, T, h, dh).permute(0, 2, 1, 3).contiguous() for i in range(3)]
    for want, got in zip(heads, (qc, kc, vc)):
        assert torch.equal(sf.quantize(want, sf.Q4_4), got)
    q, k, v = [t.double() for t in heads]
    p = torch.softmax((q @ k.transpose(-1, -2)).float().double() * 0.125, dim=-1)
    ref = sf.quantize(p.float(), sf.Q4_4)
    diff = (ref.int() - pc.int()).abs()
    assert diff.max().item() <= 1 and diff.float().mean().item() < 1e-3
    c_ref = (p @ v).permute(0, 2, 1, 3).reshape(B * T, H)
    assert (ctx.double() - c_ref).abs().max().item() <= 1e-5 * c_ref.abs().max().item()
    # argument validation: unsupported shapes are refused, not mis-computed
    with pytest.raises(Exception):
        N.call("sf_attention_fwd", y3.data_ptr(), bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr(), B, 400,
               h, dh, 0.125, 4, ctx.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
               _stream())


@pytest.mark.parametrize("T", [8, 16, 100, 124, 128])
def test_attention_backward_tensor_cores_vs_fma(sf, T):
    """The tensor-core backward (bf16 MMAs, exact 3-term splits of the fp32
    operand, exact code operands) against the FP32-FMA kernel and against an
    fp64 evaluation of the same decoded operands."""
    N = sf._native
    lib = N.load()
    g = torch.Generator(device="cuda").manual_seed(T)
    B, h, dh = 3, 12, 64
    H = h * dh
    qc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    kc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    vc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    logits = torch.randn(B, h, T, T, generator=g, device="cuda") * 2
    pc = sf.quantize(torch.softmax(logits, -1), sf.Q4_4)
    gr = torch.randn(B * T, H, generator=g, device="cuda")
    outs = []
    for impl in (0, 1, 2, 3):                      # FMA, tcgen05 fp16 planes (default), mma.sync, tcgen05 bf16
        assert lib.sf_attention_set_impl(impl) == 0
        gcat = torch.full((B * T, 3 * H), float("nan"), device="cuda")
        N.call("sf_attention_bwd", gr.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
               B, T, h, dh, 0.125, 4, gcat.data_ptr(), None, _stream())
        outs.append(gcat)
    lib.sf_attention_set_impl(1)
    q, k, v, p = [c.double() / 16 for c in (qc, kc, vc, pc)]
    G = gr.double().reshape(B, T, h, dh).permute(0, 2, 1, 3)
    dP = G @ v.transpose(-1, -2)
    dS = p * (dP - (dP * p).sum(-1, keepdim=True)) * 0.125
    ref = [dS @ k, dS.transpose(-1, -2) @ q, p.transpose(-1, -2) @ G]
    ref = torch.cat([r.permute(0, 2, 1, 3).reshape(B * T, H) for r in ref], dim=1)
    sc = ref.abs().max().item()
    for o in outs:
        assert torch.isfinite(o).all()
        assert (o.double() - ref).abs().max().item() <= 2e-6 * sc


@pytest.mark.parametrize("T", [8, 16, 99, 100, 124, 128, 130, 144, 197, 256, 300, 384])
def test_attention_forward_tcgen05_vs_mma_sync(sf, T):
    """The tcgen05 forwards (TMEM accumulators, shared-memory descriptors;
    one CTA per head for T <= 128 with T % 4 == 0 -- impl 1 on two fp16
    planes per operand, two CTAs per SM; impl 3 on three bf16 planes --
    query tiles of 128 rows
    with the score tile combined in TMEM otherwise -- ViT T = 197, BERT-large
    T = 384, ragged T) against the mma.sync forwards on the same inputs:
    q/k/v codes identical, probability codes identical up to rare
    rounding-boundary flips, context within fp32 tolerance; and both against
    fp64."""
    N = sf._native
    lib = N.load()
    g = torch.Generator(device="cuda").manual_seed(77 + T)
    B, h, dh = 3, 12, 64
    H = h * dh
    y3 = torch.randn(3, B * T, H, generator=g, device="cuda") * 0.7
    bs = [torch.randn(H, generator=g, device="cuda") * 0.1 for _ in range(3)]
    outs = []
    for impl in (1, 2, 3):
        assert lib.sf_attention_set_impl(impl) == 0
        ctx = torch.full((B * T, H), float("nan"), device="cuda")
        qc = torch.empty(B, h, T, dh, dtype=torch.int8, device="cuda")
        kc, vc = torch.empty_like(qc), torch.empty_like(qc)
        pc = torch.empty(B, h, T, T, dtype=torch.int8, device="cuda")
        N.call("sf_attention_fwd", y3.data_ptr(), bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr(), B, T, h,
               dh, 0.125, 4, ctx.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(), _stream())
        outs.append((ctx, qc, kc, vc, pc))
    lib.sf_attention_set_impl(1)
    (c5, q5, k5, v5, p5), (c2, q2, k2, v2, p2), (c3, q3, k3, v3, p3) = outs
    assert torch.equal(q5, q2) and torch.equal(k5, k2) and torch.equal(v5, v2)
    assert torch.equal(q3, q2) and torch.equal(k3, k2) and torch.equal(v3, v2)
    for pa in (p5, p3):
        d = (pa.int() - p2.int()).abs()
        assert d.max().item() <= 1 and d.float().mean().item() < 1e-3
    heads = [(y3[i] + bs[i]).double().reshape(B, T, h, dh).permute(0, 2, 1, 3) for i in range(3)]
    p = torch.softmax(heads[0] @ heads[1].transpose(-1, -2) * 0.125, dim=-1)
    ref = (p @ heads[2]).permute(0, 2, 1, 3).reshape(B * T, H)
    sc = ref.abs().max().item()
    for c in (c5, c2, c3):
        assert torch.isfinite(c).all()
        assert (c.double() - ref).abs().max().item() <= 1e-5 * sc


@pytest.mark.parametrize("T", [99, 130, 144, 197, 256, 300, 384])
@pytest.mark.parametrize("impl", [1, 2])
def test_attention_backward_wide_vs_fp64(sf, T, impl):
    """The query-tiled backward (dq per query tile; dk | dv per key tile with
    dP recomputed per block) against an fp64 evaluation of the same decoded
    operands, for T past the one-head kernels' limit: impl 1 the tcgen05
    kernels (128-row tiles, TMEM accumulators), impl 2 the mma.sync ones."""
    N = sf._native
    lib = N.load()
    assert lib.sf_attention_set_impl(impl) == 0
    g = torch.Generator(device="cuda").manual_seed(T)
    B, h, dh = 2, 12, 64
    H = h * dh
    qc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    kc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    vc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
    logits = torch.randn(B, h, T, T, generator=g, device="cuda") * 2
    pc = sf.quantize(torch.softmax(logits, -1), sf.Q4_4)
    gr = torch.randn(B * T, H, generator=g, device="cuda")
    nws = lib.sf_attention_bwd_workspace_bytes(B, T, h)
    assert nws == B * h * T * 4
    ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
    gcat = torch.full((B * T, 3 * H), float("nan"), device="cuda")
    N.call("sf_attention_bwd", gr.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
           B, T, h, dh, 0.125, 4, gcat.data_ptr(), ws.data_ptr(), _stream())
    q, k, v, p = [c.double() / 16 for c in (qc, kc, vc, pc)]
    G = gr.double().reshape(B, T, h, dh).permute(0, 2, 1, 3)
    dP = G @ v.transpose(-1, -2)
    dS = p * (dP - (dP * p).sum(-1, keepdim=True)) * 0.125
    ref = [dS @ k, dS.transpose(-1, -2) @ q, p.transpose(-1, -2) @ G]
    ref = torch.cat([r.permute(0, 2, 1, 3).reshape(B * T, H) for r in ref], dim=1)
    assert torch.isfinite(gcat).all()
    for i in range(3):
        o, r = gcat[:, i * H:(i + 1) * H].double(), ref[:, i * H:(i + 1) * H]
        assert (o - r).abs().max().item() <= 2e-6 * r.abs().max().item(), i
    with pytest.raises(Exception):                 # the wide path needs its workspace
        N.call("sf_attention_bwd", gr.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
               B, T, h, dh, 0.125, 4, gcat.data_ptr(), None, _stream())
    lib.sf_attention_set_impl(1)


@pytest.mark.parametrize("V,H,N_", [(64, 32, 200), (30522, 768, 16384), (5, 128, 1)])
def test_embedding_backward_matches_add_at(sf, V, H, N_):
    """sf_embedding_bwd (sync-free, position-ordered) equals np.add.at on
    the same float32 rows bit for bit (tensor.py:497-520)."""
    from paper_2305_18513_b200 import tensor as T_
    rng = np.random.default_rng(V + N_)
    ids = rng.integers(0, min(V, 40), size=N_)            # heavy repeats
    g = rng.standard_normal((N_, H)).astype(np.float32)
    table = torch.nn.Parameter(torch.zeros(V, H, device="cuda"))
    with T_.record(sf.CompressionConfig()):
        out = T_.embedding(table, torch.as_tensor(ids, device="cuda"))
        out.backward(torch.as_tensor(g, device="cuda"))
    want = np.zeros((V, H), np.float32)
    np.add.at(want, ids, g)
    assert np.array_equal(table.grad.cpu().numpy(), want)


def test_gelu_planes_only_into_frozen_projection(sf):
    """FFN with a frozen output projection: the GELU writes only the
    projection's operand planes (no fp32 result) -- the projection output,
    the gradients of x and the GELU bias, and the ledger are bit-identical to
    the path that writes the fp32 result; a product that would read a
    planes-only tensor without its planes is refused, not computed."""
    from paper_2305_18513_b200 import tensor as T
    g = torch.Generator(device="cuda").manual_seed(21)
    rows, H, F = 512, 256, 1024
    x0 = torch.randn(rows, H, generator=g, device="cuda")
    w1 = torch.randn(H, F, generator=g, device="cuda") * 0.05
    b1 = torch.randn(F, generator=g, device="cuda") * 0.1
    w2 = torch.randn(F, H, generator=g, device="cuda") * 0.05      # frozen (no grad)
    gout = torch.randn(rows, H, generator=g, device="cuda")
    res = []
    for po in (False, True):
        x = x0.clone().requires_grad_(True)
        bb = b1.clone().requires_grad_(True)
        with T.record(sf.CompressionConfig.all_on()) as tape:
            h = T.gelu(T.linear(x, w1, None, save_name="up"), bias=bb, save_name="gelu", planes_only=po)
            o = T.linear(h, w2, None, compress="dense8", save_name="down")
            del h
            (o * gout).sum().backward()
            led = tape.cached_bytes()
        res.append((o.detach().clone(), x.grad.clone(), bb.grad.clone(), led))
    (o1, gx1, gb1, l1), (o2, gx2, gb2, l2) = res
    assert torch.equal(o1, o2) and torch.equal(gx1, gx2) and torch.equal(gb1, gb2)
    assert l1 == l2
    # the guard: another product between the GELU and its projection takes the planes
    with T.record(sf.CompressionConfig.all_on()):
        x = x0.clone().requires_grad_(True)
        h = T.gelu(T.linear(x, w1, None, save_name="up"), bias=b1, save_name="gelu", planes_only=True)
        T.linear(x0, w1, None, save_name="other")
        with pytest.raises(sf._native.KernelError):
            T.linear(h, w2, None, compress="dense8", save_name="down")


def test_gelu_backward_planes_only_into_frozen_projection(sf):
    """FFN with a frozen input projection: the GELU backward writes only the
    row-scaled planes of dx for that projection's input-gradient product --
    x's gradient bit-identical to the path that writes dx in fp32."""
    from paper_2305_18513_b200 import tensor as T
    g = torch.Generator(device="cuda").manual_seed(22)
    rows, H, F = 512, 256, 1024
    x0 = torch.randn(rows, H, generator=g, device="cuda")
    w1 = torch.randn(H, F, generator=g, device="cuda") * 0.05          # frozen
    b1 = torch.randn(F, generator=g, device="cuda") * 0.1              # frozen
    w2 = torch.randn(F, H, generator=g, device="cuda", requires_grad=True)
    gout = torch.randn(rows, H, generator=g, device="cuda")
    res = []
    for bpo in (False, True):
        x = x0.clone().requires_grad_(True)
        w2.grad = None
        with T.record(sf.CompressionConfig.all_on()):
            h = T.gelu(T.linear(x, w1, None, save_name="up"), bias=b1, save_name="gelu", bwd_planes_only=bpo)
            o = T.linear(h, w2, None, compress="dense8", save_name="down")
            (o * gout).sum().backward()
        res.append((x.grad.clone(), w2.grad.clone()))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])


@pytest.mark.parametrize("T_", [128, 197])
def test_attention_planes_only_into_frozen_projection(sf, T_):
    """The attention core feeding a frozen output projection writes only the
    context's operand planes (fp16-plane tcgen05 forwards): projection output
    and every gradient bit-identical to the fp32-context path."""
    from paper_2305_18513_b200 import tensor as T
    g = torch.Generator(device="cuda").manual_seed(T_)
    B, H, h = 4, 768, 12
    x0 = torch.randn(B, T_, H, generator=g, device="cuda")
    ws = [torch.randn(H, H, generator=g, device="cuda", requires_grad=True) * 0.03 for _ in range(3)]
    ws = [w.detach().requires_grad_(True) for w in ws]
    bs = [torch.randn(H, generator=g, device="cuda") * 0.1 for _ in range(3)]
    bs = [b.requires_grad_(True) for b in bs]
    wo = torch.randn(H, H, generator=g, device="cuda") * 0.03          # frozen
    gout = torch.randn(B, T_, H, generator=g, device="cuda")
    res = []
    for po in (False, True):
        x = x0.clone().requires_grad_(True)
        for t in ws + bs:
            t.grad = None
        with T.record(sf.CompressionConfig.all_on()):
            c = T.self_attention(x, ws, bs, h, 0.125, (["q", "k", "v"], "s", "p", "c"), planes_only=po)
            o = T.linear(c, wo, None, save_name="out")
            del c
            (o * gout).sum().backward()
        res.append([o.detach().clone(), x.grad.clone()] + [t.grad.clone() for t in ws + bs])
    for a, b in zip(*res):
        assert torch.equal(a, b)
