"""Dense fp32 GEMMs through sf_gemm_f32 (cuBLASLt) against an fp64 product.

The reference computes `x @ W + b`, `g @ W.T`, `x.T @ g` and the batched
attention products in float32 (numpy/OpenBLAS, tensor.py:290-379).  The
bound used here: each mode's max error relative to max|C64| must stay within
a stated multiple of what strict SGEMM (CUBLAS_COMPUTE_32F) achieves on the
same inputs; for bf16x9 that multiple is 1 (emulation must be at least as
accurate as fp32 SIMT), plus an absolute 2^-22 floor.
"""

import pytest
import torch

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def G():
    from paper_2305_18513_b200 import gemm
    old = gemm.get_mode()
    yield gemm
    gemm.set_mode(old)


def _err(c, ref):
    return (c.double() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)


SHAPES = [(1, 1, 1), (3, 5, 7), (64, 96, 33), (1000, 768, 130), (2048, 768, 3072), (16384, 768, 768)]


@pytest.mark.parametrize("m,k,n", SHAPES)
@pytest.mark.parametrize("layout", ["nn", "nt", "tn", "bias"])
def test_gemm_modes_vs_fp64(G, m, k, n, layout):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(k, n, device="cuda", generator=g) * 0.02
    bias = torch.randn(n, device="cuda", generator=g) if layout == "bias" else None
    if layout == "nt":
        b = b.t().contiguous().t()          # transposed view: folded into the op
    if layout == "tn":
        a = a.t().contiguous().t()
    ref = a.double() @ b.double()
    if bias is not None:
        ref = ref + bias.double()
    G.set_mode("fp32")
    c32 = G.mm(a, b, bias)
    e32 = _err(c32, ref)
    assert e32 < 1e-5
    if G.available("bf16x9"):
        G.set_mode("bf16x9")
        c9 = G.mm(a, b, bias)
        assert c9.shape == (m, n) and c9.is_contiguous()
        assert _err(c9, ref) <= max(e32, 2.0 ** -22), (_err(c9, ref), e32)
    G.set_mode("bf16x6")
    c6 = G.mm(a, b, bias)
    assert c6.shape == (m, n) and c6.is_contiguous()
    assert _err(c6, ref) <= max(2 * e32, 2.0 ** -22), (_err(c6, ref), e32)


def _split_ref(x):
    h = x.bfloat16()
    r = x - h.float()
    mid = r.bfloat16()
    return torch.stack([h, mid, (r - mid.float()).bfloat16()])


@pytest.mark.parametrize("rows,cols,transpose", [(1000, 776, False), (333, 777, True), (4096, 768, True),
                                                 (64, 8, False), (7, 5, True)])
def test_split3_is_exact(G, rows, cols, transpose):
    """x = hi + mid + lo, each the round-to-nearest bf16 of what is left."""
    from paper_2305_18513_b200 import _native as N
    x = torch.randn(rows, cols, device="cuda") * 10
    out = torch.empty((3, cols, rows) if transpose else (3, rows, cols), dtype=torch.bfloat16, device="cuda")
    N.call("sf_split3_bf16", x.data_ptr(), rows, cols, cols, int(transpose), out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    ref = _split_ref(x.t().contiguous() if transpose else x)
    assert torch.equal(out, ref)
    # the three terms represent x exactly
    assert torch.equal(out[0].double() + out[1].double() + out[2].double(),
                       (x.t() if transpose else x).double())


@pytest.mark.parametrize("m,k,n", [(768, 16384, 768), (3072, 16384, 768), (128, 8192, 256), (16384, 3072, 768)])
def test_bf16x6_long_reductions_split_k(G, m, k, n):
    """Weight-gradient shapes (reduction over B*T tokens): split-K partials
    keep the error at strict SGEMM's level; a^T views (x^T @ g) exercise the
    transposing split."""
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    x = torch.randn(k, m, device="cuda", generator=g)
    gr = torch.randn(k, n, device="cuda", generator=g)
    ref = x.double().t() @ gr.double()
    G.set_mode("fp32")
    e32 = _err(G.mm(x.t(), gr), ref)
    G.set_mode("bf16x6")
    acc = torch.randn(m, n, device="cuda", generator=g)
    c6 = G.mm(x.t(), gr, out=acc.clone(), beta=1.0)
    assert _err(c6, ref + acc.double()) <= max(2 * e32, 2.0 ** -22), (_err(c6, ref + acc.double()), e32)


def test_gemm_bf16x9_available_on_b200(G):
    """The toolkit cuBLASLt (12.9) must load and provide emulation: the
    step's default mode depends on it."""
    assert G.N.load().sf_gemm_lt_version() >= 120900, G.N.load().sf_gemm_lt_error()
    assert G.available("bf16x9")


@pytest.mark.parametrize("mode", ["fp32", "bf16x9", "tf32"])
def test_gemm_batched_attention_shapes(G, mode):
    """(B, h, T, dh) x k^T view, probs x v, and the transposed-view gradients."""
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(4, 12, 128, 64, device="cuda", generator=g)
    k = torch.randn(4, 12, 128, 64, device="cuda", generator=g)
    G.set_mode(mode)
    for a, b in [(q, k.transpose(-1, -2)), (torch.softmax(q @ k.transpose(-1, -2), -1), k),
                 (q.transpose(-1, -2), k)]:
        ref = a.double() @ b.double()
        c = G.mm(a, b)
        tol = 1e-3 if mode == "tf32" else 1e-5
        assert _err(c, ref) < tol


def test_gemm_broadcast_and_errors(G):
    from paper_2305_18513_b200.errors import ShapeError
    G.set_mode("fp32")
    a = torch.randn(3, 4, 5, device="cuda")
    b = torch.randn(5, 6, device="cuda")
    torch.testing.assert_close(G.mm(a, b.expand(3, 5, 6)), a @ b, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(G.mm(a, b.unsqueeze(0)), a @ b, rtol=1e-5, atol=1e-5)
    with pytest.raises(ShapeError):
        G.mm(a, torch.randn(4, 6, device="cuda"))
    with pytest.raises(ShapeError):
        G.mm(a.double(), b.double())
    out = G.mm(torch.randn(3, 0, device="cuda"), torch.randn(0, 2, device="cuda"))
    assert out.shape == (3, 2) and bool((out == 0).all())


def test_gemm_strict_fp32_matches_torch_sgemm_closely(G):
    """Strict mode is plain SGEMM: it differs from torch's (cuBLAS 12.8)
    only in summation order (~1e-6 of the output scale at k=768)."""
    G.set_mode("fp32")
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.randn(512, 768, device="cuda", generator=g)
    b = torch.randn(768, 256, device="cuda", generator=g)
    c, ref = G.mm(a, b), a @ b
    assert (c - ref).abs().max().item() <= 1e-5 * ref.abs().max().item()


@pytest.mark.parametrize("m,k,n,beta", [(16384, 3072, 768, 0.0), (1000, 2048, 200, 1.0), (300, 4096, 768, 0.0),
                                        (129, 2056, 512, 0.0)])
def test_bf16x6_in_kernel_a_split(G, m, k, n, beta):
    """The A-as-fp32 variant (in-kernel split of A, taken for n <= 768 and
    k >= 2048) against fp64, with bias and accumulation, ragged m and k."""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn(m, k, device="cuda", generator=g)
    w = torch.randn(n, k, device="cuda", generator=g) * 0.02
    bias = torch.randn(n, device="cuda", generator=g)
    c0 = torch.randn(m, n, device="cuda", generator=g)
    ref = a.double() @ w.double().t() + bias.double() + beta * c0.double()
    G.set_mode("fp32")
    e32 = _err(G.mm(a, w.t(), bias, out=c0.clone(), beta=beta), ref)
    G.set_mode("bf16x6")
    old = G.in_kernel_a_split
    G.in_kernel_a_split = True
    try:
        c6 = G.mm(a, w.t(), bias, out=c0.clone(), beta=beta)
    finally:
        G.in_kernel_a_split = old
    # floor 2^-22 * k / 512: the tensor core's truncating accumulation grows
    # with the K run (strict SGEMM is sometimes luckier on small outputs)
    assert _err(c6, ref) <= max(2 * e32, 2.0 ** -22 * k / 512), (_err(c6, ref), e32)


@pytest.mark.parametrize("k,m,n", [(16384, 768, 3072), (16384, 3072, 768), (520, 40, 12), (1024, 96, 64)])
def test_wgrad_with_bias_row(G, k, m, n):
    """[x^T; 1] g in one product: dW = x^T g and db = g.sum(0) (the ones
    row of the A planes) against fp64."""
    g = torch.Generator(device="cuda").manual_seed(k + m)
    x = torch.randn(k, m, device="cuda", generator=g)
    gr = torch.randn(k, n, device="cuda", generator=g) * 0.1
    G.set_mode("bf16x6")
    dW, db = G.mm_wgrad_bias(x, gr)
    assert dW.shape == (m, n) and db.shape == (n,) and dW.is_contiguous()
    rW = x.double().t() @ gr.double()
    rb = gr.double().sum(0)
    assert (dW.double() - rW).abs().max().item() <= 2e-6 * rW.abs().max().item()
    assert (db.double() - rb).abs().max().item() <= 2e-6 * max(rb.abs().max().item(), gr.abs().sum(0).max().item())


@pytest.mark.parametrize("T,dh", [(197, 64), (384, 64), (40, 16)])
def test_bf16x6_batched_attention_products(G, T, dh):
    """The attention's batched products at T > 128 (q k^T, p v, g v^T, p^T g)
    on the batched tcgen05 path (contiguous entries, K % 8 == 0) or the
    cuBLASLt fallback, against fp64 at SGEMM-level error."""
    g = torch.Generator(device="cuda").manual_seed(T)
    q = torch.randn(2, 3, T, dh, device="cuda", generator=g)
    kk = torch.randn(2, 3, T, dh, device="cuda", generator=g)
    p = torch.rand(2, 3, T, T, device="cuda", generator=g)
    G.set_mode("bf16x6")
    old = G.batched_tc
    G.batched_tc = True
    for a, b in [(q, kk.transpose(-1, -2)), (p, kk), (p.transpose(-1, -2), q), (q, q.transpose(-1, -2))]:
        ref = a.double() @ b.double()
        c = G.mm(a, b)
        G.set_mode("fp32")
        e32 = _err(G.mm(a, b), ref)
        G.set_mode("bf16x6")
        assert _err(c, ref) <= max(2 * e32, 2.0 ** -22 * max(1, a.shape[-1] / 512)), (_err(c, ref), e32)
    G.batched_tc = old


def test_kept_weight_planes_follow_updates(G):
    """Planes of kept parameters are reused across products and re-split
    after the parameter changes: torch in-place ops (version counter) or an
    explicit weight_planes_changed (the optimizer's raw-pointer writes)."""
    g = torch.Generator(device="cuda").manual_seed(7)
    w = torch.nn.Parameter(torch.randn(256, 384, device="cuda", generator=g))
    x = torch.randn(512, 256, device="cuda", generator=g)
    G.set_mode("bf16x6")
    G.keep_weight_planes([w])
    try:
        y = torch.randn(512, 384, device="cuda", generator=g)

        def check():
            wd = w.detach()
            assert _err(G.mm(x, wd), x.double() @ wd.double()) < 1e-5            # forward: W
            assert _err(G.mm(y, wd.t()), y.double() @ wd.double().t()) < 1e-5    # input gradient: W^T
        check()
        with torch.no_grad():
            w.mul_(-2.0)                      # version bump
        check()
        w.data.copy_(torch.randn(256, 384, device="cuda", generator=g))   # no version bump
        G.weight_planes_changed([w])
        check()
    finally:
        G._wparams.clear()
        G._wplanes.clear()


def _native_split(x):
    """Planes [3][rows][cols] of x from sf_split3_bf16 (the GEMM's own split)."""
    from paper_2305_18513_b200 import _native as N
    rows, cols = x.numel() // x.shape[-1], x.shape[-1]
    out = torch.empty(3 * rows * cols, dtype=torch.bfloat16, device="cuda")
    N.call("sf_split3_bf16", x.data_ptr(), rows, cols, cols, 0, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out


@pytest.mark.parametrize("which", ["ln", "ln_res", "ln_bwd_dense", "ln_bwd_cols", "gelu_fwd", "gelu_bwd", "attn_fwd",
                                   "attn_bwd", "attn_fwd_wide", "attn_bwd_wide"])
@pytest.mark.parametrize("pf", [0, 1])
def test_producer_planes_equal_split(which, pf):
    """The `_p` producers' operand planes are bit-identical to sf_split3_bf16
    of the fp32 output they write (the split the next product would run);
    the forward producers' `_pf` form 1 to sf_split2_f16 (the f16x3 planes)."""
    from paper_2305_18513_b200 import _native as N
    from paper_2305_18513_b200 import compression as Cz
    if pf and which not in ("ln", "ln_res", "gelu_fwd", "attn_fwd", "attn_fwd_wide"):
        pytest.skip("backward producers write the bf16 planes only")
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(hash(which) % 1000)
    rows, H = 300, 768
    def planes_for(t):
        if pf:
            return torch.full((2 * t.numel(),), float("nan"), dtype=torch.float16, device="cuda")
        return torch.full((3 * t.numel(),), float("nan"), dtype=torch.bfloat16, device="cuda")
    if which in ("ln", "ln_res"):
        x = torch.randn(rows, H, generator=g, device="cuda") * 3
        gam, bet = torch.rand(H, generator=g, device="cuda") + 0.5, torch.randn(H, generator=g, device="cuda")
        y, xt, rs = torch.empty_like(x), torch.empty_like(x), torch.empty(rows, device="cuda")
        pl = planes_for(y)
        if which == "ln":
            N.call("sf_layernorm_fwd_pf", x.data_ptr(), gam.data_ptr(), bet.data_ptr(), y.data_ptr(),
                   xt.data_ptr(), rs.data_ptr(), rows, H, 1e-5, pl.data_ptr(), pf, st)
        else:
            res, b = torch.randn_like(x), torch.randn(H, generator=g, device="cuda")
            N.call("sf_layernorm_fwd_residual_pf", res.data_ptr(), x.data_ptr(), b.data_ptr(), gam.data_ptr(),
                   bet.data_ptr(), y.data_ptr(), None, xt.data_ptr(), rs.data_ptr(), rows, H, 1e-5, pl.data_ptr(),
                   pf, st)
        out = y
    elif which in ("ln_bwd_dense", "ln_bwd_cols"):
        gr = torch.randn(rows, H, generator=g, device="cuda")
        xt = torch.randn(rows, H, generator=g, device="cuda")
        gam, rs = torch.rand(H, generator=g, device="cuda") + 0.5, torch.rand(rows, generator=g, device="cuda") + 0.5
        dx = torch.empty_like(gr)
        ws = torch.empty(N.load().sf_layernorm_bwd_workspace_bytes(rows, H), dtype=torch.uint8, device="cuda")
        dg, db = (torch.empty(H, device="cuda"), torch.empty(H, device="cuda")) if which == "ln_bwd_cols" else (None, None)
        pl = planes_for(dx)
        N.call("sf_layernorm_bwd_p", gr.data_ptr(), gam.data_ptr(), xt.data_ptr(), None, None, 0, None, rs.data_ptr(),
               dx.data_ptr(), dg.data_ptr() if dg is not None else None, db.data_ptr() if db is not None else None,
               rows, H, ws.data_ptr(), pl.data_ptr(), st)
        out = dx
    elif which == "gelu_fwd":
        x = torch.randn(rows, 4 * H, generator=g, device="cuda")
        b = torch.randn(4 * H, generator=g, device="cuda")
        y = torch.empty_like(x)
        s = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = torch.empty(N.load().sf_prescale_workspace_bytes(x.numel()), dtype=torch.uint8, device="cuda")
        pl = planes_for(y)
        N.call("sf_gelu_fwd_prescale_bias_pf", x.data_ptr(), b.data_ptr(), 4 * H, y.data_ptr(), x.numel(),
               Cz._quantile(99.9), 1.75, s.data_ptr(), ws.data_ptr(), pl.data_ptr(), pf, st)
        out = y
    elif which == "gelu_bwd":
        n = rows * 4 * H
        gr = torch.randn(n, generator=g, device="cuda")
        packed = torch.randint(0, 256, ((n + 1) // 2,), generator=g, device="cuda", dtype=torch.uint8)
        s = torch.tensor([1], dtype=torch.int32, device="cuda")
        dx = torch.empty_like(gr)
        pl = planes_for(dx)
        N.call("sf_gelu_bwd_packed4_p", gr.data_ptr(), packed.data_ptr(), s.data_ptr(), 2, dx.data_ptr(), n,
               pl.data_ptr(), st)
        out = dx.reshape(rows, 4 * H)
    else:
        B, T, h, dh = 2, (128 if not which.endswith("wide") else 197), 12, 64
        Hh = h * dh
        if which.startswith("attn_fwd"):
            y3 = torch.randn(3, B * T, Hh, generator=g, device="cuda") * 0.5
            bs = [torch.randn(Hh, generator=g, device="cuda") * 0.1 for _ in range(3)]
            ctx = torch.empty(B * T, Hh, device="cuda")
            qc = torch.empty(B, h, T, dh, dtype=torch.int8, device="cuda")
            kc, vc = torch.empty_like(qc), torch.empty_like(qc)
            pc = torch.empty(B, h, T, T, dtype=torch.int8, device="cuda")
            pl = planes_for(ctx)
            N.call("sf_attention_fwd_pf", y3.data_ptr(), bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr(), B,
                   T, h, dh, 0.125, 4, ctx.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
                   pl.data_ptr(), pf, st)
            out = ctx
        else:
            qc = torch.randint(-128, 128, (B, h, T, dh), generator=g, device="cuda", dtype=torch.int8)
            kc, vc = torch.randint_like(qc, -128, 128), torch.randint_like(qc, -128, 128)
            pc = torch.randint(0, 17, (B, h, T, T), generator=g, device="cuda", dtype=torch.int8)
            gr = torch.randn(B * T, Hh, generator=g, device="cuda")
            gcat = torch.empty(B * T, 3 * Hh, device="cuda")
            nws = N.load().sf_attention_bwd_workspace_bytes(B, T, h)
            ws = torch.empty(max(nws, 1), dtype=torch.uint8, device="cuda")
            pl = planes_for(gcat)
            N.call("sf_attention_bwd_p", gr.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(), pc.data_ptr(),
                   B, T, h, dh, 0.125, 4, gcat.data_ptr(), ws.data_ptr() if nws else None, pl.data_ptr(), st)
            out = gcat
    torch.cuda.synchronize()
    if pf:
        ref = torch.empty(2 * out.numel(), dtype=torch.float16, device="cuda")
        N.call("sf_split2_f16", out.data_ptr(), out.numel() // out.shape[-1], out.shape[-1], out.shape[-1], 0,
               ref.data_ptr(), st)
        torch.cuda.synchronize()
        assert torch.equal(ref.view(2, *out.shape), _split2_ref(out))
    else:
        ref = _native_split(out)
    assert torch.equal(pl.view(torch.int16), ref.view(torch.int16))


def test_producer_planes_step_bitwise():
    """A training step with the producers writing the operand planes (and the
    products skipping their split) is bit-identical to the step with every
    split run by the GEMM path, and the planes are actually consumed."""
    import numpy as np
    import paper_2305_18513_b200 as sf
    from paper_2305_18513_b200 import gemm as G
    old_mode = G.get_mode()
    G.set_mode("bf16x6")
    cfg = sf.ModelConfig(blocks=2, hidden=256, heads=4, max_seq=64, vocab=500, num_classes=3)
    out = []
    for on in (False, True):
        G.producer_planes = on
        G.plane_hits = 0
        m = sf.build_model(cfg, seed=3)
        rc = sf.RunConfig(scheduler="ils", freeze_rate=0.5, epochs=1, batch_size=8, seed=1, lr=1e-3,
                          warmup_frac=0.0, compression=sf.CompressionConfig.all_on())
        rng = np.random.default_rng(0)
        toks, labs = rng.integers(0, 500, (24, 64)), rng.integers(0, 3, 24)
        log = sf.fine_tune(m, (toks, labs), rc)
        out.append(([p.detach().cpu().numpy() for p in m.parameters()], [mm[1] for mm in log.metrics], G.plane_hits))
    G.producer_planes = True
    G.set_mode(old_mode)
    for a, b in zip(out[0][0], out[1][0]):
        assert np.array_equal(a, b)
    assert out[0][1] == out[1][1]
    assert out[0][2] == 0 and out[1][2] > 0


def _split2_ref(x):
    h = x.half()
    return torch.stack([h, ((x - h.float()) * 2048.0).half()])


@pytest.mark.parametrize("rows,cols,transpose", [(1000, 776, False), (333, 777, True), (4096, 768, True),
                                                 (64, 8, False), (7, 5, True)])
def test_split2_f16(G, rows, cols, transpose):
    """The f16x3 operand split: hi = RN_f16(x), lo = RN_f16((x - hi) 2^11),
    bit for bit; x = hi + 2^-11 lo to 22 bits in fp16's normal range."""
    from paper_2305_18513_b200 import _native as N
    g = torch.Generator(device="cuda").manual_seed(rows + cols)
    x = torch.randn(rows, cols, device="cuda", generator=g) * torch.exp2(
        torch.randint(-12, 12, (rows, cols), device="cuda", generator=g).float())
    out = torch.empty((2, cols, rows) if transpose else (2, rows, cols), dtype=torch.float16, device="cuda")
    N.call("sf_split2_f16", x.data_ptr(), rows, cols, cols, int(transpose), out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    xs = x.t().contiguous() if transpose else x
    assert torch.equal(out, _split2_ref(xs))
    rec = out[0].double() + out[1].double() / 2048.0
    normal = xs.abs() >= 2.0 ** -14
    rel = ((rec - xs.double()).abs() / xs.double().abs().clamp_min(1e-300))[normal]
    assert rel.max().item() <= 2.0 ** -22


@pytest.mark.parametrize("m,k,n", [(1000, 768, 136), (2048, 768, 3072), (16384, 768, 768), (16384, 3072, 768),
                                   (4096, 768, 2304), (333, 520, 264)])
def test_f16x3_vs_fp64(G, m, k, n):
    """sf_gemm_f16x3 (hh + 2^-11 (hl + lh) on two fp16 planes per operand)
    against an fp64 product of the same fp32 operands: within twice strict
    SGEMM's error on activation-like A (mixed magnitudes) and weight-like B."""
    from paper_2305_18513_b200 import _native as N
    lib = N.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + k)
    a = torch.randn(m, k, device="cuda", generator=g) * torch.exp2(
        torch.randint(-6, 5, (m, 1), device="cuda", generator=g).float())
    b = torch.randn(k, n, device="cuda", generator=g) * 0.02
    bias = torch.randn(n, device="cuda", generator=g)
    ref = a.double() @ b.double() + bias.double()
    G.set_mode("fp32")
    e32 = _err(G.mm(a, b, bias), ref)
    pa = torch.empty(2, m, k, dtype=torch.float16, device="cuda")
    pb = torch.empty(2, n, k, dtype=torch.float16, device="cuda")
    N.call("sf_split2_f16", a.data_ptr(), m, k, k, 0, pa.data_ptr(), st)
    N.call("sf_split2_f16", b.data_ptr(), k, n, n, 1, pb.data_ptr(), st)
    nb = lib.sf_gemm_split6_ws_bytes(m, n, k)
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    outs = []
    # N = 256 (auto) / 128 tiles; TMA-store / direct epilogue; CTA pairs (cta_group::2) of 256 x 128 and
    # 256 x 256 tiles (opt-in)
    for stages, tstore, pair in ((0, 1, 0), (2, 1, 0), (0, 0, 0), (2, 0, 0), (0, 1, 1), (0, 1, 2)):
        assert lib.sf_gemm_split6_set_stages(stages) == 0
        assert lib.sf_gemm_set_tma_store(tstore) == 0
        assert lib.sf_gemm_set_pair(pair) == 0
        c = torch.full((m, n), float("nan"), device="cuda")
        N.call("sf_gemm_f16x3", m, n, k, pa.data_ptr(), None, pb.data_ptr(), c.data_ptr(), n, bias.data_ptr(), 0.0,
               ws.data_ptr(), nb, st)
        assert _err(c, ref) <= max(2 * e32, 2.0 ** -22), (stages, tstore, _err(c, ref), e32)
        outs.append(c)
    lib.sf_gemm_split6_set_stages(0)
    lib.sf_gemm_set_tma_store(1)
    lib.sf_gemm_set_pair(0)
    assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3])   # same sums, either epilogue
    assert torch.equal(outs[0], outs[4]) or min(m, n) >= 256      # CTA pairs only when m, n >= 256


@pytest.mark.parametrize("m,k,n", [(1000, 768, 136), (16384, 3072, 768), (4096, 2304, 768), (333, 520, 264)])
def test_f16x3_row_scaled_gradients_vs_fp64(G, m, k, n):
    """Input-gradient products: g's rows span 2^-40 .. 2^20 (far past fp16's
    range; one row does not), split per row into fp16 planes scaled by 2^e_r
    (row maximum in [2^14, 2^15)) and multiplied back by 2^-e_r in the
    epilogue -- every row's error relative to that row's own maximum within
    twice strict SGEMM's worst row."""
    from paper_2305_18513_b200 import _native as N
    lib = N.load()
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(m + n + 7 * k)
    a = torch.randn(m, k, device="cuda", generator=g) * torch.exp2(
        torch.randint(-40, 21, (m, 1), device="cuda", generator=g).float())
    a[0].zero_()                                            # an all-zero row: scale 1
    w = torch.randn(n, k, device="cuda", generator=g) * 0.02
    ref = a.double() @ w.double().t()
    G.set_mode("fp32")
    c32 = G.mm(a, w.t())
    pa = torch.empty(2, m, k, dtype=torch.float16, device="cuda")
    rs = torch.empty(m, device="cuda")
    pb = torch.empty(2, n, k, dtype=torch.float16, device="cuda")
    N.call("sf_split2_f16_rows", a.data_ptr(), m, k, k, pa.data_ptr(), rs.data_ptr(), st)
    N.call("sf_split2_f16", w.data_ptr(), n, k, k, 0, pb.data_ptr(), st)
    amax = a.abs().amax(dim=1)
    torch.cuda.synchronize()
    nz = amax > 0
    assert torch.all((amax[nz] / rs[nz] >= 2.0 ** 14) & (amax[nz] / rs[nz] < 2.0 ** 15))
    assert rs[0].item() == 1.0
    nb = lib.sf_gemm_split6_ws_bytes(m, n, k)
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    c = torch.full((m, n), float("nan"), device="cuda")
    N.call("sf_gemm_f16x3", m, n, k, pa.data_ptr(), rs.data_ptr(), pb.data_ptr(), c.data_ptr(), n, None, 0.0,
           ws.data_ptr(), nb, st)
    rowref = ref.abs().amax(dim=1).clamp_min(1e-300)
    e16 = ((c.double() - ref).abs().amax(dim=1) / rowref)[nz]
    e32 = ((c32.double() - ref).abs().amax(dim=1) / rowref)[nz]
    assert torch.isfinite(c).all() and torch.all(c[0] == 0)
    # every row at strict SGEMM's level (its worst row), however small the row
    assert e16.max().item() <= max(2 * e32.max().item(), 2.0 ** -22), (e16.max().item(), e32.max().item())


@pytest.mark.parametrize("which", ["ln_bwd_dense", "ln_bwd_cols", "ln_bwd_sparse", "gelu_bwd"])
def test_backward_producers_row_scaled_planes(which):
    """The backward producers' row-scaled fp16 planes (form 2) and row scales
    are bit-identical to sf_split2_f16_rows of the fp32 output they write."""
    from paper_2305_18513_b200 import _native as N
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(len(which))
    rows, H = 300, 768
    if which.startswith("ln"):
        gr = torch.randn(rows, H, generator=g, device="cuda") * torch.exp2(
            torch.randint(-30, 10, (rows, 1), generator=g, device="cuda").float())
        xt = torch.randn(rows, H, generator=g, device="cuda")
        gam, rstd = torch.rand(H, generator=g, device="cuda") + 0.5, torch.rand(rows, generator=g, device="cuda") + 0.5
        dx = torch.empty_like(gr)
        ws = torch.empty(N.load().sf_layernorm_bwd_workspace_bytes(rows, H), dtype=torch.uint8, device="cuda")
        dg, db = (torch.empty(H, device="cuda"), torch.empty(H, device="cuda")) if which == "ln_bwd_cols" else (None, None)
        pl = torch.empty(2 * rows * H, dtype=torch.float16, device="cuda")
        rs = torch.empty(rows, device="cuda")
        if which == "ln_bwd_sparse":
            from paper_2305_18513_b200 import compression as Cz
            sp = Cz.prune_topk(xt, 0.1, True, row_pointers=True)
            N.call("sf_layernorm_bwd_pf", gr.data_ptr(), gam.data_ptr(), None, sp.values.data_ptr(),
                   sp.indices.data_ptr(), sp.values.numel(), sp.row_ptr.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
                   None, None, rows, H, ws.data_ptr(), pl.data_ptr(), 2, rs.data_ptr(), st)
        else:
            N.call("sf_layernorm_bwd_pf", gr.data_ptr(), gam.data_ptr(), xt.data_ptr(), None, None, 0, None,
                   rstd.data_ptr(), dx.data_ptr(), dg.data_ptr() if dg is not None else None,
                   db.data_ptr() if db is not None else None, rows, H, ws.data_ptr(), pl.data_ptr(), 2,
                   rs.data_ptr(), st)
        out = dx
    else:
        L = 4 * H
        n = rows * L
        gr = torch.randn(rows, L, generator=g, device="cuda") * torch.exp2(
            torch.randint(-30, 10, (rows, 1), generator=g, device="cuda").float())
        packed = torch.randint(0, 256, ((n + 1) // 2,), generator=g, device="cuda", dtype=torch.uint8)
        s = torch.tensor([1], dtype=torch.int32, device="cuda")
        dx = torch.empty_like(gr)
        pl = torch.empty(2 * n, dtype=torch.float16, device="cuda")
        rs = torch.empty(rows, device="cuda")
        N.call("sf_gelu_bwd_packed4_pf", gr.data_ptr(), packed.data_ptr(), s.data_ptr(), 2, dx.data_ptr(), n, L,
               pl.data_ptr(), 2, rs.data_ptr(), st)
        ref_dx = torch.empty_like(gr)
        N.call("sf_gelu_bwd_packed4", gr.data_ptr(), packed.data_ptr(), s.data_ptr(), 2, ref_dx.data_ptr(), n, st)
        torch.cuda.synchronize()
        assert torch.equal(dx, ref_dx)
        out = dx
    r_, c_ = out.numel() // out.shape[-1], out.shape[-1]
    ref = torch.empty(2 * out.numel(), dtype=torch.float16, device="cuda")
    rref = torch.empty(r_, device="cuda")
    N.call("sf_split2_f16_rows", out.data_ptr(), r_, c_, c_, ref.data_ptr(), rref.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(rs, rref)
    assert torch.equal(pl.view(torch.int16), ref.view(torch.int16))


def test_step_f16x3_matches_bf16x6():
    """A few ILS fine-tune iterations with the forward and input-gradient
    products on f16x3 (the default) against the same run with every product
    on bf16x6: losses within float32 tolerance, identical freeze decisions,
    parameters within tolerance -- the operand form is a speed choice, not a
    numerics change beyond strict SGEMM's level."""
    import numpy as np
    import paper_2305_18513_b200 as sf
    from paper_2305_18513_b200 import gemm as G
    old = (G.get_mode(), G.fwd_f16, G.dgrad_f16)
    G.set_mode("bf16x6")
    cfg = sf.ModelConfig(blocks=2, hidden=256, heads=4, max_seq=64, vocab=500, num_classes=3)
    runs = []
    try:
        for f16 in (True, False):
            G.fwd_f16 = G.dgrad_f16 = f16
            m = sf.build_model(cfg, seed=5)
            rc = sf.RunConfig(scheduler="ils", freeze_rate=0.5, epochs=1, batch_size=8, seed=2, lr=1e-3,
                              warmup_frac=0.0, compression=sf.CompressionConfig.all_on())
            rng = np.random.default_rng(1)
            toks, labs = rng.integers(0, 500, (32, 64)), rng.integers(0, 3, 32)
            log = sf.fine_tune(m, (toks, labs), rc)
            runs.append(([p.detach().cpu().numpy() for p in m.parameters()], [mm[1] for mm in log.metrics],
                         [sorted(d.active_ids) for d in log.decisions]))
    finally:
        G.set_mode(old[0])
        G.fwd_f16, G.dgrad_f16 = old[1], old[2]
    (p1, l1, d1), (p0, l0, d0) = runs
    assert d1 == d0
    assert np.allclose(l1, l0, rtol=2e-5, atol=1e-6), (l1, l0)
    # per tensor: AdamW's m / sqrt(v) amplifies last-bit gradient differences
    # where |g| ~ eps, so elementwise bounds are meaningless; the tensors agree
    for a, b in zip(p1, p0):
        assert np.linalg.norm(a.astype(np.float64) - b) <= 1e-4 * np.linalg.norm(b.astype(np.float64)) + 1e-7
