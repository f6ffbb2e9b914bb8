"""Per-kernel HBM roofline measurement at BASELINE shapes (CUDA events on the
launching stream, inputs larger than L2 or L2 flushed between launches).

    python -m paper_2305_18513_b200.kernel_bench [--json] [--iters N] [--core]

Algorithmic bytes per element follow SURVEY.md §8(d):
quant8/dequant8 5, pack4/unpack4 4.5 (+4 when the prescale pass is counted),
prune/restore 4 + 8k/n, distance 8 per param, AdamW+distance 28 per param.
"""

from __future__ import annotations

import json
import os
import sys

import torch

from . import _native as N
from . import compression as Cz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak_hbm_gbs() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class L2Flush:
    """Write a buffer larger than L2 (126 MB), then read another one: the
    written lines' write-back happens here, not inside the timed kernel, and
    L2 is left holding clean lines that no timed input shares."""

    def __init__(self, nbytes=256 << 20):
        self.buf = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
        self.rbuf = torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda")
        self.sink = torch.empty((), dtype=torch.float32, device="cuda")

    def __call__(self):
        self.buf.fill_(0.0)
        torch.sum(self.rbuf, dim=0, out=self.sink)


def time_launches(fn, iters=20, warmup=None, flush=None):
    """Average device ms per call of fn() (events on the current stream)."""
    if warmup is None:
        warmup = 3 if iters >= 5 else 1
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    total = 0.0
    for _ in range(iters):
        if flush is not None:
            flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        total += a.elapsed_time(b)
    return total / iters


def measure(B=128, T=128, H=768, heads=12, iters=20, core=False):
    """core: the step's kernels at BERT-base shapes only (no ViT / BERT-large
    attention rows, no GEMM variants) -- the set the ncu capture profiles."""
    peak, peak_kind = peak_hbm_gbs()
    g = torch.Generator(device="cuda").manual_seed(0)
    BTH, BT4H, BhTT = B * T * H, B * T * 4 * H, B * heads * T * T
    flush = L2Flush()
    res = {}
    st = torch.cuda.current_stream().cuda_stream
    lib = N.load()

    def rec(name, n, bpe, ms, extra=None):
        gbs = n * bpe / (ms * 1e-3) / 1e9
        r = {"n": n, "bytes_per_elt": bpe, "ms": ms, "gbs": gbs, "frac": gbs / peak}
        if extra:
            r.update(extra)
        res[name] = r

    x = torch.randn(BT4H, generator=g, device="cuda")
    codes = torch.empty(BT4H, dtype=torch.int8, device="cuda")
    y = torch.empty_like(x)
    rec("quant8_dense", BT4H, 5, time_launches(
        lambda: lib.sf_quant8(x.data_ptr(), codes.data_ptr(), BT4H, 4, 1, st), iters, flush=flush))
    rec("dequant8_dense", BT4H, 5, time_launches(
        lambda: lib.sf_dequant8(codes.data_ptr(), y.data_ptr(), BT4H, 4, 1, st), iters, flush=flush))

    s = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(lib.sf_prescale_workspace_bytes(BT4H), dtype=torch.uint8, device="cuda")
    packed = torch.empty((BT4H + 1) // 2, dtype=torch.uint8, device="cuda")
    q = float(Cz._quantile(99.9))
    rec("prescale_hist", BT4H, 4, time_launches(
        lambda: lib.sf_prescale_exp(x.data_ptr(), BT4H, q, 1.75, s.data_ptr(), None, ws.data_ptr(), st),
        iters, flush=flush))
    rec("quant4_pack", BT4H, 4.5, time_launches(
        lambda: lib.sf_quant4_pack(x.data_ptr(), packed.data_ptr(), BT4H, s.data_ptr(), 2, st),
        iters, flush=flush))

    def packed_all():
        lib.sf_prescale_exp(x.data_ptr(), BT4H, q, 1.75, s.data_ptr(), None, ws.data_ptr(), st)
        lib.sf_quant4_pack(x.data_ptr(), packed.data_ptr(), BT4H, s.data_ptr(), 2, st)
    ms = time_launches(packed_all, iters, flush=flush)
    rec("packed4_total", BT4H, 4.5, ms, {"bytes_per_elt_with_prescale_pass": 8.5})
    rec("unpack4", BT4H, 4.5, time_launches(
        lambda: lib.sf_unpack4_dequant(packed.data_ptr(), y.data_ptr(), BT4H, s.data_ptr(), 2, st),
        iters, flush=flush))
    # the step's GELU forward: bias added in place, GELU, K3 histogram in one
    # read (x in; x + b and y out: 12 B/elt), then the exponent select
    bias4 = torch.randn(4 * H, generator=g, device="cuda")
    xg = torch.empty_like(x)
    rec("gelu_fwd_prescale_bias", BT4H, 12, time_launches(
        lambda: lib.sf_gelu_fwd_prescale_bias(xg.data_ptr(), bias4.data_ptr(), 4 * H, y.data_ptr(), BT4H, q,
                                              1.75, s.data_ptr(), ws.data_ptr(), st), iters,
        flush=lambda: (xg.copy_(x), flush())))
    del xg
    gg = torch.randn(BT4H, generator=g, device="cuda")
    rec("gelu_bwd_packed4", BT4H, 8.5, time_launches(
        lambda: lib.sf_gelu_bwd_packed4(gg.data_ptr(), packed.data_ptr(), s.data_ptr(), 2,
                                        y.data_ptr(), BT4H, st), iters, flush=flush))
    del gg

    sc = torch.randn(BhTT, generator=g, device="cuda")
    pc = torch.empty(BhTT, dtype=torch.int8, device="cuda")
    pr = torch.empty_like(sc)
    rec("softmax_fwd_q8", BhTT, 9, time_launches(
        lambda: lib.sf_softmax_fwd_q8(sc.data_ptr(), pr.data_ptr(), pc.data_ptr(), B * heads * T, T,
                                      0.125, 4, 1, st), iters, flush=flush))
    del sc, pc, pr

    xt = torch.randn(B * T, H, generator=g, device="cuda")
    xt = (xt - xt.mean(-1, keepdim=True)) / xt.std(-1, keepdim=True, unbiased=False)
    xt = xt.reshape(-1).contiguous()
    k = Cz.keep_count(BTH, 0.1)
    vals = torch.empty(k, device="cuda")
    idx = torch.empty(k, dtype=torch.int32, device="cuda")
    pws = torch.empty(lib.sf_prune_workspace_bytes(BTH), dtype=torch.uint8, device="cuda")
    bpe = 4 + 8 * k / BTH
    rec("prune_topk", BTH, bpe, time_launches(
        lambda: lib.sf_prune_topk(xt.data_ptr(), BTH, k, 1, vals.data_ptr(), idx.data_ptr(),
                                  pws.data_ptr(), st), iters, flush=flush))
    # the model path's form: row pointers and a per-site hint, alternating two
    # batches of the same LayerNorm site (the hint always comes from the other)
    xt2 = torch.randn(B * T, H, generator=g, device="cuda")
    xt2 = ((xt2 - xt2.mean(-1, keepdim=True)) / xt2.std(-1, keepdim=True, unbiased=False)).reshape(-1).contiguous()
    hint = Cz.new_prune_hint()
    rph = torch.empty(B * T + 1, dtype=torch.int32, device="cuda")
    flip = [0]

    def _hinted():
        flip[0] ^= 1
        src = xt if flip[0] else xt2
        return lib.sf_prune_topk_hint(src.data_ptr(), BTH, k, 1, vals.data_ptr(), idx.data_ptr(), H,
                                      rph.data_ptr(), hint.data_ptr(), pws.data_ptr(), st)
    _hinted()
    rec("prune_topk_hint", BTH, bpe, time_launches(_hinted, iters, flush=flush))
    del xt2
    dense = torch.empty(BTH, device="cuda")
    rec("restore", BTH, bpe, time_launches(
        lambda: lib.sf_restore(vals.data_ptr(), idx.data_ptr(), k, dense.data_ptr(), BTH, st),
        iters, flush=flush))
    # with the CSR row pointers the rows variant of the prune writes (the model path's form)
    rp = torch.empty(B * T + 1, dtype=torch.int32, device="cuda")
    lib.sf_prune_topk_rows(xt.data_ptr(), BTH, k, 1, vals.data_ptr(), idx.data_ptr(), H, rp.data_ptr(),
                           pws.data_ptr(), st)
    rec("restore_rows", BTH, bpe, time_launches(
        lambda: lib.sf_restore_rows(vals.data_ptr(), idx.data_ptr(), k, rp.data_ptr(), H, dense.data_ptr(), BTH, st),
        iters, flush=flush))

    # LayerNorm forward (y + x~) and the frozen/pruned backward (sparse x~)
    rows = B * T
    xin = torch.randn(rows, H, generator=g, device="cuda")
    gam = torch.ones(H, device="cuda")
    bet = torch.zeros(H, device="cuda")
    yln = torch.empty_like(xin)
    xtl = torch.empty_like(xin)
    rs = torch.empty(rows, device="cuda")
    rec("layernorm_fwd", BTH, 12, time_launches(
        lambda: lib.sf_layernorm_fwd(xin.data_ptr(), gam.data_ptr(), bet.data_ptr(), yln.data_ptr(),
                                     xtl.data_ptr(), rs.data_ptr(), rows, H, 1e-5, st), iters, flush=flush))
    resid = torch.randn(rows, H, generator=g, device="cuda")
    bH = torch.randn(H, generator=g, device="cuda")
    rec("layernorm_fwd_residual", BTH, 16, time_launches(
        lambda: lib.sf_layernorm_fwd_residual(resid.data_ptr(), xin.data_ptr(), bH.data_ptr(), gam.data_ptr(),
                                              bet.data_ptr(), yln.data_ptr(), None, xtl.data_ptr(), rs.data_ptr(),
                                              rows, H, 1e-5, st), iters, flush=flush))
    del resid
    # head split (+ bias) / merge: pure moves, 8 B/elt
    hs = torch.empty(B, heads, T, H // heads, device="cuda")
    rec("split_heads", BTH, 8, time_launches(
        lambda: lib.sf_split_heads(xin.data_ptr(), bH.data_ptr(), hs.data_ptr(), None, B, T, heads, H // heads,
                                   0, 0, st), iters, flush=flush))
    rec("merge_heads", BTH, 8, time_launches(
        lambda: lib.sf_merge_heads(hs.data_ptr(), yln.data_ptr(), B, T, heads, H // heads, st), iters,
        flush=flush))
    del hs
    lws = torch.empty(lib.sf_layernorm_bwd_workspace_bytes(rows, H), dtype=torch.uint8, device="cuda")
    rp = torch.empty(rows + 1, dtype=torch.int32, device="cuda")      # CSR rows of the pruned x~
    lib.sf_prune_topk_rows(xt.data_ptr(), BTH, k, 1, vals.data_ptr(), idx.data_ptr(), H, rp.data_ptr(),
                           pws.data_ptr(), st)
    gln = torch.randn(rows, H, generator=g, device="cuda")
    rec("layernorm_bwd_sparse", BTH, 8 + 8 * k / BTH, time_launches(
        lambda: lib.sf_layernorm_bwd(gln.data_ptr(), gam.data_ptr(), None, vals.data_ptr(), idx.data_ptr(),
                                     k, rp.data_ptr(), rs.data_ptr(), yln.data_ptr(), None, None, rows, H,
                                     lws.data_ptr(), st), iters, flush=flush))
    rec("layernorm_bwd_dense", BTH, 12, time_launches(
        lambda: lib.sf_layernorm_bwd(gln.data_ptr(), gam.data_ptr(), xtl.data_ptr(), None, None, 0,
                                     None, rs.data_ptr(), yln.data_ptr(), None, None, rows, H,
                                     lws.data_ptr(), st), iters, flush=flush))
    dgm = torch.empty(H, device="cuda")
    dbt = torch.empty(H, device="cuda")
    rec("layernorm_bwd_dense_cols", BTH, 12, time_launches(
        lambda: lib.sf_layernorm_bwd(gln.data_ptr(), gam.data_ptr(), xtl.data_ptr(), None, None, 0,
                                     None, rs.data_ptr(), yln.data_ptr(), dgm.data_ptr(), dbt.data_ptr(), rows, H,
                                     lws.data_ptr(), st), iters, flush=flush))
    del xin, yln, xtl, gln

    # fused attention core (fp32-accurate tensor-core MMAs): TFLOP/s, not HBM.
    # BERT-base (T = 128: one CTA per head), ViT-B/16 (T = 197) and
    # BERT-large (T = 384): the query-tiled kernels
    def attention_rows(tag, Ba, Ta, ha, Ha):
        dh = Ha // ha
        ra = Ba * Ta
        y3 = torch.randn(3, ra, Ha, generator=g, device="cuda")
        bqkv = [torch.randn(Ha, generator=g, device="cuda") * 0.1 for _ in range(3)]
        ctxo = torch.empty(ra, Ha, device="cuda")
        cq = torch.empty(Ba, ha, Ta, dh, dtype=torch.int8, device="cuda")
        ck, cv = torch.empty_like(cq), torch.empty_like(cq)
        cp = torch.empty(Ba, ha, Ta, Ta, dtype=torch.int8, device="cuda")
        gcat = torch.empty(ra, 3 * Ha, device="cuda")
        nws = lib.sf_attention_bwd_workspace_bytes(Ba, Ta, ha)
        ws = torch.empty(max(nws, 16), dtype=torch.uint8, device="cuda")
        flops_f = 4.0 * Ba * ha * Ta * Ta * dh
        ms = time_launches(lambda: lib.sf_attention_fwd(y3.data_ptr(), bqkv[0].data_ptr(), bqkv[1].data_ptr(),
                                                        bqkv[2].data_ptr(), Ba, Ta, ha, dh, 0.125, 4, ctxo.data_ptr(),
                                                        cq.data_ptr(), ck.data_ptr(), cv.data_ptr(), cp.data_ptr(), st),
                           iters, flush=flush)
        res["attention_fwd" + tag] = {"n": Ba * ha, "ms": ms, "tflops": flops_f / (ms * 1e-3) / 1e12,
                                      "bound": "tensor (fp32-accurate bf16 split products)", "T": Ta}
        ms = time_launches(lambda: lib.sf_attention_bwd(ctxo.data_ptr(), cq.data_ptr(), ck.data_ptr(), cv.data_ptr(),
                                                        cp.data_ptr(), Ba, Ta, ha, dh, 0.125, 4, gcat.data_ptr(),
                                                        ws.data_ptr() if nws else None, st),
                           iters, flush=flush)
        res["attention_bwd" + tag] = {"n": Ba * ha, "ms": ms, "tflops": 2 * flops_f / (ms * 1e-3) / 1e12,
                                      "bound": "tensor (fp32-accurate bf16 split products)", "T": Ta}

    attention_rows("", B, T, heads, H)
    if not core:
        attention_rows("_t197", 128, 197, 12, 768)
        attention_rows("_t384", 16, 384, 16, 1024)

    # operand split (10 B/elt) and the tcgen05 split-bf16 GEMM at the step's shapes
    xs = torch.randn(rows, 4 * H, generator=g, device="cuda")
    planes = torch.empty(3 * rows * 4 * H, dtype=torch.bfloat16, device="cuda")
    rec("split3_bf16", xs.numel(), 10, time_launches(
        lambda: N.call("sf_split3_bf16", xs.data_ptr(), rows, 4 * H, 4 * H, 0, planes.data_ptr(), st), iters,
        flush=flush))
    rec("split3_bf16_t", xs.numel(), 10, time_launches(
        lambda: N.call("sf_split3_bf16", xs.data_ptr(), rows, 4 * H, 4 * H, 1, planes.data_ptr(), st), iters,
        flush=flush))
    del xs, planes
    for tag, (m, n, k) in {"ffn_up": (rows, 4 * H, H), "ffn_down": (rows, H, 4 * H), "attn_out": (rows, H, H),
                           "wgrad_ffn": (4 * H, H, rows)}.items():
        pa = torch.randn(3 * m * k, generator=g, device="cuda").bfloat16()
        pb = torch.randn(3 * n * k, generator=g, device="cuda").bfloat16()
        cc = torch.empty(m, n, device="cuda")
        nb = lib.sf_gemm_split6_ws_bytes(m, n, k)
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
        ms = time_launches(lambda: N.call("sf_gemm_split6", m, n, k, pa.data_ptr(), pb.data_ptr(), cc.data_ptr(), n,
                                          None, 0.0, ws.data_ptr(), nb, st), iters, flush=flush)
        tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
        res[f"gemm_{tag}"] = {"n": m * n, "ms": ms, "tflops": tf, "bf16_tflops": 6 * tf,
                              "shape": [m, n, k], "bound": "tensor (6 bf16 products per fp32 product)"}
        del pa, pb, cc, ws

    # the forward products in the f16x3 form (two fp16 planes per operand,
    # three MMAs): N = 256 tiles (auto) and N = 128 tiles
    xs = torch.randn(rows, 4 * H, generator=g, device="cuda")
    planes = torch.empty(2 * rows * 4 * H, dtype=torch.float16, device="cuda")
    rec("split2_f16", xs.numel(), 8, time_launches(
        lambda: N.call("sf_split2_f16", xs.data_ptr(), rows, 4 * H, 4 * H, 0, planes.data_ptr(), st), iters,
        flush=flush))
    del xs, planes
    for tag, (m, n, k) in {"ffn_up": (rows, 4 * H, H), "ffn_down": (rows, H, 4 * H), "attn_out": (rows, H, H),
                           "qkv": (rows, 3 * H, H)}.items():
        pa = torch.randn(2 * m * k, generator=g, device="cuda").half()
        pb = torch.randn(2 * n * k, generator=g, device="cuda").half()
        cc = torch.empty(m, n, device="cuda")
        nb = lib.sf_gemm_split6_ws_bytes(m, n, k)
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
        variants = ((0, "", 1, 0), (0, "_pair", 1, 1), (0, "_pair256", 1, 2), (2, "_n128", 1, 0), (0, "_direct", 0, 0))
        for st_mode, sfx, tstore, pair in variants[:1] if core else variants:
            lib.sf_gemm_split6_set_stages(st_mode)
            lib.sf_gemm_set_tma_store(tstore)
            lib.sf_gemm_set_pair(pair)
            ms = time_launches(lambda: N.call("sf_gemm_f16x3", m, n, k, pa.data_ptr(), None, pb.data_ptr(), cc.data_ptr(),
                                              n, None, 0.0, ws.data_ptr(), nb, st), iters, flush=flush)
            tf = 2.0 * m * n * k / (ms * 1e-3) / 1e12
            res[f"f16x3_{tag}{sfx}"] = {"n": m * n, "ms": ms, "tflops": tf, "bf16_tflops": 3 * tf,
                                        "shape": [m, n, k], "bound": "tensor (3 fp16 products per fp32 product)"}
        lib.sf_gemm_split6_set_stages(0)
        lib.sf_gemm_set_tma_store(1)
        lib.sf_gemm_set_pair(0)
        del pa, pb, cc, ws

    # fused AdamW + distance over one BERT-base block's FFN pair + the word embedding
    from .scheduler import DistancePlan
    shapes = [(768, 3072), (3072,), (3072, 768), (768,), (30522, 768)]
    ps = [torch.randn(s, generator=g, device="cuda") * 0.02 for s in shapes]
    gs = [torch.randn(s, generator=g, device="cuda") * 0.01 for s in shapes]
    ms_ = [torch.zeros(s, device="cuda") for s in shapes]
    vs_ = [torch.zeros(s, device="cuda") for s in shapes]
    plan = DistancePlan([p.numel() for p in ps])
    c = dict(b1=0.9, ob1=0.1, b2=0.999, ob2=0.001, bc1=0.1, bc2=0.001, eps=1e-8, wd=0.01, lr=5e-5)
    rows_ = [{"slot": j, "A": ps[j].data_ptr(), "B": gs[j].data_ptr(), "M": ms_[j].data_ptr(),
              "V": vs_[j].data_ptr(), "consts": c} for j in range(len(ps))]
    layers = [(0, 2, 0, ps[0].numel() + ps[1].numel()), (2, 2, 1, ps[2].numel() + ps[3].numel()),
              (4, 1, 2, ps[4].numel())]
    dd = torch.zeros(3, dtype=torch.float64, device="cuda")
    nparam = sum(p.numel() for p in ps)
    # the launch alone (tables uploaded once by run(); the host-side table
    # build is part of the step, timed there)
    plan.run(rows_, layers, dd, N.UPDATE_ADAMW)
    rec("adamw_distance", nparam, 28, time_launches(plan.relaunch, iters, flush=flush))
    rows_s = [{"slot": j, "A": ps[j].data_ptr(), "B": gs[j].data_ptr(), "lr": 5e-5} for j in range(len(ps))]
    # SGD + distance: 12 B per param (p, g read; p written)
    plan.run(rows_s, layers, dd, N.UPDATE_SGD)
    rec("sgd_distance", nparam, 12, time_launches(plan.relaunch, iters, flush=flush))
    torch.cuda.synchronize()
    return {"peak_hbm_gbs": peak, "peak_kind": peak_kind, "kernels": res,
            "shape": {"B": B, "T": T, "H": H, "heads": heads}}


if __name__ == "__main__":
    it = 20
    if "--iters" in sys.argv:
        it = int(sys.argv[sys.argv.index("--iters") + 1])
    out = measure(iters=it, core="--core" in sys.argv)
    if "--json" in sys.argv:
        print(json.dumps(out))
    else:
        print(f"peak {out['peak_hbm_gbs']} GB/s ({out['peak_kind']})")
        for k, v in out["kernels"].items():
            if "tflops" in v:
                extra = f"  = {v['bf16_tflops']:.0f} bf16-TFLOP/s {v['shape']}" if "bf16_tflops" in v else ""
                print(f"{k:22s} n={v['n']:>11d} {v['ms']*1e3:9.1f} us  {v['tflops']:8.1f} TFLOP/s (fp32 flops){extra}")
            else:
                print(f"{k:22s} n={v['n']:>11d} {v['ms']*1e3:9.1f} us  {v['gbs']:8.1f} GB/s  frac {v['frac']:.3f}")
