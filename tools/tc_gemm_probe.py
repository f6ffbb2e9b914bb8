#!/usr/bin/env python
"""Probe the tcgen05 split-bf16 fp32 GEMM (csrc/gemm_tc.cu) against fp64 and
cuBLASLt BF16x9 on the step's shapes: accuracy, time, stage count.

    python tools/tc_gemm_probe.py
"""

from __future__ import annotations

import sys

import torch

sys.path.insert(0, ".")
from paper_2305_18513_b200 import _native as N  # noqa: E402
from paper_2305_18513_b200 import gemm as G  # noqa: E402


def split_ref(x):
    h = x.bfloat16()
    r = x - h.float()
    m = r.bfloat16()
    lo = (r - m.float()).bfloat16()
    return torch.stack([h, m, lo])


def planes(x, transpose=False):
    rows, cols = x.shape
    out = torch.empty((3, cols, rows) if transpose else (3, rows, cols), dtype=torch.bfloat16, device=x.device)
    N.call("sf_split3_bf16", x.data_ptr(), rows, cols, x.stride(0), int(transpose), out.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    return out


WS = {}


def tc(ap, bp, m, n, k, out, bias=None, beta=0.0):
    nb = N.load().sf_gemm_split6_ws_bytes(m, n, k)
    ws = WS.get(nb)
    if ws is None:
        ws = WS[nb] = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    N.call("sf_gemm_split6", m, n, k, ap.data_ptr(), bp.data_ptr(), out.data_ptr(), n,
           bias.data_ptr() if bias is not None else None, beta, ws.data_ptr(), nb,
           torch.cuda.current_stream().cuda_stream)
    return out


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def main():
    torch.manual_seed(0)
    lib = N.load()
    x = torch.randn(1000, 776, device="cuda")
    y = torch.randn(333, 777, device="cuda")
    ok = torch.equal(planes(x), split_ref(x)) and torch.equal(planes(y, True), split_ref(y.t().contiguous()))
    print("split3 exact:", ok)
    shapes = [(256, 128, 64), (300, 200, 72), (16384, 3072, 768), (16384, 768, 3072), (16384, 768, 768),
              (16384, 2304, 768), (768, 768, 16384), (3072, 768, 16384), (768, 3072, 16384)]
    for m, n, k in shapes:
        a = torch.randn(m, k, device="cuda")
        b = torch.randn(n, k, device="cuda")
        bias = torch.randn(n, device="cuda")
        ref = (a.double() @ b.double().t() + bias.double())
        scale = ref.abs().max().item()
        ap, bp = planes(a), planes(b)
        line = f"{m:6d}x{n:5d}x{k:6d} z{lib.sf_gemm_split6_splits(m, n, k)}"
        for st in (0, 1):
            lib.sf_gemm_split6_set_stages(st)
            out = torch.empty(m, n, device="cuda")
            tc(ap, bp, m, n, k, out, bias)
            torch.cuda.synchronize()
            err = (out.double() - ref).abs().max().item() / scale
            us = timeit(lambda: tc(ap, bp, m, n, k, out, bias))
            tf = 2.0 * m * n * k / us / 1e6
            line += f" | s{st} {us:7.1f}us {tf:5.0f}TF err {err:.2e}"
        lib.sf_gemm_split6_set_stages(0)
        out = torch.empty(m, n, device="cuda")
        nb = lib.sf_gemm_split6_ws_bytes(m, n, k)
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")

        def a32():
            N.call("sf_gemm_split6_a32", m, n, k, a.data_ptr(), k, bp.data_ptr(), out.data_ptr(), n,
                   bias.data_ptr(), 0.0, ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
        a32()
        torch.cuda.synchronize()
        err = (out.double() - ref).abs().max().item() / scale
        us = timeit(a32)
        line += f" | a32 {us:7.1f}us err {err:.2e}"
        o2 = torch.empty(m, n, device="cuda")
        us9 = timeit(lambda: G.mm(a, b.t(), bias=bias, out=o2, mode="bf16x9"))
        err9 = (o2.double() - ref).abs().max().item() / scale
        usf = timeit(lambda: G.mm(a, b.t(), bias=bias, out=o2, mode="fp32"), reps=3)
        errf = (o2.double() - ref).abs().max().item() / scale
        usp = timeit(lambda: planes(a)) + timeit(lambda: planes(b))
        line += f" | bf16x9 {us9:7.1f}us err {err9:.2e} | sgemm err {errf:.2e} ({usf:.0f}us) | split {usp:.1f}us"
        print(line, flush=True)
    # beta accumulation
    lib.sf_gemm_split6_set_stages(2)
    m, n, k = 512, 384, 256
    a, b = torch.randn(m, k, device="cuda"), torch.randn(n, k, device="cuda")
    c0 = torch.randn(m, n, device="cuda")
    out = c0.clone()
    tc(planes(a), planes(b), m, n, k, out, None, 1.0)
    ref = a.double() @ b.double().t() + c0.double()
    print("beta=1 err", ((out.double() - ref).abs().max() / ref.abs().max()).item())


if __name__ == "__main__":
    main()
