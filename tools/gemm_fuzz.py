#!/usr/bin/env python
"""Fuzz G.mm (every layout: plain, a^T, b^T, broadcast batch, bias, beta)
against an fp64 product in the active mode."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_18513_b200 import gemm as G  # noqa: E402


def main(mode=None):
    g = torch.Generator(device="cuda").manual_seed(0)
    bad = 0
    for trial in range(300):
        m, n, k = [int(v) for v in torch.randint(1, 300, (3,))]
        if trial % 3 == 0:
            k = 8 * max(1, k // 8)
            n = 4 * max(1, n // 4)
        ta, tb = trial % 2 == 0, trial % 4 < 2
        a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
        b = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
        A, Bm = (a.t() if ta else a), (b.t() if tb else b)
        bias = torch.randn(n, device="cuda", generator=g) if trial % 5 == 0 else None
        beta = 1.0 if trial % 7 == 0 else 0.0
        out = torch.randn(m, n, device="cuda", generator=g) if beta else None
        ref = A.double() @ Bm.double()
        if bias is not None:
            ref += bias.double()
        if beta:
            ref += out.double()
        y = G.mm(A, Bm, bias=bias, out=out, beta=beta, mode=mode)
        err = ((y.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
        if not err < 1e-5:
            bad += 1
            print("BAD", m, n, k, ta, tb, bias is not None, beta, err)
    # broadcast batch
    x = torch.randn(200, 64, device="cuda")
    w = torch.randn(3, 64, 96, device="cuda")
    y = G.mm(x.expand(3, 200, 64), w, mode=mode)
    err = ((y.double() - x.double() @ w.double()).abs().max()).item()
    print("bcast err", err)
    print("bad", bad, "of 300")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
