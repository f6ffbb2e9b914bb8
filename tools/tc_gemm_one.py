#!/usr/bin/env python
"""One bf16x6 product of a given shape (for ncu captures):
    python tools/tc_gemm_one.py M N K"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_18513_b200 import gemm as G  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
a = torch.randn(m, k, device="cuda")
w = torch.randn(n, k, device="cuda")
for _ in range(3):
    G.mm(a, w.t(), mode="bf16x6")
torch.cuda.synchronize()
