"""Inspect the prune kernel's state after one call (mode, bracket, counts)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2305_18513_b200 import _native as N  # noqa: E402
from paper_2305_18513_b200 import compression as Cz  # noqa: E402

B, T, H = 128, 128, 768
g = torch.Generator(device="cuda").manual_seed(0)
xt = torch.randn(B * T, H, generator=g, device="cuda")
xt = ((xt - xt.mean(-1, keepdim=True)) / xt.std(-1, keepdim=True, unbiased=False)).reshape(-1).contiguous()
n = xt.numel()
k = Cz.keep_count(n, 0.1)
lib = N.load()
vals = torch.empty(k, device="cuda")
idx = torch.empty(k, dtype=torch.int32, device="cuda")
ws = torch.zeros(lib.sf_prune_workspace_bytes(n), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
N.call("sf_prune_topk", xt.data_ptr(), n, k, 1, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), st)
torch.cuda.synchronize()
hdr = ws[:64].cpu().numpy()
u32 = hdr.view(np.uint32)
u64 = hdr.view(np.uint64)
print("tickets", u32[0:4], "T", hex(u32[4]), "fine_lo", hex(u32[5]), "fine_hi", hex(u32[6]),
      "mode", u32[7], "cand_count", u32[8])
print("above", u64[5], "need_f", u64[6], "need_eq", u64[7], "k", k, "n", n)
fine = ws[64:64 + 16384 * 4].cpu().numpy().view(np.uint32)
print("fine total", fine.sum(), "nonzero bins", (fine > 0).sum(), "max bin", fine.max())
keys = (xt.abs().view(torch.int32) + 1).cpu().numpy()
kth = np.sort(keys)[::-1][k - 1]
print("true k-th key", hex(kth))
