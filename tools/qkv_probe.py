"""Probe: q/k/v projections as one broadcast-batched emulated GEMM vs three;
the dgrad sum g_q Wq^T + g_k Wk^T + g_v Wv^T with beta-accumulation vs three
GEMMs and two adds (BERT-base B=128 shapes)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_18513_b200 import gemm


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / it * 1e3


M, H = 16384, 768
x = torch.randn(M, H, device="cuda")
W = torch.randn(3, H, H, device="cuda") * 0.02
G = torch.randn(3, M, H, device="cuda")
gemm.set_mode("bf16x9")
sep = lambda: [gemm.mm(x, W[i]) for i in range(3)]
bat = lambda: gemm.mm(x.expand(3, M, H), W, mode="bf16x9")
ref = torch.stack([x.double() @ W[i].double() for i in range(3)])
e = (bat().double() - ref).abs().max().item() / ref.abs().max().item()
print(f"fwd: 3 separate {t(sep):.0f}us | batched(stride-0 x) {t(bat):.0f}us err {e:.2e}")
def dsep():
    d = gemm.mm(G[0], W[0].t())
    d = d + gemm.mm(G[1], W[1].t())
    return d + gemm.mm(G[2], W[2].t())
out = torch.empty(M, H, device="cuda")
def dacc():
    gemm.mm(G[0], W[0].t(), out=out)
    gemm.mm(G[1], W[1].t(), out=out, beta=1.0)
    gemm.mm(G[2], W[2].t(), out=out, beta=1.0)
    return out
Gcat = G.permute(1, 0, 2).reshape(M, 3 * H).contiguous()
Wt = W.transpose(1, 2).reshape(3 * H, H).contiguous()
dcat = lambda: gemm.mm(Gcat, Wt)
ref = sum(G[i].double() @ W[i].double().t() for i in range(3))
for name, f in [("3 GEMMs + 2 adds", dsep), ("beta-accumulate", dacc), ("one K=2304 GEMM (concat)", dcat)]:
    e = (f().double() - ref).abs().max().item() / ref.abs().max().item()
    print(f"dgrad {name}: {t(f):.0f}us err {e:.2e}")
