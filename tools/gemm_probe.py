"""Which kernels do the step's fp32 GEMM call forms launch, and how long do
they take?  (FFN1 / FFN2 / QKV shapes at BERT-base B=128.)"""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
M = 128 * 128
shapes = [(768, 3072), (3072, 768), (768, 768)]


def t(fn, it=10):
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


for K, N in shapes:
    x = torch.randn(M, K, device=dev)
    w = torch.randn(K, N, device=dev)
    wt = w.t().contiguous()
    bias = torch.randn(N, device=dev)
    out = torch.empty(M, N, device=dev)
    print(f"M={M} K={K} N={N}",
          f"addmm {t(lambda: torch.addmm(bias, x, w)):.1f}us",
          f"mm {t(lambda: x @ w):.1f}us",
          f"mm_out {t(lambda: torch.mm(x, w, out=out)):.1f}us",
          f"linear(wT) {t(lambda: torch.nn.functional.linear(x, wt, bias)):.1f}us",
          f"mm(wT.t()) {t(lambda: x @ wt.t()):.1f}us",
          f"gflops(mm) {2*M*K*N / t(lambda: x @ w) / 1e3:.0f}")
