"""Time and accuracy of the step's GEMM shapes (BERT-base B=128 T=128) in
each sf_gemm_f32 mode against torch's strict-fp32 matmul; error is the max
|C - C64| / max|C64| against an fp64 product of the same fp32 inputs."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_18513_b200 import gemm

torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
M = 128 * 128
B = 128 * 12


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


g = torch.Generator(device=dev).manual_seed(0)
cases = []
for K, N in [(768, 768), (768, 3072), (3072, 768)]:
    x = torch.randn(M, K, device=dev, generator=g)
    w = torch.randn(K, N, device=dev, generator=g) * 0.02
    gy = torch.randn(M, N, device=dev, generator=g)
    cases += [(f"fwd {M}x{K}x{N}", x, w), (f"dgrad {M}x{N}x{K}", gy, w.t()), (f"wgrad {K}x{M}x{N}", x.t(), gy)]
q = torch.randn(B, 128, 64, device=dev, generator=g)
k = torch.randn(B, 128, 64, device=dev, generator=g)
p = torch.softmax(torch.randn(B, 128, 128, device=dev, generator=g), -1)
cases += [("scores", q, k.transpose(-1, -2)), ("context", p, q), ("ctx-dgrad", q, k.transpose(-1, -2)),
          ("p^T g", p.transpose(-1, -2), q)]
print("lt version", gemm.N.load().sf_gemm_lt_version(), "bf16x9", gemm.available("bf16x9"))
for name, a, b in cases:
    ref = torch.matmul(a.double(), b.double())
    scale = ref.abs().max().item()
    flops = 2 * a.shape[-2] * a.shape[-1] * b.shape[-1] * (a.shape[0] if a.dim() == 3 else 1)
    row = [f"{name:22s}"]
    tt = t(lambda: torch.matmul(a, b))
    e = (torch.matmul(a, b).double() - ref).abs().max().item() / scale
    row.append(f"torch {tt:8.1f}us {flops / tt / 1e6:6.1f}TF err {e:.2e}")
    for mode in ("fp32", "bf16x9", "tf32"):
        gemm.set_mode(mode)
        try:
            tt = t(lambda: gemm.mm(a, b))
            e = (gemm.mm(a, b).double() - ref).abs().max().item() / scale
            row.append(f"{mode} {tt:8.1f}us {flops / tt / 1e6:6.1f}TF err {e:.2e}")
        except Exception as exc:
            row.append(f"{mode} FAILED {exc}")
    print(" | ".join(row), flush=True)
