"""Run the fused attention kernels once at BERT-base B=128 shapes (for ncu)
and time them with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_18513_b200 as sf

N = sf._native
B, T, h, dh = 128, 128, 12, 64
H = h * dh
g = torch.Generator(device="cuda").manual_seed(0)
y3 = torch.randn(3, B * T, H, generator=g, device="cuda")
bs = [torch.randn(H, generator=g, device="cuda") * 0.1 for _ in range(3)]
ctx = torch.empty(B * T, H, device="cuda")
qc = torch.empty(B, h, T, dh, dtype=torch.int8, device="cuda")
kc, vc = torch.empty_like(qc), torch.empty_like(qc)
pc = torch.empty(B, h, T, T, dtype=torch.int8, device="cuda")
gr = torch.randn(B * T, H, generator=g, device="cuda")
gcat = torch.empty(B * T, 3 * H, device="cuda")
s = torch.cuda.current_stream().cuda_stream
fwd = lambda: N.call("sf_attention_fwd", y3.data_ptr(), bs[0].data_ptr(), bs[1].data_ptr(), bs[2].data_ptr(),
                     B, T, h, dh, 0.125, 4, ctx.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                     pc.data_ptr(), s)
bwd = lambda: N.call("sf_attention_bwd", gr.data_ptr(), qc.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                     pc.data_ptr(), B, T, h, dh, 0.125, 4, gcat.data_ptr(), s)
iters = int(os.environ.get("ITERS", "20"))
for name, f in (("fwd", fwd), ("bwd", bwd)):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        f()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) / iters * 1e3
    fl = (4 if name == "fwd" else 8) * B * h * T * T * dh
    print(f"{name}: {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s")
