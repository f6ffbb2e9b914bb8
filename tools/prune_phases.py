"""Phase timeline of one sf_prune_topk_rows call at BERT-base x~ size
(%globaltimer stamps CTA 0 writes into the workspace state)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_18513_b200 import _native as N

lib = N.load()
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(16384, 768, generator=g, device="cuda")
x = (x - x.mean(-1, keepdim=True)) / x.std(-1, keepdim=True)
n, H = x.numel(), 768
k = -(-n // 10)
vals = torch.empty(k, device="cuda")
idx = torch.empty(k, dtype=torch.int32, device="cuda")
rp = torch.empty(n // H + 1, dtype=torch.int32, device="cuda")
ws = torch.empty(lib.sf_prune_workspace_bytes(n), dtype=torch.uint8, device="cuda")
# PruneState: bar u32, inf_count u32, staged u64, blist_n u32, blist_ovf u32, fine[2048] u32,
# rhist[4][256] u32, t[10] u64
off_t = 4 + 4 + 8 + 4 + 4 + 2048 * 4 + 4 * 256 * 4
a_ = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(200):                            # clocks at boost
    a_ @ a_
torch.cuda.synchronize()
names = ["start", "hist", "sample", "select+stream", "barrier1", "gather", "barrier2", "rank", "barrier3", "emit"]
for it in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.sf_prune_topk_rows(x.data_ptr(), n, k, 1, vals.data_ptr(), idx.data_ptr(), H, rp.data_ptr(),
                                ws.data_ptr(), None)
    e1.record()
    torch.cuda.synchronize()
    t = ws[off_t + 8:off_t + 88].view(torch.int64).cpu().tolist()
    nc = int(ws[4:8].view(torch.int32).item())
    order = [0, 2, 1, 3, 4, 5, 6, 7, 8, 9]
    parts = [(names[i], (t[i] - t[order[j - 1]]) / 1e3 if j else 0.0) for j, i in enumerate(order)]
    print(f"call {it}: {e0.elapsed_time(e1) * 1e3:.1f} us (events), F keys {nc}; "
          + ", ".join(f"{a} {b:.1f}" for a, b in parts) + f"; start->end {(t[9] - t[0]) / 1e3:.1f} us")

# hinted: alternate two batches of the same site; raw stamps relative to the start
x2 = torch.randn(16384, 768, generator=g, device="cuda")
x2 = (x2 - x2.mean(-1, keepdim=True)) / x2.std(-1, keepdim=True)
hint = torch.zeros(lib.sf_prune_hint_bytes() // 4, dtype=torch.int32, device="cuda")
for it in range(6):
    src = x if it % 2 == 0 else x2
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.sf_prune_topk_hint(src.data_ptr(), n, k, 1, vals.data_ptr(), idx.data_ptr(), H, rp.data_ptr(),
                                hint.data_ptr(), ws.data_ptr(), None)
    e1.record()
    torch.cuda.synchronize()
    hs = hint.view(torch.uint8)[16:]
    t = hs[off_t + 8:off_t + 88].view(torch.int64).cpu().tolist()
    bl = hs[16:24].view(torch.int32).cpu().tolist()
    h = hint[:4].cpu().tolist()
    rel = [round((v - t[0]) / 1e3, 1) if v else None for v in t]
    print(f"hinted {it}: rc {rc} {e0.elapsed_time(e1) * 1e3:.1f} us; hint {h}; blist n/ovf {bl}; stamps {rel}")
