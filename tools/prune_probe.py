"""Time sf_prune_topk_rows at BERT-base x~ size (12.6M, k=10%): L2 flushed
between calls and back to back (L2-warm), after a clock warm-up; used with
ncu for the per-line split."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_18513_b200 as sf
from paper_2305_18513_b200.kernel_bench import L2Flush, time_launches

g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(16384, 768, generator=g, device="cuda")
x = (x - x.mean(-1, keepdim=True)) / x.std(-1, keepdim=True)
iters = int(os.environ.get("ITERS", "20"))
flush = L2Flush()
if iters > 1:                                   # ~0.5 s of back-to-back work: clocks at boost
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(200):
        a @ a
    torch.cuda.synchronize()
for warm in (False, True):
    ms = time_launches(lambda: sf.prune_topk(x, 0.1, row_pointers=True), iters=iters,
                       flush=None if warm else flush)
    print(f"prune ({'L2-warm' if warm else 'L2 flushed'}): {ms * 1e3:.1f} us")
