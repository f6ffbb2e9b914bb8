"""In-step sparse LayerNorm backward vs the synthetic kernel bench: capture a
real frozen-LN x~ from a BERT-base forward, prune it, and time
sf_layernorm_bwd on it; print the per-row kept-count distribution."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2305_18513_b200 as sf
from paper_2305_18513_b200 import compression as Cz
from paper_2305_18513_b200.kernel_bench import L2Flush, time_launches

torch.cuda.set_device(0)
cfg = sf.ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522, num_classes=2)
m = sf.build_model(cfg, seed=0)
ids = torch.from_numpy(np.random.default_rng(0).integers(0, 30522, size=(128, 128))).cuda()
captured = {}
orig = sf.tensor._LayerNorm.forward


def spy(ctx, x, gamma, beta, eps, prune, keep_frac, by_mag, name, res=None, bias=None):
    y = orig(ctx, x, gamma, beta, eps, prune, keep_frac, by_mag, name, res, bias)
    if name.endswith("encoder.layer.5.output.LayerNorm"):
        captured["sv"] = ctx.sv
    return y


sf.tensor._LayerNorm.forward = staticmethod(spy)
m.freeze_set(range(len(m.registry)))
with sf.tensor.record(sf.CompressionConfig.all_on()):
    m.forward(sf.Batch(ids, None))
sv_xt, sv_r = captured["sv"]
sp = sv_xt.value.wait().sparse
rp = sp.row_ptr.cpu().numpy()
cnt = np.diff(rp)
print("kept per row: mean %.1f  min %d  max %d  p99 %d" % (cnt.mean(), cnt.min(), cnt.max(), np.percentile(cnt, 99)))
rows, H = 128 * 128, 768
N = sf._native
lib = N.load()
g = torch.randn(rows, H, device="cuda")
dx = torch.empty_like(g)
gam = torch.ones(H, device="cuda")
ws = torch.empty(lib.sf_layernorm_bwd_workspace_bytes(rows, H), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
flush = L2Flush()
f = lambda: lib.sf_layernorm_bwd(g.data_ptr(), gam.data_ptr(), None, sp.values.data_ptr(), sp.indices.data_ptr(),
                                 sp.values.numel(), sp.row_ptr.data_ptr(), sv_r.value.data_ptr(), dx.data_ptr(),
                                 None, None, rows, H, ws.data_ptr(), st)
print("real x~  : %.1f us" % (time_launches(f, 20, flush=flush) * 1e3))
# synthetic: standardized rows
xt = torch.randn(rows, H, device="cuda")
xt = (xt - xt.mean(-1, keepdim=True)) / xt.std(-1, keepdim=True, unbiased=False)
sp2 = Cz.prune_topk(xt, 0.1, True, row_pointers=True)
f2 = lambda: lib.sf_layernorm_bwd(g.data_ptr(), gam.data_ptr(), None, sp2.values.data_ptr(), sp2.indices.data_ptr(),
                                  sp2.values.numel(), sp2.row_ptr.data_ptr(), sv_r.value.data_ptr(), dx.data_ptr(),
                                  None, None, rows, H, ws.data_ptr(), st)
print("synthetic: %.1f us" % (time_launches(f2, 20, flush=flush) * 1e3))
