"""Catch an occasional slow step: profile 60 steady-state steps with CUPTI,
split the timeline per step (by the per-step D2H read-back), and for the
slowest step print its largest GPU gaps and longest kernels vs a median step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2305_18513_b200 as sf
from paper_2305_18513_b200.trainer import StepEngine

torch.cuda.set_device(0)
cfg = sf.ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522, num_classes=2)
model = sf.build_model(cfg, seed=0)
n = len(model.registry)
rc = sf.RunConfig(scheduler="ils", freeze_rate=0.95, epochs=1, batch_size=128, seed=0, lr=5e-5,
                  warmup_frac=0.0, compression=sf.CompressionConfig.all_on())
sched = sf.Scheduler("ils", n, 0.95, 0)
dv = sf.init_distances(n, 0)
eng = StepEngine(model, rc)
eng.load_distances(dv)
rng = np.random.default_rng(0)
S = 60
tok = torch.from_numpy(rng.integers(0, 30522, size=(S + 10, 128, 128))).cuda()
lab = torch.from_numpy(rng.integers(0, 2, size=(S + 10, 128))).cuda()
marks = []


def step(i):
    dec = sched.decide(dv, i)
    eng.step(sf.Batch(tok[i], lab[i]), dec, 5e-5, i)
    eng.fetch_distances(dv, sorted(dec.active_ids))
    return sorted(dec.active_ids)


for i in range(10):
    step(i)
torch.cuda.synchronize()
acts = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(10, 10 + S):
        acts.append(step(i))
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
# step boundaries: the D2H copy of the distances ends each step
ends = [e.time_range.end for e in ev if "DtoH" in e.name]
ends = ends[1::2] if len(ends) >= 2 * S else ends      # loss + distances per step
bounds = [ev[0].time_range.start] + ends[:S]
walls = np.diff(bounds) / 1e3
print("steps:", len(walls), "median %.1f ms  max %.1f ms at %d" % (np.median(walls), walls.max(), walls.argmax()))
k = int(walls.argmax())
lo, hi = bounds[k], bounds[k + 1]
mine = [e for e in ev if lo <= e.time_range.start < hi]
gaps, cur = [], mine[0].time_range.end
for e in mine[1:]:
    if e.time_range.start > cur:
        gaps.append(((e.time_range.start - cur) / 1e3, e.name[:60]))
    cur = max(cur, e.time_range.end)
print("slow step active:", acts[k] if k < len(acts) else None)
print("largest gaps (ms):", sorted(gaps, reverse=True)[:6])
print("longest kernels (ms):", sorted(((round((e.time_range.end - e.time_range.start) / 1e3, 2), e.name[:60]) for e in mine), reverse=True)[:6])
print("all walls:", np.round(walls, 1).tolist())
