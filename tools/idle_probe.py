"""GPU busy vs idle inside steady-state steps (torch.profiler / CUPTI):
sum of kernel + memcpy durations (merged intervals) against wall time."""
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
tok = torch.from_numpy(rng.integers(0, 30522, size=(12, 128, 128))).cuda()
lab = torch.from_numpy(rng.integers(0, 2, size=(12, 128))).cuda()


def step(i):
    dec = sched.decide(dv, i)
    eng.step(sf.Batch(tok[i], lab[i]), dec, 5e-5, i)
    eng.fetch_distances(dv, sorted(dec.active_ids))


for i in range(6):
    step(i)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(6, 10):
        step(i)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
wall = iv[-1][1] - iv[0][0]
print(f"4 steps: wall {wall / 1e3:.1f} ms, GPU busy {busy / 1e3:.1f} ms ({100 * busy / wall:.1f}%), idle {(wall - busy) / 1e3:.1f} ms")
# biggest gaps
gaps = []
prev_e = iv[0][1]
names = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev))
for (s, e, nm), (s0, e0, nm0) in zip(names[1:], names[:-1]):
    pass
cur = names[0][1]
for s, e, nm in names[1:]:
    if s > cur:
        gaps.append((s - cur, nm[:70]))
    cur = max(cur, e)
gaps.sort(reverse=True)
print("largest gaps (us) before:", [(round(g), nm) for g, nm in gaps[:12]])
print("gap total by size: >100us %.1f ms, 10-100us %.1f ms, <10us %.1f ms" % (
    sum(g for g, _ in gaps if g > 100) / 1e3, sum(g for g, _ in gaps if 10 < g <= 100) / 1e3,
    sum(g for g, _ in gaps if g <= 10) / 1e3))
# host-side synchronisations inside the profiled steps and their enclosing ops
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
syncs = [e for e in cpu if ("Synchronize" in e.name or e.name in ("cudaMemcpy", "cudaStreamWaitEvent_sync"))]
print("host sync calls:", len(syncs))
for e in sorted(syncs, key=lambda e: -(e.time_range.end - e.time_range.start))[:8]:
    par = e.cpu_parent
    chain = []
    while par is not None and len(chain) < 4:
        chain.append(par.name[:40])
        par = par.cpu_parent
    print(f"  {e.name} {(e.time_range.end - e.time_range.start) / 1e3:.2f} ms  <- {chain}")
big = sorted(cpu, key=lambda e: -(e.time_range.end - e.time_range.start))
print("longest aten ops:", [(e.name[:40], round((e.time_range.end - e.time_range.start) / 1e3, 2)) for e in big if e.name.startswith("aten::")][:10])
