"""Which torch (aten) ops launch GPU work inside a steady-state BERT-base
SlimFit step, with their CUDA time -- the kernels that are not ours.

    python tools/torch_ops_profile.py [--steps 2]
"""
import argparse
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2305_18513_b200 as sf                          # noqa: E402
from paper_2305_18513_b200.trainer import StepEngine        # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()

L, H, nh, T, V, Cn, B, F = 12, 768, 12, 128, 30522, 2, 128, 0.95
cfg = sf.ModelConfig(blocks=L, hidden=H, heads=nh, max_seq=T, vocab=V, num_classes=Cn)
model = sf.build_model(cfg, seed=0)
n = len(model.registry)
rc = sf.RunConfig(scheduler="ils", freeze_rate=F, epochs=1, batch_size=B, seed=0, lr=5e-5, warmup_frac=0.0,
                  compression=sf.CompressionConfig.all_on())
sched = sf.Scheduler("ils", n, F, 0)
dv = sf.init_distances(n, 0)
eng = StepEngine(model, rc, None)
eng.load_distances(dv)
rng = np.random.default_rng(0)
tok = torch.from_numpy(rng.integers(0, V, size=(8, B, T))).cuda()
lab = torch.from_numpy(rng.integers(0, Cn, size=(8, B))).cuda()


def step(i):
    dec = sched.decide(dv, i)
    eng.step(sf.Batch(tok[i], lab[i]), dec, rc.lr, i)
    eng.fetch_distances(dv, sorted(dec.active_ids))


for i in range(4):
    step(i)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile   # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], record_shapes=True) as prof:
    for i in range(4, 4 + args.steps):
        step(i)
    torch.cuda.synchronize()
tot = collections.Counter()
cnt = collections.Counter()
for e in prof.key_averages(group_by_input_shape=True):
    if e.device_time_total <= 0 or e.key.startswith("sf") or not e.key.startswith("aten::"):
        continue
    k = f"{e.key} {str(e.input_shapes)[:90]}"
    tot[k] += e.device_time_total
    cnt[k] += e.count
print(f"aten ops with device time, per step ({args.steps} steps):")
for k, v in tot.most_common(40):
    print(f"{v / args.steps / 1e3:8.3f} ms  x{cnt[k] / args.steps:5.1f}  {k}")
