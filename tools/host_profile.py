"""Is the step host-bound?  Times, per step, the host wall time spent
enqueueing forward+backward (no sync inside), the wait for the device at the
loss check, and the optimizer/fetch tail, next to the device step time.

    python tools/host_profile.py [--steps 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2305_18513_b200 as sf
from paper_2305_18513_b200.trainer import StepEngine
from paper_2305_18513_b200 import tensor as T

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--batch", type=int, default=128)
args = ap.parse_args()
torch.cuda.set_device(0)
cfg = sf.ModelConfig(blocks=12, hidden=768, heads=12, max_seq=128, vocab=30522, num_classes=2)
model = sf.build_model(cfg, seed=0)
n = len(model.registry)
rc = sf.RunConfig(scheduler="ils", freeze_rate=0.95, epochs=1, batch_size=args.batch, seed=0, lr=5e-5,
                  warmup_frac=0.0, compression=sf.CompressionConfig.all_on())
sched = sf.Scheduler("ils", n, 0.95, 0)
dv = sf.init_distances(n, 0)
eng = StepEngine(model, rc)
eng.load_distances(dv)
rng = np.random.default_rng(0)
tok = torch.from_numpy(rng.integers(0, 30522, size=(args.steps + 3, args.batch, 128))).cuda()
lab = torch.from_numpy(rng.integers(0, 2, size=(args.steps + 3, args.batch))).cuda()

rows = []
tok = torch.from_numpy(rng.integers(0, 30522, size=(args.steps + 3, args.batch, 128))).cuda()
lab = torch.from_numpy(rng.integers(0, 2, size=(args.steps + 3, args.batch))).cuda()
for i in range(args.steps + 3):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    dec = sched.decide(dv, i)
    loss, logits, labels, tape = eng.forward_backward(sf.Batch(tok[i], lab[i]), dec.frozen_ids)
    t1 = time.perf_counter()
    active = sorted(dec.active_ids)
    eng.opt.step(model, 5e-5, active, eng.d_dev)
    t2 = time.perf_counter()
    eng.fetch_distances(dv, active)
    ev1.record()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    if i >= 3:
        names = [model.registry.by_id(a).name.replace("encoder.layer.", "L") for a in active]
        rows.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), ev0.elapsed_time(ev1)))
        print(f"step {i}: enqueue {rows[-1][0]:.1f} opt {rows[-1][1]:.1f} wait {rows[-1][2]:.1f} "
              f"device {rows[-1][3]:.1f}  active {names}", flush=True)
r = np.array(rows)
print("per step (ms): host enqueue fwd+bwd %.1f | optimizer enqueue %.1f | wait %.1f | device %.1f"
      % tuple(r.mean(0)))
print("launches per step (own):", sf._native.launch_count / (args.steps + 3))
