"""Per-layer distance deviations of a fine-tune golden run (tests/golden)
against this repo's run: which entries sit nearest the test's tolerance.

    python tools/finetune_golden_diff.py finetune_vit_b_sgd.npz
"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_18513_b200 as sf

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", sys.argv[1]))
L, H, nh, T, V, Cn, B, iters, seed, pre = g["cfg"].tolist()
optimizer = str(g["optimizer"]) if "optimizer" in g.files else "adamw"
cfg = sf.ModelConfig(blocks=L, hidden=H, heads=nh, max_seq=T, vocab=V, num_classes=Cn, pre_norm=bool(pre))
m = sf.build_model(cfg, seed=seed)
rc = sf.RunConfig(scheduler="ils", freeze_rate=float(g["freeze"]), epochs=1, batch_size=B, seed=seed,
                  lr=float(g["lr"]), warmup_frac=0.0, optimizer=optimizer,
                  compression=sf.CompressionConfig.all_on() if bool(g["codecs"]) else None)
log = sf.fine_tune(m, (g["tokens"], g["labels"]), rc)
ours, ref = log.distance_matrix(), g["d"]
names = m.registry.names()
rel = np.abs(ours - ref) / np.maximum(np.abs(ref), 1e-300)
for it in range(ref.shape[0]):
    j = int(np.argmax(rel[it]))
    print(f"iter {it}: worst layer {j} {names[j]:45s} ours {ours[it, j]:.6e} ref {ref[it, j]:.6e} rel {rel[it, j]:.3e}")
