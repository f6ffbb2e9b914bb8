"""Two ranks (gloo, both on cuda:0) running real SlimFit steps: the
layer-owner sharded optimizer must leave parameters,
distances and freeze decisions bit-identical to the replicated optimizer,
and every rank must agree."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

STEPS = 5


def _worker(rank, world, port, sharded, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2305_18513_b200 as sf
        from paper_2305_18513_b200.distributed import DataParallel
        from paper_2305_18513_b200.trainer import StepEngine
        dp = DataParallel(sharded_optimizer=sharded)
        cfg = sf.ModelConfig(blocks=2, hidden=64, heads=4, max_seq=32, vocab=100, num_classes=3)
        m = sf.build_model(cfg, seed=7)
        n = len(m.registry)
        rc = sf.RunConfig(scheduler="ils", freeze_rate=0.6, epochs=1, batch_size=8, seed=0, lr=1e-3,
                          warmup_frac=0.0, compression=sf.CompressionConfig.all_on())
        sched = sf.Scheduler("ils", n, 0.6, 0)
        dv = sf.init_distances(n, 0)
        eng = StepEngine(m, rc, dp)
        eng.load_distances(dv)
        rng = np.random.default_rng(3)
        frozen = []
        for it in range(STEPS):
            ids = rng.integers(0, 100, size=(8, 32))
            lab = rng.integers(0, 3, size=8)
            b = dp.shard_batch(sf.Batch(ids, lab))
            dec = sched.decide(dv, it)
            eng.step(b, dec, rc.lr, it)
            eng.fetch_distances(dv, sorted(dec.active_ids))
            frozen.append(sorted(dec.frozen_ids))
        torch.cuda.synchronize()
        params = [p.detach().cpu().numpy() for p in m.parameters()]
        q.put((rank, params, dv.d.copy(), frozen, len(eng.opt.moments)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(sharded):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sharded, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    return res


def test_sharded_optimizer_is_bit_identical_to_replicated():
    rep = _run(False)
    sh = _run(True)
    for res in (rep, sh):                              # ranks agree
        for a, b in zip(res[0][1], res[1][1]):
            assert np.array_equal(a, b)
        assert np.array_equal(res[0][2], res[1][2]) and res[0][3] == res[1][3]
    for a, b in zip(rep[0][1], sh[0][1]):              # sharded == replicated
        assert np.array_equal(a, b)
    assert np.array_equal(rep[0][2], sh[0][2])
    assert rep[0][3] == sh[0][3]
    # moments live only on the owner: the two ranks split them
    assert sh[0][4] + sh[1][4] == rep[0][4]
