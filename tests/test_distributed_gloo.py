"""Data-parallel host logic on CPU with world_size 2 over gloo: batch
sharding, C1 (only active layers' gradients are averaged, in buckets), the
loss average, and the C2 distance consistency check."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _Entry:
    def __init__(self, lid, params):
        self.layer_id = lid
        self.params = params


class _Reg:
    def __init__(self, entries):
        self.entries = entries

    def by_id(self, lid):
        return self.entries[lid]

    def __len__(self):
        return len(self.entries)


class _Model:
    def __init__(self, shapes, rank):
        g = torch.Generator().manual_seed(100 + rank)
        ents = []
        for lid, ss in enumerate(shapes):
            ps = []
            for s in ss:
                p = torch.zeros(s)
                p.grad = torch.randn(s, generator=g)
                ps.append(p)
            ents.append(_Entry(lid, ps))
        self.registry = _Reg(ents)


SHAPES = [[(50, 8)], [(8,), (8,)], [(8, 32), (32,)], [(32, 8), (8,)], [(3,)]]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18513_b200.distributed import DataParallel
        from paper_2305_18513_b200.model import Batch
        from paper_2305_18513_b200.scheduler import init_distances, select_frozen
        dp = DataParallel(bucket_bytes=200)     # tiny buckets: several collectives
        m = _Model(SHAPES, rank)
        before = {l: [p.grad.clone() for p in e.params] for l, e in enumerate(m.registry.entries)}
        active = [0, 2, 4]
        dp.allreduce_active_grads(m, active)
        out = {l: [p.grad.clone() for p in e.params] for l, e in enumerate(m.registry.entries)}
        ids = np.arange(8 * 4).reshape(8, 4)
        b = dp.shard_batch(Batch(ids, np.arange(8)))
        loss = dp.average_scalar(torch.tensor(float(rank + 1)))
        dv = init_distances(22, 3)
        dec = select_frozen(dv, 0.5)
        chk = dp.check_distances(torch.from_numpy(dv.d))
        # plain numpy across the queue (torch tensors would travel as shared-memory
        # handles that die with this process)
        before = {l: [t.numpy() for t in v] for l, v in before.items()}
        out = {l: [t.numpy() for t in v] for l, v in out.items()}
        q.put((rank, before, out, b.token_ids.tolist(), b.labels.tolist(), float(loss),
               sorted(dec.frozen_ids), chk, dp.bytes_reduced))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    return res


def test_active_grads_averaged_frozen_untouched(results):
    b0, b1 = results[0][1], results[1][1]
    for rank in (0, 1):
        out = results[rank][2]
        for lid in range(len(SHAPES)):
            for j in range(len(SHAPES[lid])):
                if lid in (0, 2, 4):
                    want = (b0[lid][j] + b1[lid][j]) / 2
                    assert np.allclose(out[lid][j], want, atol=1e-6)
                else:
                    assert np.array_equal(out[lid][j], results[rank][1][lid][j])


def test_only_active_bytes_cross_the_wire(results):
    active_elems = 50 * 8 + (8 * 32 + 32) + 3
    assert results[0][8] == active_elems * 4


def test_batch_sharding(results):
    assert results[0][3] == np.arange(16).reshape(4, 4).tolist()
    assert results[1][3] == np.arange(16, 32).reshape(4, 4).tolist()
    assert results[0][4] == [0, 1, 2, 3] and results[1][4] == [4, 5, 6, 7]


def test_loss_average_and_decisions_agree(results):
    assert results[0][5] == results[1][5] == 1.5
    assert results[0][6] == results[1][6]
    assert results[0][7] == 0.0


# ---------------------------------------------------------------- sharded optimizer (§8(f)4)

def _sharded_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18513_b200.distributed import DataParallel
        dp = DataParallel(sharded_optimizer=True)
        m = _Model(SHAPES, rank)
        for e in m.registry.entries:
            for j, p in enumerate(e.params):
                p.data.fill_(float(10 * e.layer_id + j))
        before = {l: [p.grad.clone().numpy() for p in e.params] for l, e in enumerate(m.registry.entries)}
        active = [0, 1, 2, 4]
        dp.reduce_grads_to_owners(m, active)
        owned_grads = {l: [p.grad.clone().numpy() for p in m.registry.by_id(l).params]
                       for l in dp.owned(active)}
        dp.release_foreign_grads(m, active)
        released = [l for l in active if all(p.grad is None for p in m.registry.by_id(l).params)]
        # owners "update" their layers; everyone receives the result
        stepped = {l: list(m.registry.by_id(l).params) for l in active}
        for l in dp.owned(active):
            for p in m.registry.by_id(l).params:
                p.data.add_(1000.0 * (rank + 1))
        dp.broadcast_owned_params(m, active, stepped)
        params = {l: [p.data.clone().numpy() for p in e.params] for l, e in enumerate(m.registry.entries)}
        d = torch.full((5,), -1.0, dtype=torch.float64)
        d_owned = torch.zeros(5, dtype=torch.float64)
        for l in dp.owned(active):
            d_owned[l] = 0.1 * (l + 1) + 1e-17 * l
        dp.combine_distances(d, d_owned, active)
        q.put((rank, before, owned_grads, released, params, d.numpy(), dp.owned(active)))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    return res


def test_sharded_owners_get_averaged_grads_others_release(sharded):
    b0, b1 = sharded[0][1], sharded[1][1]
    assert sharded[0][6] == [0, 2, 4] and sharded[1][6] == [1]
    for rank in (0, 1):
        for lid, gs in sharded[rank][2].items():
            for j, g in enumerate(gs):
                assert np.allclose(g, (b0[lid][j] + b1[lid][j]) / 2, atol=1e-6)
        assert sharded[rank][3] == [l for l in (0, 1, 2, 4) if l % 2 != rank]


def test_sharded_params_broadcast_from_owners(sharded):
    p0, p1 = sharded[0][4], sharded[1][4]
    for lid in range(len(SHAPES)):
        for j in range(len(SHAPES[lid])):
            assert np.array_equal(p0[lid][j], p1[lid][j])
            base = float(10 * lid + j)
            want = base + (1000.0 * (lid % 2 + 1) if lid in (0, 1, 2, 4) else 0.0)
            assert np.all(p0[lid][j] == want)


def test_sharded_distance_exchange_is_exact(sharded):
    for rank in (0, 1):
        d = sharded[rank][5]
        for l in (0, 1, 2, 4):
            assert d[l] == 0.1 * (l + 1) + 1e-17 * l
        assert d[3] == -1.0


# ---------------------------------------------------------------- C1 overlapped with backward

def _overlap_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_18513_b200.distributed import DataParallel
        dp = DataParallel()
        g = torch.Generator().manual_seed(7)
        ents = []
        for lid, ss in enumerate(SHAPES):
            ents.append(_Entry(lid, [torch.randn(s, generator=g).requires_grad_(lid in (0, 2, 4)) for s in ss]))
        m = _Model.__new__(_Model)
        m.registry = _Reg(ents)
        xs = [[torch.full(p.shape, float(rank + 1 + lid)) for p in e.params] for lid, e in enumerate(ents)]
        dp.begin_backward(m, [0, 2, 4])
        loss = sum((p * x).sum() for e, xx in zip(ents, xs) for p, x in zip(e.params, xx) if p.requires_grad)
        loss.backward()
        dp.finish_backward()
        q.put((rank, {l: [p.grad.numpy().copy() if p.grad is not None else None for p in e.params]
                      for l, e in enumerate(ents)}, dp.bytes_reduced, len(dp._hooks)))
    finally:
        dist.destroy_process_group()


def test_overlapped_c1_averages_active_grads():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
    for rank in (0, 1):
        grads = res[rank][1]
        for lid in range(len(SHAPES)):
            for j, gr in enumerate(grads[lid]):
                if lid in (0, 2, 4):
                    # d/dp of sum(p * (rank + 1 + lid)) averaged over ranks 0, 1
                    assert np.allclose(gr, (1 + lid + 2 + lid) / 2)
                else:
                    assert gr is None
        assert res[rank][3] == 0                       # hooks removed after the step
    active_elems = 50 * 8 + (8 * 32 + 32) + 3
    assert res[0][2] == active_elems * 4
