"""Batch-sharded data parallelism for the SlimFit step (one process per GPU).

Only the exchange steps the algorithm actually has:
  C1  average of the ACTIVE layers' gradients — frozen layers have no
      gradient buffers, so they contribute no bytes.  Post-accumulate hooks
      gather gradients in the order autograd produces them into ~16 MB
      buckets whose all-reduces start as soon as they fill (overlapped with
      the rest of the backward pass; `begin_backward` / `finish_backward`);
      `allreduce_active_grads` is the non-overlapped form (flat buckets in
      registry order);
  C2  the per-layer distance vector is computed redundantly and identically
      on every rank (replicated AdamW on identical averaged gradients), so
      decisions agree with no collective; `check_distances` allreduces it
      (max - min) as an optional consistency check;
  the loss scalar is averaged for logging and the non-finite check.
The freeze decision is a pure function of the distance vector, so every
rank freezes the same layers without communication.

Layer-owner sharded optimizer (`sharded_optimizer=True`):
layer l is owned by rank l % world.  After backward each active layer's
gradients are reduced to its owner only; the owner runs the fused AdamW +
distance launch (K9) for its layers and keeps their moments (other ranks
hold no moments for them); the updated parameters are broadcast from the
owners, and C2 becomes a real exchange: every rank contributes the
distances of the layers it owns (zeros elsewhere) to one fp64 all-reduce,
which reproduces each owner's value exactly (x + 0 + ... + 0 = x).
Per-rank AdamW / distance work and moment memory drop by the world size;
parameters and decisions stay bit-identical to the replicated path.

Backend: NCCL over NVLink on B200 boxes, gloo in the CPU tests.
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from .model import Batch


class DataParallel:
    def __init__(self, bucket_bytes: int = 16 << 20, group=None, sharded_optimizer: bool = False):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.bucket_elems = max(1, bucket_bytes // 4)
        self.bytes_reduced = 0
        self.sharded_optimizer = bool(sharded_optimizer)
        self.collectives_last_step = 0
        self._hooks, self._pending, self._bucket, self._bucket_n = [], [], [], 0

    # ------------------------------------------------- C1 overlapped with backward
    def begin_backward(self, model, active_ids):
        """Register, for this step's active layers, a post-accumulate hook per
        parameter: gradients are gathered in the order autograd produces them
        (identical on every rank: identical graphs) into buckets of about
        `bucket_bytes`; each full bucket's all-reduce starts at once, so C1
        runs under the rest of the backward pass as one collective per
        bucket, not one per parameter (F = 0.75 activates 100+ tensors).
        A gradient at least as large as a bucket is reduced in place (no
        flatten copy)."""
        self.abort_backward()        # hooks left by a step that raised mid-backward
        if self.world == 1:
            return
        for lid in sorted(active_ids):
            for p in model.registry.by_id(lid).params:
                if p.requires_grad:
                    self._hooks.append(p.register_post_accumulate_grad_hook(self._on_grad))

    def _on_grad(self, p):
        g = p.grad
        self.bytes_reduced += g.numel() * 4
        if g.numel() >= self.bucket_elems:
            work = dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            self._pending.append(([g], None, work))
            return
        self._bucket.append(g)
        self._bucket_n += g.numel()
        if self._bucket_n >= self.bucket_elems:
            self._flush_bucket()

    def _flush_bucket(self):
        if not self._bucket:
            return
        flat = torch.cat([t.reshape(-1) for t in self._bucket])
        work = dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self._pending.append((self._bucket, flat, work))
        self._bucket, self._bucket_n = [], 0

    def finish_backward(self):
        """Start the last partial bucket, wait for the overlapped all-reduces
        (the stream waits, not the host) and turn the sums into averages."""
        self._flush_bucket()
        for grads, flat, work in self._pending:
            work.wait()
            if flat is None:
                grads[0].div_(self.world)
                continue
            flat.div_(self.world)
            off = 0
            for t in grads:
                n = t.numel()
                t.copy_(flat[off:off + n].view_as(t))
                off += n
        self.collectives_last_step = len(self._pending)
        self.abort_backward()

    def abort_backward(self):
        """Drop this step's hooks and pending buckets (after finish_backward,
        or when forward/backward raised in between)."""
        for h in getattr(self, "_hooks", []):
            h.remove()
        self._hooks, self._pending, self._bucket, self._bucket_n = [], [], [], 0

    # ------------------------------------------------------------ ownership
    def owner(self, layer_id: int) -> int:
        return int(layer_id) % self.world

    def owned(self, active_ids):
        return [l for l in sorted(active_ids) if self.owner(l) == self.rank]

    def _reduce_to(self, t: torch.Tensor, dst: int):
        """Sum onto rank `dst` (NCCL reduce; gloo has no CUDA reduce, so it
        all-reduces and the other ranks simply ignore the result)."""
        if dist.get_backend(self.group) == "nccl" or not t.is_cuda:
            dist.reduce(t, dst=dist.get_global_rank(self.group, dst) if self.group else dst, group=self.group)
        else:
            dist.all_reduce(t, group=self.group)

    def _by_owner(self, model, active_ids, what):
        """{owner: [tensors]} of each active layer's `what` ('grad' / 'param'),
        registry order, layers without gradients skipped (as K9 skips them)."""
        out = {}
        for lid in sorted(active_ids):
            ps = [p for p in model.registry.by_id(lid).params if p.grad is not None]
            if ps:
                out.setdefault(self.owner(lid), []).extend(p.grad if what == "grad" else p.data for p in ps)
        return out

    def reduce_grads_to_owners(self, model, active_ids):
        """C1 for the sharded optimizer: one reduce per owner (its layers'
        gradients flattened), averaged on the owner; non-owners drop their
        gradient buffers for those layers afterwards (`release_foreign_grads`)."""
        if self.world == 1:
            return
        for own, grads in sorted(self._by_owner(model, active_ids, "grad").items()):
            flat = torch.cat([g.reshape(-1) for g in grads])
            self._reduce_to(flat, own)
            self.bytes_reduced += flat.numel() * 4
            if own == self.rank:
                flat.div_(self.world)
                off = 0
                for g in grads:
                    n = g.numel()
                    g.copy_(flat[off:off + n].view_as(g))
                    off += n

    def release_foreign_grads(self, model, active_ids):
        for lid in sorted(active_ids):
            if self.owner(lid) != self.rank:
                for p in model.registry.by_id(lid).params:
                    p.grad = None

    def broadcast_owned_params(self, model, active_ids, stepped):
        """Updated parameters from each owner to every rank, one broadcast
        per owner.  `stepped`: {layer_id: [param tensors]} the owners updated
        (identical on every rank: it only depends on which grads existed)."""
        if self.world == 1:
            return
        groups = {}
        for lid in sorted(stepped):
            groups.setdefault(self.owner(lid), []).extend(stepped[lid])
        for own, params in sorted(groups.items()):
            flat = torch.cat([p.data.reshape(-1) for p in params])
            src = dist.get_global_rank(self.group, own) if self.group else own
            dist.broadcast(flat, src=src, group=self.group)
            if own != self.rank:
                off = 0
                for p in params:
                    n = p.numel()
                    p.data.copy_(flat[off:off + n].view_as(p))
                    off += n

    def combine_distances(self, d: torch.Tensor, d_owned: torch.Tensor, active_ids):
        """C2: every rank holds the distances of the layers it owns in
        `d_owned` (zeros elsewhere); one fp64 all-reduce gives every rank all
        of them exactly, copied into `d` at the active ids only."""
        if self.world > 1:
            dist.all_reduce(d_owned, group=self.group)
        idx = torch.as_tensor(sorted(active_ids), dtype=torch.long, device=d.device)
        if idx.numel():
            d.index_copy_(0, idx, d_owned.index_select(0, idx))

    @staticmethod
    def init_from_env(backend: str | None = None, sharded_optimizer: bool = False):
        """torchrun-style env (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_*)."""
        if not dist.is_initialized():
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            if torch.cuda.is_available():
                torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
            dist.init_process_group(backend=backend)
        return DataParallel(sharded_optimizer=sharded_optimizer)

    def shard_batch(self, batch: Batch) -> Batch:
        """Rank r takes rows [r*B/W, (r+1)*B/W) of the global batch."""
        if self.world == 1:
            return batch
        ids, lab = batch.token_ids, batch.labels
        B = len(lab)
        if B % self.world:
            raise ValueError(f"global batch {B} not divisible by world size {self.world}")
        s = B // self.world
        sl = slice(self.rank * s, (self.rank + 1) * s)
        mask = None if batch.attention_mask is None else batch.attention_mask[sl]
        return Batch(ids[sl], lab[sl], mask)

    def allreduce_active_grads(self, model, active_ids):
        """C1: average the active layers' gradients in flat buckets."""
        if self.world == 1:
            return
        grads = []
        for lid in sorted(active_ids):
            for p in model.registry.by_id(lid).params:
                if p.grad is not None:
                    grads.append(p.grad)
        bucket, size = [], 0
        for g in grads:
            bucket.append(g)
            size += g.numel()
            if size >= self.bucket_elems:
                self._reduce_bucket(bucket)
                bucket, size = [], 0
        if bucket:
            self._reduce_bucket(bucket)

    def _reduce_bucket(self, tensors):
        flat = torch.cat([t.reshape(-1) for t in tensors])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        flat.div_(self.world)
        self.bytes_reduced += flat.numel() * 4
        off = 0
        for t in tensors:
            n = t.numel()
            t.copy_(flat[off:off + n].view_as(t))
            off += n

    def average_scalar(self, x: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return x
        y = x.detach().clone().reshape(1).float()
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y / self.world

    def check_distances(self, d: torch.Tensor) -> float:
        """C2 as a consistency check: max over ranks of |d - d_rank0|."""
        if self.world == 1:
            return 0.0
        hi = d.detach().clone()
        lo = d.detach().clone()
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
        return float((hi - lo).abs().max())

    def gather_floats(self, value: float) -> list:
        """Every rank's `value`, in rank order (for per-rank reporting)."""
        if self.world == 1:
            return [value]
        t = torch.tensor([value], dtype=torch.float64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        out = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [float(x.item()) for x in out]

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)

    def max_over_ranks(self, value: float) -> float:
        if self.world == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())
