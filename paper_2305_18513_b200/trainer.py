"""Fine-tuning loop — the drop-in for trainer.py (/root/reference/pkg/src/slimfit).

Iteration protocol (trainer.py:172-215): decide -> freeze -> recorded
forward/backward -> non-finite check -> optimizer step on the active layers
-> refresh the active layers' distances -> logs.  On the device the
optimizer step and the distance refresh are ONE launch (K9): the f32 AdamW
update keeps the pre-update value in registers and feeds the
numpy-pairwise-exact distance reduction, so the reference's full
`clone_layer_data` copy (trainer.py:194-195) disappears.  Per iteration the
host reads back one loss scalar and the n-entry distance vector.

Data parallel (one process per GPU, torch.distributed NCCL): each rank takes
an equal slice of every global batch; after backward the active layers'
gradients — and only those — are averaged in flat buckets (C1); the
distance vector is computed redundantly and identically on every rank
(replicated AdamW), so decisions agree without a collective; `check_sync`
allreduces it (C2) as a consistency check.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import gemm as G
from . import tensor as T
from .errors import ConfigError, TrainingDiverged
from .model import Batch, Model
from .scheduler import DistancePlan, DistanceVector, Scheduler, init_distances
from .tensor import CompressionConfig


@dataclass
class OptimizerState:
    """AdamW or SGD with per-layer step counters; frozen layers pause
    (no moments, no decay, no step advance) — trainer.py:27-76."""

    kind: str = "adamw"
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
    global_step_bias: bool = False
    moments: dict = field(default_factory=dict)      # id(param) -> (m, v) device tensors
    layer_steps: dict = field(default_factory=dict)  # layer_id -> steps taken
    global_steps: int = 0

    def __post_init__(self):
        if self.kind not in ("sgd", "adamw"):
            raise ConfigError(f"unknown optimizer kind {self.kind!r}")
        self._plan = None
        self._plan_key = None

    def _plan_for(self, model: Model) -> DistancePlan:
        key = id(model)
        if self._plan_key != key:
            self._plan = DistancePlan([p.numel() for p in model.parameters()], model.device)
            self._slot = {id(p): j for j, p in enumerate(model.parameters())}
            self._plan_key = key
        return self._plan

    def _consts(self, t: int, lr: float):
        f = np.float32
        return dict(b1=f(self.beta1), ob1=f(1 - self.beta1), b2=f(self.beta2),
                    ob2=f(1 - self.beta2), bc1=f(1 - self.beta1 ** t), bc2=f(1 - self.beta2 ** t),
                    eps=f(self.eps), wd=f(self.weight_decay), lr=f(lr))

    def step(self, model: Model, lr: float, active_ids, d_out: torch.Tensor | None = None,
             guard: torch.Tensor | None = None):
        """One update of the active layers (trainer.py:50-76) fused with the
        refresh of their distances (trainer.py:194-200, scheduler.py:92-120)
        in one K9 launch, for both optimizers: every active layer's entry of
        d_out (float64 device vector) is rewritten -- a layer none of whose
        parameters has a gradient did not move and gets 0.0, a parameter
        without a gradient counts toward its layer's element count.
        guard: optional device float (the step's loss); if it is not finite
        the launch changes nothing (the caller raises TrainingDiverged and
        rolls the step counters back with `restore_counters`)."""
        self.global_steps += 1
        plan = self._plan_for(model)
        rows, layers = [], []
        for lid in active_ids:
            entry = model.registry.by_id(lid)
            j0, count = len(rows), sum(p.numel() for p in entry.params)
            if any(p.grad is not None for p in entry.params):
                self.layer_steps[lid] = self.layer_steps.get(lid, 0) + 1
                t = self.global_steps if self.global_step_bias else self.layer_steps[lid]
                consts = self._consts(t, lr) if self.kind == "adamw" else None
                for p in entry.params:
                    if p.grad is None:
                        continue
                    g = p.grad if p.grad.is_contiguous() else p.grad.contiguous()
                    row = {"slot": self._slot[id(p)], "A": p.data_ptr(), "B": g.data_ptr(), "_keep": g}
                    if consts is not None:
                        mv = self.moments.get(id(p))
                        if mv is None:
                            mv = (torch.zeros_like(p, memory_format=torch.contiguous_format),
                                  torch.zeros_like(p, memory_format=torch.contiguous_format))
                            self.moments[id(p)] = mv
                        row.update(M=mv[0].data_ptr(), V=mv[1].data_ptr(), consts=consts)
                    else:
                        row["lr"] = np.float32(lr)
                    rows.append(row)
            layers.append((j0, len(rows) - j0, int(lid), count))
        if not layers:
            return
        if d_out is None:
            d_out = torch.zeros(len(model.registry), dtype=torch.float64, device=model.device)
        plan.run(rows, layers, d_out, N.UPDATE_ADAMW if self.kind == "adamw" else N.UPDATE_SGD, guard=guard)
        # K9 writes the parameters through raw pointers: re-split their GEMM planes
        G.weight_planes_changed([p for lid in active_ids for p in model.registry.by_id(lid).params])

    def preallocate(self, params) -> None:
        """Allocate the AdamW moments of `params` now (zeros, exactly what the
        first activation would allocate): the optimizer state then never
        allocates inside a step.  SGD keeps no state."""
        if self.kind != "adamw":
            return
        for p in params:
            if id(p) not in self.moments:
                self.moments[id(p)] = (torch.zeros_like(p, memory_format=torch.contiguous_format),
                                       torch.zeros_like(p, memory_format=torch.contiguous_format))

    def save_counters(self):
        """Step counters and the set of allocated moments, for `restore_counters`."""
        return dict(self.layer_steps), self.global_steps, set(self.moments)

    def restore_counters(self, saved):
        """Undo the bookkeeping of a step whose launch the loss guard
        cancelled: the reference raises TrainingDiverged before its
        optimizer touches any state (trainer.py:182-190)."""
        steps, gsteps, keys = saved
        self.layer_steps, self.global_steps = steps, gsteps
        for k in [k for k in self.moments if k not in keys]:
            del self.moments[k]


def linear_schedule(base_lr: float, step: int, total_steps: int, warmup_frac: float) -> float:
    """Linear warmup to base_lr, then linear decay to 0 (trainer.py:79-87)."""
    warmup = int(warmup_frac * total_steps)
    if warmup > 0 and step < warmup:
        return base_lr * (step + 1) / warmup
    if total_steps <= warmup:
        return base_lr
    return base_lr * max(0.0, 1.0 - (step - warmup) / max(1, total_steps - warmup))


@dataclass
class RunConfig:
    scheduler: str = "ils"              # ils | random | progressive | none
    freeze_rate: float = 0.0
    epochs: int = 3
    batch_size: int = 32
    seed: int = 0
    lr: float = 1e-3
    warmup_frac: float = 0.1
    optimizer: str = "adamw"
    weight_decay: float = 0.01
    global_step_bias: bool = False
    compression: CompressionConfig | None = None
    pinned_active: tuple = ()
    track_memory: bool = True
    # allocate every AdamW moment when the engine is built instead of at a
    # layer's first activation (the reference's lazy allocation; same values)
    preallocate_state: bool = False

    def validate(self):
        if not 0.0 <= self.freeze_rate < 1.0:
            raise ConfigError(f"freeze rate must lie in [0, 1), got {self.freeze_rate}")
        if self.epochs < 1 or self.batch_size < 1:
            raise ConfigError("epochs and batch size must be >= 1")
        if self.scheduler not in ("ils", "random", "progressive", "none"):
            raise ConfigError(f"unknown scheduler {self.scheduler!r}")


@dataclass
class RunLog:
    metrics: list = field(default_factory=list)     # (iteration, loss, accuracy, lr)
    schedule: list = field(default_factory=list)    # (iteration, layer_id, frozen, d_i)
    memory: list = field(default_factory=list)      # (iteration, dynamic, static, total)
    update_counts: np.ndarray | None = None
    layer_names: list = field(default_factory=list)
    decisions: list = field(default_factory=list)
    final_train_loss: float = float("nan")
    initial_train_loss: float = float("nan")
    final_accuracy: float = float("nan")
    distances_over_time: list = field(default_factory=list)
    peak_activation_bytes: list = field(default_factory=list)   # allocator peak per iteration

    def distance_matrix(self) -> np.ndarray:
        return np.asarray(self.distances_over_time)


def batches(data, batch_size: int, rng: np.random.Generator, shuffle: bool = True):
    """Deterministically shuffled drop-tail minibatches (trainer.py:134-141)."""
    tokens, labels = data
    n = len(labels)
    order = rng.permutation(n) if shuffle else np.arange(n)
    for start in range(0, n - batch_size + 1, batch_size):
        idx = order[start:start + batch_size]
        yield Batch(tokens[idx], labels[idx])


class StepEngine:
    """One SlimFit iteration on the device (used by fine_tune and bench.py).

    `dist` is an optional DataParallel helper (distributed.py); without it
    the engine is single-GPU.
    """

    def __init__(self, model: Model, run_config: RunConfig, dist=None):
        self.model = model
        self.rc = run_config
        self.dist = dist
        self.opt = OptimizerState(kind=run_config.optimizer, weight_decay=run_config.weight_decay,
                                  global_step_bias=run_config.global_step_bias)
        n = len(model.registry)
        self.d_dev = torch.zeros(n, dtype=torch.float64, device=model.device)
        self.d_host = torch.zeros(n, dtype=torch.float64).pin_memory()
        self.loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
        # the weights only change through this engine's optimizer (or torch
        # in-place ops, which bump their version): keep their GEMM planes
        G.keep_weight_planes(list(model.parameters()))
        if run_config.preallocate_state:
            # moments up front (for the layers this rank steps): a layer's first
            # activation then costs no allocation inside the step
            own = [p for e in model.registry
                   if dist is None or not dist.sharded_optimizer or dist.owner(e.id) == dist.rank
                   for p in e.params]
            self.opt.preallocate(own)

    def load_distances(self, dv: DistanceVector):
        self.d_host.copy_(torch.from_numpy(dv.d))
        self.d_dev.copy_(self.d_host)

    def forward_backward(self, batch: Batch, frozen_ids):
        model = self.model
        model.freeze_set(frozen_ids)
        model.zero_grad()
        labels = batch.labels
        if not isinstance(labels, torch.Tensor):
            labels = torch.as_tensor(np.asarray(labels))
        labels = labels.to(model.device, non_blocking=True)
        with T.record(self.rc.compression) as tape:
            logits = model.forward(batch)
            loss = T.cross_entropy(logits, labels)
            T.backward(loss)
        return loss.detach(), logits.detach(), labels, tape

    def step(self, batch: Batch, decision, lr: float, iteration: int):
        """Returns (loss, logits, labels, tape); updates params and d_dev."""
        active = sorted(decision.active_ids)
        dp = self.dist
        overlap = dp is not None and dp.world > 1 and not dp.sharded_optimizer
        if overlap:
            # freeze first so only the active layers' parameters get hooks
            self.model.freeze_set(decision.frozen_ids)
            dp.begin_backward(self.model, active)
        try:
            loss, logits, labels, tape = self.forward_backward(batch, decision.frozen_ids)
        except BaseException:
            if overlap:
                dp.abort_backward()
            raise
        if dp is not None:
            loss = dp.average_scalar(loss)
            if dp.sharded_optimizer:
                return self._step_sharded(loss, logits, labels, tape, active, decision, lr, iteration)
            if overlap:
                dp.finish_backward()
            else:
                dp.allreduce_active_grads(self.model, active)
        self.loss_host.copy_(loss.reshape(1), non_blocking=True)
        # no host round trip before the optimizer: the fused update +
        # distance launch (AdamW or SGD) is guarded by the loss on the
        # device (a non-finite loss leaves every parameter, moment and
        # distance untouched), and the host checks the loss once the step's
        # work has drained -- the reference's raise-before-update semantics
        # (trainer.py:175-190) without a pipeline bubble
        saved = self.opt.save_counters()
        self.opt.step(self.model, lr, active, self.d_dev, guard=loss)
        torch.cuda.current_stream().synchronize()
        loss_val = float(self.loss_host[0])
        if not math.isfinite(loss_val):
            self.opt.restore_counters(saved)
        self._check_finite(loss_val, iteration, lr, decision)
        return loss_val, logits, labels, tape

    def _step_sharded(self, loss, logits, labels, tape, active, decision, lr, iteration):
        """Layer-owner sharded optimizer step (distributed.py): C1 reduce to
        owners, K9 on the owned layers only, parameter broadcast, C2."""
        dp = self.dist
        stepped = {lid: [p for p in self.model.registry.by_id(lid).params if p.grad is not None]
                   for lid in active}
        stepped = {lid: ps for lid, ps in stepped.items() if ps}
        dp.reduce_grads_to_owners(self.model, active)
        dp.release_foreign_grads(self.model, active)
        self.loss_host.copy_(loss.reshape(1), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        loss_val = float(self.loss_host[0])
        self._check_finite(loss_val, iteration, lr, decision)
        d_owned = torch.zeros_like(self.d_dev)
        self.opt.step(self.model, lr, dp.owned(active), d_owned)
        dp.broadcast_owned_params(self.model, active, stepped)
        G.weight_planes_changed([p for ps in stepped.values() for p in ps])
        # owners wrote every owned active layer (0.0 where nothing moved)
        dp.combine_distances(self.d_dev, d_owned, active)
        return loss_val, logits, labels, tape

    def _check_finite(self, loss_val: float, iteration: int, lr: float, decision):
        if not math.isfinite(loss_val):
            raise TrainingDiverged(f"non-finite loss {loss_val} at iteration {iteration}",
                                   snapshot={"iteration": iteration, "loss": loss_val, "lr": lr,
                                             "frozen_ids": sorted(decision.frozen_ids),
                                             "distances": self.d_host.numpy().copy()})

    def fetch_distances(self, dv: DistanceVector, active):
        self.d_host.copy_(self.d_dev, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = self.d_host.numpy()
        for lid in active:
            dv.d[lid] = h[lid]
            dv.initialized_mask[lid] = True
            # scheduler.py:119 keeps a copy of the active layers' parameters
            # after the update.  A layer's parameters change only while it is
            # active, and then this entry is refreshed, so the live
            # parameters always equal that copy: alias them (no HBM copy)
            dv.snapshot[lid] = [p.detach() for p in self.model.registry.by_id(lid).params]


def fine_tune(model: Model, train_data, run_config: RunConfig, val_data=None,
              scheduler: Scheduler | None = None, dist=None, max_iters: int | None = None) -> RunLog:
    """The iterative-freezing loop (trainer.py:144-222) on the device.
    train_data / val_data are (tokens, labels) arrays (global batches; with
    `dist`, each rank trains on its slice of every batch)."""
    run_config.validate()
    tokens, labels = train_data
    if len(labels) == 0:
        raise ConfigError("training data is empty")
    n_layers = len(model.registry)
    iters_per_epoch = len(labels) // run_config.batch_size
    if iters_per_epoch == 0:
        raise ConfigError("batch size exceeds the training set")
    total_iters = iters_per_epoch * run_config.epochs
    if scheduler is None:
        scheduler = Scheduler(run_config.scheduler, n_layers, run_config.freeze_rate,
                              run_config.seed, total_iters, run_config.pinned_active)
    dv = init_distances(n_layers, run_config.seed)
    eng = StepEngine(model, run_config, dist)
    eng.load_distances(dv)
    log = RunLog(update_counts=np.zeros(n_layers, dtype=np.int64), layer_names=model.registry.names())
    data_rng = np.random.default_rng([run_config.seed, 0xDA7A])
    it = 0
    for _ in range(run_config.epochs):
        for batch in batches(train_data, run_config.batch_size, data_rng):
            if max_iters is not None and it >= max_iters:
                break
            if dist is not None:
                batch = dist.shard_batch(batch)
            decision = scheduler.decide(dv, it)
            lr = linear_schedule(run_config.lr, it, total_iters, run_config.warmup_frac)
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            loss_val, logits, lab, tape = eng.step(batch, decision, lr, it)
            active = sorted(decision.active_ids)
            eng.fetch_distances(dv, active)
            log.peak_activation_bytes.append(torch.cuda.max_memory_allocated() - base)
            acc = float((logits.argmax(dim=1) == lab).float().mean())
            log.metrics.append((it, loss_val, acc, lr))
            for lid in range(n_layers):
                log.schedule.append((it, lid, int(lid in decision.frozen_ids), float(dv.d[lid])))
            log.update_counts[active] += 1
            log.decisions.append(decision)
            log.distances_over_time.append(dv.d.copy())
            if run_config.track_memory:
                cb = tape.cached_bytes()
                log.memory.append((it, cb["dynamic"], cb["static"] + cb["semi_static"], cb["total"]))
            if it == 0:
                log.initial_train_loss = loss_val
            it += 1
    if log.metrics:
        log.final_train_loss = log.metrics[-1][1]
    model.freeze_set(())
    if val_data is not None:
        log.final_accuracy, _ = evaluate(model, val_data, run_config.batch_size)
    return log


def evaluate(model: Model, data, batch_size: int = 64) -> tuple[float, float]:
    """Accuracy and mean loss, forward only (trainer.py:225-247)."""
    tokens, labels = data
    correct, loss_sum, seen = 0, 0.0, 0
    with T.no_grad():
        for s in range(0, len(labels), batch_size):
            b = Batch(tokens[s:s + batch_size], labels[s:s + batch_size])
            logits = model.forward(b)
            lab = torch.as_tensor(np.asarray(b.labels), device=model.device).long()
            loss = torch.nn.functional.cross_entropy(logits, lab)
            nb = len(b.labels)
            correct += int((logits.argmax(dim=1) == lab).sum())
            loss_sum += float(loss) * nb
            seen += nb
    return correct / seen, loss_sum / seen
