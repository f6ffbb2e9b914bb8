"""ILS scheduler — the drop-in for scheduler.py (/root/reference/pkg/src/slimfit).

Decisions (warm start, stable freeze selection, the random/progressive
baselines) stay on the host in numpy: they are O(n_layers) with n <= 198 and
must match the reference bit for bit, which numpy's own argsort/PCG64
guarantee.  The per-layer update distance (scheduler.py:92-120) runs on the
device: one launch of the numpy-pairwise-exact K8 kernel over all active
layers, or fused into the AdamW step (K9, see trainer.OptimizerState).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError

INIT_LOW = 1.0e6      # warm-start range: any real distance ranks below it (scheduler.py:19-20)
INIT_HIGH = 2.0e6
EPS_DIV = 1.0e-12     # |b| + eps guard of the relative change (scheduler.py:21)


@dataclass
class DistanceVector:
    """Per-layer distance state (scheduler.py:24-46).  `d` is the host copy
    the decisions read; `snapshot` is kept for API parity only."""

    d: np.ndarray
    initialized_mask: np.ndarray
    snapshot: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.d.size


@dataclass(frozen=True)
class FreezeDecision:
    iteration: int
    frozen_ids: frozenset
    active_ids: frozenset

    @property
    def frozen_count(self) -> int:
        return len(self.frozen_ids)


def init_distances(n: int, seed: int) -> DistanceVector:
    """Uniform warm-start values in [1e6, 2e6) from default_rng(seed) (scheduler.py:53-59)."""
    if n < 1:
        raise ConfigError(f"need at least one layer, got n={n}")
    d = np.random.default_rng(seed).uniform(INIT_LOW, INIT_HIGH, size=n)
    return DistanceVector(d=d, initialized_mask=np.zeros(n, dtype=bool))


def frozen_count(n: int, freeze_rate: float) -> int:
    return int(n * freeze_rate)


def _check_rate(freeze_rate: float):
    if not 0.0 <= freeze_rate < 1.0:
        raise ConfigError(f"freeze rate must lie in [0, 1), got {freeze_rate}")


def select_frozen(dv: DistanceVector, freeze_rate: float, iteration: int = 0,
                  pinned_active=()) -> FreezeDecision:
    """Freeze the int(n*F) smallest distances; stable order breaks ties toward
    the lower id; pinned layers rank as +inf (scheduler.py:71-89)."""
    _check_rate(freeze_rate)
    n = dv.n
    d = dv.d
    if pinned_active:
        d = np.array(d, copy=True)
        d[list(pinned_active)] = np.inf
    order = np.argsort(d, kind="stable")
    frozen = frozenset(int(i) for i in order[:frozen_count(n, freeze_rate)])
    return FreezeDecision(iteration, frozen, frozenset(range(n)) - frozen)


def baseline_random(n: int, freeze_rate: float, seed: int, iteration: int) -> FreezeDecision:
    """Random frozen subset from default_rng([seed, iteration]) (scheduler.py:123-129)."""
    _check_rate(freeze_rate)
    pick = np.random.default_rng([seed, iteration]).choice(n, size=frozen_count(n, freeze_rate),
                                                          replace=False)
    frozen = frozenset(int(i) for i in pick)
    return FreezeDecision(iteration, frozen, frozenset(range(n)) - frozen)


def baseline_progressive(n: int, freeze_rate: float, iteration: int,
                         total_iterations: int) -> FreezeDecision:
    """Fixed prefix of int(n*F) frozen layers (scheduler.py:132-142)."""
    _check_rate(freeze_rate)
    frozen = frozenset(range(frozen_count(n, freeze_rate)))
    return FreezeDecision(iteration, frozen, frozenset(range(n)) - frozen)


class Scheduler:
    """Decision source for the loop: "ils" | "random" | "progressive" | "none"
    (scheduler.py:145-173)."""

    def __init__(self, kind: str, n: int, freeze_rate: float, seed: int,
                 total_iterations: int = 0, pinned_active=()):
        if kind not in ("ils", "random", "progressive", "none"):
            raise ConfigError(f"unknown scheduler kind {kind!r}")
        _check_rate(freeze_rate)
        self.kind, self.n, self.freeze_rate, self.seed = kind, n, freeze_rate, seed
        self.total_iterations = total_iterations
        self.pinned_active = tuple(pinned_active)

    def decide(self, dv: DistanceVector, iteration: int) -> FreezeDecision:
        if self.kind == "ils":
            return select_frozen(dv, self.freeze_rate, iteration, self.pinned_active)
        if self.kind == "random":
            return baseline_random(self.n, self.freeze_rate, self.seed, iteration)
        if self.kind == "progressive":
            return baseline_progressive(self.n, self.freeze_rate, iteration, self.total_iterations)
        return FreezeDecision(iteration, frozenset(), frozenset(range(self.n)))


# --------------------------------------------------------------------------- device distance

def _split(n: int) -> int:
    h = n // 2
    return h - h % 8


_TREE_CACHE: dict[int, tuple] = {}


def pairwise_plan(n: int):
    """Chunks (offset, length) and the level-ordered combine tree above them
    for numpy's pairwise add-reduce of n elements (see distance.cu)."""
    hit = _TREE_CACHE.get(n)
    if hit is not None:
        return hit
    chunks: list[tuple[int, int]] = []
    nodes: list[list] = []          # [left_ref, right_ref, height]

    def rec(off, m):
        if m <= N.DIST_CHUNK:
            chunks.append((off, m))
            return ("c", len(chunks) - 1), 0
        h = _split(m)
        lref, lh = rec(off, h)
        rref, rh = rec(off + h, m - h)
        nodes.append([lref, rref, max(lh, rh) + 1])
        return ("n", len(nodes) - 1), max(lh, rh) + 1

    rec(0, n)
    nc = len(chunks)
    order = sorted(range(len(nodes)), key=lambda i: (nodes[i][2], i))
    new_id = {old: nc + k for k, old in enumerate(order)}

    def ref_id(r):
        return r[1] if r[0] == "c" else new_id[r[1]]

    tree = np.array([[ref_id(nodes[i][0]), ref_id(nodes[i][1])] for i in order],
                    dtype=np.int32).reshape(-1, 2)
    heights = [nodes[i][2] for i in order]
    bounds = [0]
    for k in range(1, len(heights)):
        if heights[k] != heights[k - 1]:
            bounds.append(k)
    bounds.append(len(heights))
    levels = np.array(bounds if heights else [0], dtype=np.int32)
    out = (np.array(chunks, dtype=np.int32).reshape(-1, 2), tree, levels)
    _TREE_CACHE[n] = out
    return out


_PROG_CACHE: dict[int, np.ndarray] = {}


def chunk_program(length: int) -> np.ndarray:
    """Shape of numpy's pairwise tree over one chunk of `length` (<= 4096)
    elements, as the device kernel consumes it:
    [nleaves, nnodes, nlevels, (off, len) * nleaves, (left, right) * nnodes,
     level bounds * (nlevels + 1)]; operand ids < nleaves name leaf sums,
    larger ids name internal nodes (id - nleaves), levels bottom-up."""
    hit = _PROG_CACHE.get(length)
    if hit is not None:
        return hit
    leaves: list[tuple[int, int]] = []
    nodes: list[list] = []

    def rec(off, m):
        if m <= 128:
            leaves.append((off, m))
            return ("l", len(leaves) - 1), 0
        h = _split(m)
        lref, lh = rec(off, h)
        rref, rh = rec(off + h, m - h)
        nodes.append([lref, rref, max(lh, rh) + 1])
        return ("n", len(nodes) - 1), max(lh, rh) + 1

    rec(0, length)
    nl = len(leaves)
    order = sorted(range(len(nodes)), key=lambda i: (nodes[i][2], i))
    new_id = {old: nl + k for k, old in enumerate(order)}

    def rid(r):
        return r[1] if r[0] == "l" else new_id[r[1]]

    heights = [nodes[i][2] for i in order]
    bounds = [0] + [k for k in range(1, len(heights)) if heights[k] != heights[k - 1]]
    bounds = bounds + [len(heights)] if heights else [0]
    prog = [nl, len(nodes), len(bounds) - 1 if heights else 0, 0]   # 4-int header keeps pairs 8 B aligned
    for o, m in leaves:
        prog += [o, m]
    for i in order:
        prog += [rid(nodes[i][0]), rid(nodes[i][1])]
    prog += bounds
    out = np.array(prog, dtype=np.int32)
    _PROG_CACHE[length] = out
    return out


class DistancePlan:
    """Static device tables for a fixed list of parameter shapes (built once
    per model) and the per-call launcher of K8 / K9."""

    def __init__(self, sizes, device="cuda"):
        self.device = torch.device(device)
        chunk_rows, tree_rows, level_rows = [], [], []
        progs, prog_off = [], {}
        self.meta = []       # per slot: (n, chunk0, nchunk, tree0, nnode, level0, nlevel)
        c0 = t0 = l0 = 0
        p0 = 0
        for n in sizes:
            ch, tr, lv = pairwise_plan(int(n))
            nlev = len(lv) - 1 if tr.shape[0] else 0
            self.meta.append((int(n), c0, ch.shape[0], t0, tr.shape[0], l0, nlev))
            rows4 = np.zeros((ch.shape[0], 4), dtype=np.int32)
            rows4[:, :2] = ch
            for r, length in enumerate(ch[:, 1].tolist()):
                if length not in prog_off:
                    pg = chunk_program(length)
                    prog_off[length] = p0
                    progs.append(pg)
                    p0 += pg.size
                rows4[r, 2] = prog_off[length]
            ch = rows4
            chunk_rows.append(ch)
            tree_rows.append(tr)
            level_rows.append(lv)
            c0 += ch.shape[0]
            t0 += tr.shape[0]
            l0 += len(lv)
        self.total_nodes = t0

        def dev(parts, dtype, width):
            arr = np.concatenate(parts) if parts else np.zeros((0, width), dtype)
            if arr.size == 0:
                arr = np.zeros(max(width, 1), dtype)
            return torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype)).to(self.device)

        self.h2d_bytes = 0       # per-call table uploads, for bench.py's e2e accounting
        # per-call tables are staged through pinned buffers allocated once:
        # a fresh pin_memory() per call goes to cudaHostAlloc whenever the
        # active set yields a new table size, a multi-millisecond stall
        ns = max(1, len(self.meta))
        self._tab_h = torch.zeros((ns, N.SLOT_WORDS), dtype=torch.int64).pin_memory()
        self._lay_h = torch.zeros((ns, 3), dtype=torch.int32).pin_memory()
        self._cnt_h = torch.zeros(ns, dtype=torch.int64).pin_memory()
        self._tab_d = torch.empty((ns, N.SLOT_WORDS), dtype=torch.int64, device=self.device)
        self._lay_d = torch.empty((ns, 3), dtype=torch.int32, device=self.device)
        self._cnt_d = torch.empty(ns, dtype=torch.int64, device=self.device)
        self._staged = None      # event after the last upload from the staging buffers
        self._ws = None
        self._all_chunks = sum(m[2] for m in self.meta)
        self.chunk_tab = dev(chunk_rows, np.int32, 4)
        self.prog_tab = dev(progs, np.int32, 1)
        self.tree_tab = dev(tree_rows, np.int32, 2)
        self.level_tab = dev([lv.reshape(-1) for lv in level_rows], np.int32, 1)

    def run(self, rows, layers, d_out: torch.Tensor, update: int = N.UPDATE_NONE,
            guard: torch.Tensor | None = None):
        """rows: list of dicts {slot, A, B, M, V, consts...}; layers: list of
        (first_row, n_rows, out_index, count) -- a layer's moved parameters
        are rows first_row .. first_row + n_rows - 1 (n_rows may be 0: an
        active layer that did not move gets d = 0.0); count covers all its
        elements.  Writes d_out[out_index] only.  update: N.UPDATE_NONE
        (rows hold before/after), N.UPDATE_ADAMW or N.UPDATE_SGD (rows hold
        param/grad; the parameters are stepped in the same launch)."""
        if not rows and not layers:
            return
        tab = np.zeros((len(rows), N.SLOT_WORDS), dtype=np.int64)
        cbase = 0
        for j, r in enumerate(rows):
            n, c0, nc, t0, nn, l0, nl = self.meta[r["slot"]]
            w = tab[j]
            w[N.SLOT["A"]] = r["A"]
            w[N.SLOT["B"]] = r["B"]
            w[N.SLOT["M"]] = r.get("M", 0)
            w[N.SLOT["V"]] = r.get("V", 0)
            w[N.SLOT["N"]] = n
            w[N.SLOT["CHUNK0"]] = c0
            w[N.SLOT["NCHUNK"]] = nc
            w[N.SLOT["TREE0"]] = t0
            w[N.SLOT["NNODE"]] = nn
            w[N.SLOT["LEVEL0"]] = l0
            w[N.SLOT["NLEVEL"]] = nl
            w[N.SLOT["CBASE"]] = cbase
            if update == N.UPDATE_ADAMW:
                c = r["consts"]
                w[N.SLOT["BETA1"]] = _pack(c["b1"], c["ob1"])
                w[N.SLOT["BETA2"]] = _pack(c["b2"], c["ob2"])
                w[N.SLOT["BC"]] = _pack(c["bc1"], c["bc2"])
                w[N.SLOT["EPSWD"]] = _pack(c["eps"], c["wd"])
                w[N.SLOT["LR"]] = _pack(c["lr"], 0.0)
            elif update == N.UPDATE_SGD:
                w[N.SLOT["LR"]] = _pack(r["lr"], 0.0)
            cbase += nc
        lay = np.array([[a, b, o] for a, b, o, _ in layers], dtype=np.int32).reshape(-1, 3)
        cnt = np.array([c for *_, c in layers], dtype=np.int64)
        if self._staged is not None:
            self._staged.synchronize()          # the previous upload has left the staging buffers
        nr, nl = max(1, len(rows)), max(1, len(layers))
        self._tab_h.numpy()[:len(rows)] = tab
        if lay.size:
            self._lay_h.numpy()[:len(layers)] = lay
            self._cnt_h.numpy()[:len(layers)] = cnt
        tab_d = self._tab_d[:nr]
        lay_d = self._lay_d[:nl]
        cnt_d = self._cnt_d[:nl]
        tab_d.copy_(self._tab_h[:nr], non_blocking=True)
        lay_d.copy_(self._lay_h[:nl], non_blocking=True)
        cnt_d.copy_(self._cnt_h[:nl], non_blocking=True)
        self._staged = torch.cuda.Event()
        self._staged.record()
        lib = N.load()
        N.distance_params = int(tab[:, N.SLOT["N"]].sum())
        self.h2d_bytes += tab.nbytes + lay.nbytes + cnt.nbytes
        need = lib.sf_distance_workspace_bytes(cbase, len(rows), self.total_nodes)
        if self._ws is None or self._ws.numel() < need:
            # sized for every parameter active at once, allocated once
            full = lib.sf_distance_workspace_bytes(self._all_chunks, max(1, len(self.meta)), self.total_nodes)
            self._ws = torch.empty(max(need, full), dtype=torch.uint8, device=self.device)
        ws = self._ws
        self._last = (tab_d.data_ptr(), len(rows), cbase, self.chunk_tab.data_ptr(),
                      self.prog_tab.data_ptr(), self.tree_tab.data_ptr(), self.level_tab.data_ptr(), self.total_nodes,
                      lay_d.data_ptr(), cnt_d.data_ptr(), len(layers), d_out.data_ptr(), int(update),
                      guard.data_ptr() if guard is not None else None, ws.data_ptr())
        self.relaunch()

    def relaunch(self):
        """Issue the last `run`'s launch again on the current stream, with
        the tables it uploaded (kernel timing without the host-side table
        build; with an update mode the parameters step again)."""
        N.call("sf_layer_distance", *self._last, torch.cuda.current_stream().cuda_stream)


def _pack(a, b) -> int:
    lo = int(np.float32(a).view(np.uint32))
    hi = int(np.float32(b).view(np.uint32))
    v = lo | (hi << 32)
    return v - (1 << 64) if v >= (1 << 63) else v


def _as_dev(p) -> torch.Tensor:
    t = p if isinstance(p, torch.Tensor) else torch.as_tensor(np.asarray(p))
    if not t.is_cuda:
        t = t.cuda()
    return t.detach().to(torch.float32).contiguous()


def layer_distances_device(before: dict, after: dict, active_ids, d_out: torch.Tensor):
    """K8 over all active layers in one launch: before/after map layer_id ->
    list of tensors (any number per layer, pooled in order as
    scheduler.py:100-105 does); writes d_out[layer_id] (float64, device)."""
    rows, layers, sizes, keep = [], [], [], []
    for lid in active_ids:
        j0, count = len(rows), 0
        for b, a in zip(before[lid], after[lid]):
            tb, ta = _as_dev(b), _as_dev(a)
            if tb.numel() != ta.numel():
                raise ConfigError(f"layer {lid}: before/after sizes differ ({tb.numel()} vs {ta.numel()})")
            count += tb.numel()
            if tb.numel() == 0:
                continue
            keep += [tb, ta]
            rows.append({"slot": len(sizes), "A": tb.data_ptr(), "B": ta.data_ptr()})
            sizes.append(tb.numel())
        layers.append((j0, len(rows) - j0, int(lid), count))
    if not layers:
        return
    DistancePlan(sizes, d_out.device).run(rows, layers, d_out, N.UPDATE_NONE)


def layer_distance(params_before, params_after) -> float:
    """Pooled mean |after - before| / (|before| + 1e-12) over one layer's
    params, float64, bit-identical to the reference (scheduler.py:92-105).
    Synchronises to return a float."""
    if not list(params_before):
        return 0.0
    d = torch.zeros(1, dtype=torch.float64, device="cuda")
    layer_distances_device({0: list(params_before)}, {0: list(params_after)}, [0], d)
    return float(d.item())


def update_distances(dv: DistanceVector, params_before: dict, params_after: dict,
                     active_ids) -> DistanceVector:
    """Refresh the active layers' entries (scheduler.py:108-120); frozen
    entries, masks and snapshots are untouched."""
    active = list(active_ids)
    if not active:
        return dv
    d = torch.from_numpy(np.array(dv.d, dtype=np.float64)).cuda()
    layer_distances_device(params_before, params_after, active, d)
    host = d.cpu().numpy()
    for lid in active:
        dv.d[lid] = host[lid]
        dv.initialized_mask[lid] = True
        dv.snapshot[lid] = [_as_dev(p).clone() for p in params_after[lid]]
    return dv
