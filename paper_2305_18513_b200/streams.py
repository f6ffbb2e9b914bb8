"""Codec side stream: encoders whose output is only read by the backward pass.

The forward pass of a SlimFit step interleaves compute-bound GEMMs with
HBM-bound cache encoders (the frozen-LayerNorm top-k prune, the q/k/v and
dense 8-bit codes, the GELU 4-bit pack; reference call sites tensor.py:282,
:396, :474).  Nothing in the forward consumes those payloads, so they are
enqueued on a second CUDA stream that waits for the producer and then runs
alongside the following GEMMs.  The payload carries the completion event;
its first consumer (`CompressedActivation.wait`) makes the consuming stream
wait on it and re-tags the payload's memory for that stream, so the caching
allocator never hands the blocks out early.

`SLIMFIT_SIDE_STREAM=0` (or `set_enabled(False)`) runs every encoder inline
on the current stream — bench.py does so for its per-kernel timing pass so
each kernel's CUDA-event time is measured without overlap.
"""

from __future__ import annotations

import os

import torch

_enabled = os.environ.get("SLIMFIT_SIDE_STREAM", "1") != "0"
_streams: dict = {}


def enabled() -> bool:
    return _enabled


def set_enabled(flag: bool) -> None:
    global _enabled
    _enabled = bool(flag)


def side_stream(device=None) -> torch.cuda.Stream:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if dev is None:
        dev = torch.cuda.current_device()
    s = _streams.get(dev)
    if s is None:
        s = _streams[dev] = torch.cuda.Stream(device=dev)
    return s


def run(fn, *inputs):
    """fn() ordered after all work already queued on the current stream.
    Returns (result, event): with the side stream on, fn runs on it and
    `event` marks its completion (None when run inline).  `inputs` are
    tensors produced on the current stream that fn reads; they are tagged
    for the side stream so freeing them early stays safe."""
    if not _enabled:
        return fn(), None
    main = torch.cuda.current_stream()
    side = side_stream(main.device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        out = fn()
    for t in inputs:
        if t is not None:
            t.record_stream(side)
    ev = torch.cuda.Event()
    ev.record(side)
    return out, ev


def consume(event, tensors):
    """Make the current stream wait for `event` and tag `tensors` (allocated
    on the side stream) as used by it."""
    if event is None:
        return
    cur = torch.cuda.current_stream()
    cur.wait_event(event)
    for t in tensors:
        if t is not None:
            t.record_stream(cur)
