"""SlimFit activation-memory hot path, B200-native (sm_100a kernels behind a C ABI).

Drop-in for the reference package's hot path (reference
`slimfit/__init__.py:18-41` names): codecs, freeze-aware ops with the cached
activation ledger, the freezable-layer model and registry, the ILS scheduler
and the fine-tuning loop.  Device work goes through libslimfit_b200.so; a
missing library raises `NativeUnavailable` (no CPU fallback).
"""

import os as _os

_threads = _os.environ.get("SLIMFIT_THREADS")
if _threads:
    for _var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        _os.environ.setdefault(_var, _threads)

from .errors import (  # noqa: E402
    CodecError, ConfigError, RegistryError, ShapeError, SlimfitError, TrainingDiverged,
)
from .compression import (  # noqa: E402
    CompressedActivation, FixedPointSpec, PrunedSparse, Q0_8_UNSIGNED, Q2_2, Q4_4,
    choose_prescale_exp, dequantize, pack4, prune_topk, quantize, restore, unpack4,
)

__version__ = "0.1.0"


def _lazy():
    # heavier modules (model/trainer) import on first attribute access
    from . import memory, model, scheduler, tensor, trainer  # noqa: F401


def __getattr__(name):
    lazy = {
        "tensor": ("tensor", None), "model": ("model", None), "scheduler": ("scheduler", None),
        "trainer": ("trainer", None), "memory": ("memory", None),
        "CompressionConfig": ("tensor", "CompressionConfig"), "SavedValue": ("tensor", "SavedValue"),
        "Tape": ("tensor", "Tape"), "record": ("tensor", "record"), "no_grad": ("tensor", "no_grad"),
        "Model": ("model", "Model"), "ModelConfig": ("model", "ModelConfig"),
        "LayerRegistry": ("model", "LayerRegistry"), "Batch": ("model", "Batch"),
        "build_model": ("model", "build_model"),
        "DistanceVector": ("scheduler", "DistanceVector"), "FreezeDecision": ("scheduler", "FreezeDecision"),
        "Scheduler": ("scheduler", "Scheduler"), "init_distances": ("scheduler", "init_distances"),
        "select_frozen": ("scheduler", "select_frozen"), "update_distances": ("scheduler", "update_distances"),
        "layer_distance": ("scheduler", "layer_distance"),
        "baseline_random": ("scheduler", "baseline_random"),
        "baseline_progressive": ("scheduler", "baseline_progressive"),
        "OptimizerState": ("trainer", "OptimizerState"), "RunConfig": ("trainer", "RunConfig"),
        "RunLog": ("trainer", "RunLog"), "fine_tune": ("trainer", "fine_tune"),
        "evaluate": ("trainer", "evaluate"),
        "MemoryReport": ("memory", "MemoryReport"), "account_iteration": ("memory", "account_iteration"),
        "account_budget": ("memory", "account_budget"), "audit_runtime": ("memory", "audit_runtime"),
        "enumerate_records": ("memory", "enumerate_records"), "imbalance_ratio": ("memory", "imbalance_ratio"),
    }
    if name in lazy:
        import importlib
        mod, attr = lazy[name]
        m = importlib.import_module(f".{mod}", __name__)
        return m if attr is None else getattr(m, attr)
    raise AttributeError(name)
