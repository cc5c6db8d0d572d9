"""Per-thread cache of device contexts (one CUDA stream + buffers per (device, k, field dtype)).

Engines are cheap to construct (the reference builds one per temporal frame,
temporal.py:190-197); re-using the context keeps device buffers resident across
frames instead of re-allocating them.
"""

from __future__ import annotations

import threading

import numpy as np

from ._lib import Context

_tls = threading.local()


def get_context(k: int, device: int = 0, precision: str = "float32") -> Context:
    """The calling thread's context for (device, k, precision); precision is a field_dtype
    ("float32", "float64" or "mixed")."""
    cache = getattr(_tls, "cache", None)
    if cache is None:
        cache = _tls.cache = {}
    key = (device, k, precision)
    ctx = cache.get(key)
    if ctx is None:
        ctx = cache[key] = Context(k, device=device, precision=precision)
    return ctx


def region_ranks(ids) -> np.ndarray:
    """Rank of every region in ascending region_id order (raster.py:142)."""
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    rank = np.empty(len(ids), dtype=np.int32)
    rank[np.asarray(order, dtype=np.int64)] = np.arange(len(ids), dtype=np.int32)
    return rank
