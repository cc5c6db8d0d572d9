"""Multi-GPU plumbing: one process per GPU, independent units sharded, final gather only.

The DET iteration does not shard; independent cartograms
(direct-mode time steps, parameter sweeps) do.  Frames are dealt out in
contiguous blocks so every rank's batch runs in the same kernel launches; the
only collective is the end-of-run gather of per-frame results.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of units owned by `rank` (sizes differ by at most one)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_frame_results(local: dict, dist=None) -> dict:
    """Concatenate per-rank dicts of equally-keyed numpy arrays (rank order) via torch.distributed."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return {k: np.asarray(v) for k, v in local.items()}
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, {k: np.asarray(v) for k, v in local.items()})
    return {k: np.concatenate([o[k] for o in out]) for k in local}
