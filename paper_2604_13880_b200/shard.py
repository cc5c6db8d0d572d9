"""Multi-GPU plumbing: one process per GPU, independent units sharded, final gather only.

The DET iteration does not shard; independent cartograms do: direct-mode time
steps (temporal.py:185-246 runs them one after another), bdv-multiplier sweeps (cli.py:265-300)
and the cartograms of a batch.  Units are dealt out in contiguous blocks (``shard_bounds``), so
every process's block runs in the same kernel launches of its GPU, and the only exchange is the
gather of the per-unit results at the end.

Two ways to run a sharded job (``run_sharded``):

* ``devices=[0, 1, ...]`` from one Python process: one persistent worker process per GPU
  (spawned on first use, its device contexts cached between calls) computes its block; the
  caller collects the blocks in unit order.
* ``distributed=True`` under ``torchrun`` (one process per GPU, ``torch.distributed``
  initialised by the caller, any backend): rank r computes block r on its local GPU
  (``LOCAL_RANK``) and an ``all_gather_object`` gives every rank the full result list.

Cumulative chains are sequential and do not shard (replicas only).
"""

from __future__ import annotations

import atexit
import os
from concurrent.futures import ProcessPoolExecutor

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


def gather_objects(local: list, group=None) -> list:
    """Every rank's list of per-unit results, concatenated in rank order, on every rank."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(local)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, list(local), group=group)
    return [x for part in out for x in part]


_EXECUTORS: dict = {}


def _worker_init(device: int):
    os.environ.setdefault("DET_WORKER_DEVICE", str(device))


def _executor(device: int) -> ProcessPoolExecutor:
    """The persistent worker process of one GPU (spawned: CUDA state is never forked)."""
    ex = _EXECUTORS.get(device)
    if ex is None:
        import multiprocessing as mp

        ex = ProcessPoolExecutor(max_workers=1, mp_context=mp.get_context("spawn"), initializer=_worker_init,
                                 initargs=(device,))
        _EXECUTORS[device] = ex
    return ex


@atexit.register
def shutdown_workers():
    """Stop the per-GPU worker processes (also runs at interpreter exit)."""
    while _EXECUTORS:
        _, ex = _EXECUTORS.popitem()
        ex.shutdown(wait=True, cancel_futures=True)


def run_sharded(n_units: int, task, *, devices=None, distributed: bool = False, group=None) -> list:
    """``task(lo, hi, device) -> list`` (one entry per unit of [lo, hi)) over every unit.

    ``task`` must be picklable (a module-level function or a ``functools.partial`` of one) when
    ``devices`` names more than one GPU.  Returns the results of all units in unit order.
    """
    if distributed:
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("distributed=True needs an initialised torch.distributed process group")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        lo, hi = shard_bounds(n_units, rank, world)
        dev = int(os.environ.get("LOCAL_RANK", "0")) if devices is None else int(list(devices)[rank % len(devices)])
        local = task(lo, hi, dev) if hi > lo else []
        return gather_objects(local, group)
    devs = [0] if devices is None else [int(d) for d in devices]
    if not devs:
        raise ValueError("devices must name at least one GPU")
    if len(devs) == 1:
        return list(task(0, n_units, devs[0])) if n_units else []
    futures = []
    for r, d in enumerate(devs):
        lo, hi = shard_bounds(n_units, r, len(devs))
        if hi > lo:
            futures.append(_executor(d).submit(task, lo, hi, d))
    out = []
    for f in futures:
        out.extend(f.result())
    return out
