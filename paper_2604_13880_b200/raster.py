"""Label / density textures -- drop-in for cartomorph/raster.py, computed on the GPU.

``rasterize_labels`` (raster.py:136-155) runs the sm_100a rasteriser
(``k_region`` + ``k_row``, csrc/det_raster.cuh) through the C-ABI
``det_rasterize``; ``build_density`` (raster.py:166-184) runs ``det_density``.
Labels are int32 ``[j, i]`` with ``BACKGROUND = -1`` and equal the reference's
bit for bit (tests/test_gpu_parity.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._context import get_context, region_ranks
from .errors import RasterizationError
from .geomodel import ring_layout

BACKGROUND = -1


class _LazyLabels:
    """Deferred label texture of a run result: read back from the device while the context
    still holds it, otherwise re-rasterised from the result's own vertices (the raster is
    deterministic, so both give the same array).  Pickles without its context (a result sent
    from a per-GPU worker process re-rasterises on first access)."""

    def __init__(self, ctx, b, generation, mapmodel, k, device):
        self.ctx, self.b, self.gen, self.mapmodel, self.k, self.device = ctx, b, generation, mapmodel, k, device

    def __getstate__(self):
        return dict(self.__dict__, ctx=None, gen=None, device=0)

    def materialize(self) -> np.ndarray:
        if self.ctx is not None and getattr(self.ctx, "generation", None) == self.gen:
            return self.ctx.labels(self.b)
        return rasterize_labels(self.mapmodel, self.k, check_collapse=False, device=self.device).labels


@dataclass(frozen=True)
class LabelTexture:
    """Per-pixel region index; BACKGROUND (-1) marks unclaimed pixels (raster.py:102-118).

    ``labels`` may be backed by a device buffer and materialised on first access.
    """

    size: int
    _labels: object
    region_ids: tuple
    _counts: np.ndarray | None = field(default=None, repr=False, compare=False)

    def __init__(self, size, labels, region_ids, _counts=None):
        object.__setattr__(self, "size", size)
        object.__setattr__(self, "_labels", labels)
        object.__setattr__(self, "region_ids", tuple(region_ids))
        object.__setattr__(self, "_counts", _counts)

    @property
    def labels(self) -> np.ndarray:
        if isinstance(self._labels, _LazyLabels):
            object.__setattr__(self, "_labels", self._labels.materialize())
        return self._labels

    def pixel_counts(self) -> np.ndarray:
        if self._counts is not None:
            return self._counts[:-1].astype(np.int64)
        flat = self.labels[self.labels >= 0]
        return np.bincount(flat, minlength=len(self.region_ids)).astype(np.int64)

    def background_count(self) -> int:
        if self._counts is not None:
            return int(self._counts[-1])
        return int((self.labels == BACKGROUND).sum())

    def map_pixel_count(self) -> int:
        return self.size * self.size - self.background_count()


@dataclass(frozen=True)
class DensityTexture:
    """Piecewise-constant density with its domain mean d0 and the applied BDV (raster.py:121-133)."""

    size: int
    d: np.ndarray
    d0: float
    bdv: float
    pixel_counts: np.ndarray

    @property
    def total(self) -> float:
        return float(self.d.sum())


def _check_k(k: int):
    if not (4 <= k <= 13):
        raise ValueError("texture exponent k must be in [4, 13]")


def rasterize_labels(mapmodel, k: int, check_collapse: bool = True, device: int = 0) -> LabelTexture:
    """Rasterise all regions at resolution 2^k (raster.py:136-155) on the GPU."""
    _check_k(k)
    xy, rs, rr, ids, stats = ring_layout(mapmodel)
    ctx = get_context(k, device)
    ctx.load_map(xy, rs, rr, region_ranks(ids))
    ctx.set_batch(stats[None, :])
    lab, cnt = ctx.rasterize(0)
    tex = LabelTexture(size=1 << k, labels=lab, region_ids=tuple(ids), _counts=cnt)
    if check_collapse:
        empty = [rid for rid, c in zip(ids, cnt[:-1]) if c == 0]
        if empty:
            n = 1 << k
            raise RasterizationError(f"zero-pixel region(s) at resolution {n}x{n}: {empty} (resolution too low)")
    return tex


def default_bdv(statistics: np.ndarray, labels: LabelTexture) -> float:
    """Mean density over the map pixels (raster.py:158-163)."""
    n_map = labels.map_pixel_count()
    if n_map == 0:
        raise RasterizationError("map rasterized to zero pixels")
    return float(np.sum(statistics)) / n_map


def build_density(statistics: np.ndarray, labels: LabelTexture, bdv: float, device: int = 0) -> DensityTexture:
    """Per-pixel density s/o inside regions and ``bdv`` on the background, on the GPU."""
    if bdv <= 0:
        raise ValueError("bdv must be positive")
    from ._lib import DET_E_RASTER, DetError

    k = int(labels.size).bit_length() - 1
    ctx = get_context(k, device)
    lab = np.ascontiguousarray(labels.labels, dtype=np.int32)
    stats = np.ascontiguousarray(statistics, dtype=np.float64)
    d = np.empty((labels.size, labels.size), dtype=np.float64)
    cnt = np.empty(stats.shape[0] + 1, dtype=np.int64)
    import ctypes

    rc = ctx.lib.det_density(ctx.h, lab.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                             stats.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), stats.shape[0], float(bdv),
                             d.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc == DET_E_RASTER:
        raise RasterizationError("cannot build density with zero-pixel regions")
    if rc != 0:
        raise DetError(rc, ctx.lib.det_last_error(ctx.h).decode())
    m = labels.size * labels.size
    return DensityTexture(size=labels.size, d=d, d0=float(d.sum()) / m, bdv=float(bdv), pixel_counts=cnt[:-1])


def write_pgm16(path, array: np.ndarray) -> None:
    """Debug dump as a 16-bit binary PGM, values min-max scaled to [0, 65535] (raster.py:187-196)."""
    a = np.asarray(array, dtype=float)
    lo, hi = float(a.min()), float(a.max())
    scaled = np.zeros_like(a) if hi == lo else (a - lo) / (hi - lo)
    with open(path, "wb") as fh:
        fh.write(f"P5\n{a.shape[1]} {a.shape[0]}\n65535\n".encode())
        fh.write((scaled * 65535).round().astype(">u2").tobytes())


def write_raw_f32(path, array: np.ndarray) -> None:
    """Headerless little-endian float32 row-major dump (raster.py:199-201)."""
    np.asarray(array, dtype="<f4").tofile(path)


def write_raw_f64(path, array: np.ndarray) -> None:
    """Headerless little-endian float64 row-major dump (raster.py:204-206)."""
    np.asarray(array, dtype="<f8").tofile(path)
