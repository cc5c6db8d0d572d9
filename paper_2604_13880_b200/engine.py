"""Iterative cartogram construction -- drop-in for cartomorph/engine.py.

Same public surface as the reference (engine.py:27-233): ``StoppingCriteria``,
``IterationRecord``, ``CartogramState``, ``RunResult``, ``target_weights``,
``cartographic_error_arrays``, ``CartogramEngine`` (constructor arguments,
attributes, ``run``/``step``/``evaluate``/``current_bdv``) and ``run``.

What changes is where the loop runs.  ``CartogramEngine.run`` uploads the
vertex rows once and executes the whole iteration loop on the GPU (CUDA-graph
captured kernels, device-side stopping rule, csrc/det_api.cu); only the final
state comes back.  ``BatchEngine`` runs many independent cartograms that share
a topology in the same kernel launches (direct-mode time steps, parameter
sweeps) -- the B200-native way to fill 148 SMs.

One-time host work is the reference's: ``densify`` (engine.py:119-120) and the
scalar bookkeeping of ``__init__`` (engine.py:122-139), evaluated with the same
float64 expressions so the target weights are bit-identical.
"""

from __future__ import annotations

import functools
from collections.abc import Sequence as _Sequence
import itertools
import os
import time
from dataclasses import dataclass, field, replace

import numpy as np

from ._context import get_context, region_ranks
from ._lib import PRECISIONS, STOP_BDV, STOP_COLLAPSED, STOP_NAMES, STOP_NEGINDEX
from .errors import NumericError, RasterizationError, RegionCollapsedError
from .geomodel import deferred_rebuild, densify, rebuild, ring_layout
from .raster import LabelTexture, _LazyLabels, rasterize_labels
from .shard import run_sharded

DENSIFY_EDGE_PIXELS = 4.0


@dataclass(frozen=True)
class StoppingCriteria:
    error_threshold: float = 0.01
    stagnation_window: int = 32
    max_iterations: int = 512

    def __post_init__(self):
        if self.error_threshold <= 0 or self.stagnation_window <= 0 or self.max_iterations <= 0:
            raise ValueError("stopping criteria must all be positive")


@dataclass(frozen=True)
class IterationRecord:
    iteration: int
    epsilon: float
    xi: float
    millis: float


def trace_records(tr: np.ndarray, it_off: int = 0) -> tuple:
    """(T, 4) device trace rows -> IterationRecord tuple (built without the frozen-dataclass
    __setattr__ path: one trace per cartogram per run is thousands of records)."""
    new = object.__new__
    out = []
    for it, eps, xi, ms in tr.tolist():
        rec = new(IterationRecord)
        rec.__dict__.update(iteration=int(it) + it_off, epsilon=eps, xi=xi, millis=ms)
        out.append(rec)
    return tuple(out)


class TraceView(_Sequence):
    """A run's trace as a read-only sequence of IterationRecord (engine.py:38-43, 189-195) that
    builds the records on first access: a 296-frame batch returns 59k records, most of them never
    read.  Length is known without building; pickles and compares as the plain tuple."""

    __slots__ = ("_rows", "_off", "_recs")

    def __init__(self, rows: np.ndarray, it_off: int = 0):
        self._rows, self._off, self._recs = rows, it_off, None

    def _mat(self) -> tuple:
        if self._recs is None:
            self._recs = trace_records(self._rows, self._off)
            self._rows = None
        return self._recs

    def __len__(self):
        return len(self._rows) if self._recs is None else len(self._recs)

    def __getitem__(self, i):
        return self._mat()[i]

    def __iter__(self):
        return iter(self._mat())

    def __eq__(self, other):
        if isinstance(other, TraceView):
            other = other._mat()
        return self._mat() == (tuple(other) if isinstance(other, list) else other)

    def __ne__(self, other):
        return not self.__eq__(other)

    __hash__ = None

    def __repr__(self):
        return repr(self._mat())

    def __add__(self, other):
        return self._mat() + tuple(other)

    def __radd__(self, other):
        return tuple(other) + self._mat()

    def __reduce__(self):
        return (tuple, (self._mat(),))


@dataclass(frozen=True)
class CartogramState:
    """Map geometry at one iteration plus the errors measured on it (engine.py:46-57)."""

    mapmodel: object
    iteration: int
    labels: LabelTexture = field(repr=False)
    pixel_counts: np.ndarray
    per_region_error: np.ndarray
    epsilon: float
    xi: float
    clamp_events: int = 0


@dataclass(frozen=True)
class RunResult:
    state: CartogramState
    trace: tuple
    stop_reason: str  # converged | stagnation | max-iterations
    weights_px: np.ndarray
    background_mass: float

    def trace_csv(self) -> str:
        lines = ["iteration,epsilon,xi,millis"]
        for rec in self.trace:
            lines.append(f"{rec.iteration},{rec.epsilon:.9g},{rec.xi:.9g},{rec.millis:.3f}")
        return "\n".join(lines) + "\n"


def target_weights(mapmodel, total_pixels_map: int) -> np.ndarray:
    """engine.py:75-80."""
    s = np.array([float(r.statistic) for r in mapmodel.regions])
    if (s <= 0).any():
        raise ValueError("statistics must be positive")
    return s / s.sum() * total_pixels_map


def cartographic_error_arrays(o: np.ndarray, w: np.ndarray):
    """engine.py:83-85."""
    e = np.abs(o - w) / np.maximum(o, w)
    return e, float(e.mean()), float(e.max())


_load_serial = itertools.count()


class BatchEngine:
    """B independent cartograms of one map topology, run in the same kernel launches.

    ``statistics``: (B, R); ``bdv_multiplier``: scalar or (B,); ``background_mass``:
    None, scalar or (B,); ``start_vertices``: None (the map's vertices for all) or
    (B, N_rows, 2).  Each cartogram follows CartogramEngine semantics exactly.
    """

    def __init__(self, mapmodel, statistics, criteria=None, k: int = 10, bdv_multiplier=1.0,
                 background_mass=None, bdv_mode: str = "fixed-mass", apply_densify: bool = True,
                 start_vertices=None, *, device: int = 0, field_dtype: str = "float64", devices=None,
                 distributed: bool = False):
        if bdv_mode not in ("fixed-mass", "rederive"):
            raise ValueError("bdv_mode must be 'fixed-mass' or 'rederive'")
        # sharded runs (shard.run_sharded): one process per GPU, a contiguous block of the
        # cartograms each, results gathered at the end; set-up here runs on the local device
        self.devices = None if devices is None else [int(d) for d in devices]
        self.distributed = bool(distributed)
        if self.distributed:
            device = int(os.environ.get("LOCAL_RANK", "0")) if self.devices is None else device
        elif self.devices:
            device = self.devices[0]
        if field_dtype not in PRECISIONS:
            raise ValueError("field_dtype must be 'float64', 'mixed' or 'float32'")
        if not (4 <= k <= 13):
            raise ValueError("texture exponent k must be in [4, 13]")
        stats = np.atleast_2d(np.asarray(statistics, dtype=float))
        B = stats.shape[0]
        mult = np.broadcast_to(np.asarray(bdv_multiplier, dtype=float), (B,)).copy()
        if (mult <= 0).any():
            raise ValueError("bdv multiplier must be positive")
        self.criteria = criteria or StoppingCriteria()
        self.k, self.n = k, 1 << k
        self.m = self.n * self.n
        self.bdv_mode = bdv_mode
        self.device, self.field_dtype = device, field_dtype
        if apply_densify:
            mapmodel = densify(mapmodel, DENSIFY_EDGE_PIXELS / self.n)
        self.initial_map = mapmodel
        xy, rs, rr, ids, _ = ring_layout(mapmodel)
        if stats.shape[1] != len(ids):
            raise ValueError("statistics column count must match region count")
        self._xy, self._rs, self._rr, self.region_ids = xy, rs, rr, ids
        self._sizes = np.diff(rs).astype(np.int64)
        self._rank = region_ranks(ids)
        self.B = B
        self.statistics = stats
        self.total_statistic = stats.sum(axis=1)
        if (self.total_statistic <= 0).any():
            raise NumericError("total statistic mass must be positive")
        if start_vertices is not None:
            sv = np.asarray(start_vertices, dtype=np.float64).reshape(B, xy.shape[0], 2)
        else:
            sv = None
        self._start = sv
        self._token = None
        ctx = self._ctx()
        # initial rasterisation of every start geometry (engine.py:128-136)
        cnt0 = np.empty((B, len(ids) + 1), dtype=np.int64)
        lab0 = []
        for b in range(B if sv is not None else 1):
            lab, cnt = ctx.rasterize(b)
            lab0.append(lab)
            cnt0[b] = cnt
        if sv is None:
            cnt0[:] = cnt0[0]
            lab0 = lab0 * B
        for b in range(B):
            empty = [rid for rid, c in zip(ids, cnt0[b, :-1]) if c == 0]
            if empty:
                raise RasterizationError(
                    f"zero-pixel region(s) at resolution {self.n}x{self.n}: {empty} (resolution too low)")
        self._labels0 = [LabelTexture(size=self.n, labels=lab0[b], region_ids=tuple(ids), _counts=cnt0[b])
                         for b in range(B)]
        self.background_pixels0 = cnt0[:, -1].copy()
        self.map_pixels0 = self.m - self.background_pixels0
        self.mean_density0 = self.total_statistic / self.map_pixels0
        bm = None if background_mass is None else np.broadcast_to(np.asarray(background_mass, dtype=float), (B,))
        self.bdv_multiplier = mult
        self.background_mass = np.array([
            float(bm[b]) if bm is not None else mult[b] * self.mean_density0[b] * self.background_pixels0[b]
            for b in range(B)])
        total_mass = self.total_statistic + self.background_mass
        self.weights_px = stats / total_mass[:, None] * self.m
        # page-locked host block for the result vertices of one run_all (setup, like device buffers)
        ctx.pinned.reserve(B * self._xy.shape[0] * 16)

    # -- device context ----------------------------------------------------------
    def _ctx(self):
        ctx = get_context(self.k, self.device, self.field_dtype)
        if getattr(ctx, "_owner_token", None) is not self._token or self._token is None:
            ctx.load_map(self._xy, self._rs, self._rr, self._rank)
            ctx.set_batch(self.statistics, None if self._start is None else self._start)
            self._token = object()
            ctx._owner_token = self._token
        return ctx

    def _params(self):
        mode = 0 if self.bdv_mode == "fixed-mass" else 1
        return [dict(background_mass=float(self.background_mass[b]), bdv_multiplier=float(self.bdv_multiplier[b]),
                     mean_density0=float(self.mean_density0[b]), total_statistic=float(self.total_statistic[b]),
                     bdv_mode=mode) for b in range(self.B)]

    def launch(self, criteria=None):
        """Run every cartogram to its stopping rule on the device; results stay resident."""
        c = criteria or self.criteria
        ctx = self._ctx()
        ctx.set_params(self._params(), self.weights_px)
        ctx.run(c.error_threshold, c.stagnation_window, c.max_iterations)
        return ctx

    def _sharded(self) -> bool:
        return self.distributed or (self.devices is not None and len(self.devices) > 1)

    def run_all(self, criteria=None, iteration_offset: int = 0, clamp_offset: int = 0):
        """List of RunResult (or the CartomorphError/ValueError instance a cartogram raised)."""
        if self._sharded():
            task = functools.partial(_batch_shard, self.initial_map, self.statistics, criteria or self.criteria,
                                     self.k, self.bdv_multiplier, self.background_mass, self.bdv_mode, self._start,
                                     self.field_dtype, iteration_offset, clamp_offset)
            return run_sharded(self.B, task, devices=self.devices, distributed=self.distributed)
        t0 = time.perf_counter()
        ctx = self.launch(criteria)
        t1 = time.perf_counter()
        verts = ctx.pinned.empty((self.B, self._xy.shape[0], 2))
        res = [ctx.result(b) for b in range(self.B)]
        counts, errs, traces = ctx.results_all(verts, max([r.trace_len for r in res] + [0]))
        out = [self._collect(ctx, b, iteration_offset, clamp_offset, verts[b], (res[b], counts[b], errs[b], traces[b]))
               for b in range(self.B)]
        self.last_timing = {"launch_s": t1 - t0, "collect_s": time.perf_counter() - t1,
                            "pinned_misses": ctx.pinned.misses}
        return out

    def _collect(self, ctx, b, it_off=0, cl_off=0, verts_out=None, fetched=None):
        """RunResult of cartogram b; ``fetched`` = (result, counts, errors, trace) already read back
        for every cartogram at once (run_all), else read here."""
        r = ctx.result(b) if fetched is None else fetched[0]
        if r.stop_reason == STOP_COLLAPSED:
            return RegionCollapsedError(self.region_ids[r.collapsed_region], r.iteration + it_off)
        if r.stop_reason == STOP_BDV:
            return ValueError("bdv must be positive")
        if r.stop_reason == STOP_NEGINDEX:
            return ValueError("'list' argument must have no negative elements")
        if fetched is None:
            tr = ctx.trace(b, r.trace_len)
            verts = ctx.vertices(b, verts_out)
            counts = ctx.counts(b)
            rerr = ctx.region_error(b)
        else:
            tr = fetched[3][: r.trace_len]
            verts, counts, rerr = verts_out, fetched[1], fetched[2]
        records = TraceView(np.array(tr, dtype=np.float64), it_off)  # (copy: the batch block is reused)
        clamps = int(r.clamp_events) + (cl_off if r.stop_reason != 2 else 0)
        result_map = deferred_rebuild(self.initial_map, verts, self.statistics[b], self._sizes)
        lazy = _LazyLabels(ctx, b, getattr(ctx, "generation", None), result_map, self.k, self.device)
        labels = LabelTexture(size=self.n, labels=lazy, region_ids=tuple(self.region_ids), _counts=counts)
        state = CartogramState(mapmodel=result_map, iteration=int(r.iteration) + it_off,
                               labels=labels, pixel_counts=counts[:-1].copy(),
                               per_region_error=rerr, epsilon=float(r.epsilon), xi=float(r.xi),
                               clamp_events=clamps)
        return RunResult(state=state, trace=records, stop_reason=STOP_NAMES[r.stop_reason],
                         weights_px=self.weights_px[b].copy(), background_mass=float(self.background_mass[b]))

    def areas(self, b: int = 0) -> np.ndarray:
        """Per-region shoelace areas of cartogram b's last state, on the device (Region.area())."""
        return self._ctx().areas(b)


def _batch_shard(mapmodel, stats, criteria, k, mult, masses, bdv_mode, start, field_dtype, it_off, cl_off, lo, hi,
                 device):
    """Cartograms [lo, hi) of a sharded BatchEngine on `device` (runs in that GPU's process); the
    map is already densified and the background masses are the parent's, so every cartogram is
    exactly the one the unsharded batch would run."""
    be = BatchEngine(mapmodel, stats[lo:hi], criteria=criteria, k=k, bdv_multiplier=mult[lo:hi],
                     background_mass=masses[lo:hi], bdv_mode=bdv_mode, apply_densify=False,
                     start_vertices=None if start is None else start[lo:hi], device=device, field_dtype=field_dtype)
    return be.run_all(criteria, it_off, cl_off)


class CartogramEngine:
    """Owns one run's fixed data: resolution, target weights, background mass (engine.py:87-219)."""

    def __init__(self, mapmodel, criteria: StoppingCriteria | None = None, k: int = 10,
                 bdv_multiplier: float = 1.0, background_mass: float | None = None,
                 bdv_mode: str = "fixed-mass", apply_densify: bool = True, *, device: int = 0,
                 field_dtype: str = "float64"):
        if bdv_mode not in ("fixed-mass", "rederive"):
            raise ValueError("bdv_mode must be 'fixed-mass' or 'rederive'")
        if bdv_multiplier <= 0:
            raise ValueError("bdv multiplier must be positive")
        stats = np.array([float(r.statistic) for r in mapmodel.regions])
        if float(stats.sum()) <= 0:
            raise NumericError("total statistic mass must be positive")
        self._be = BatchEngine(mapmodel, stats[None, :], criteria=criteria, k=k, bdv_multiplier=bdv_multiplier,
                               background_mass=background_mass, bdv_mode=bdv_mode, apply_densify=apply_densify,
                               device=device, field_dtype=field_dtype)
        be = self._be
        self.criteria = be.criteria
        self.k, self.n, self.m = be.k, be.n, be.m
        self.bdv_multiplier = bdv_multiplier
        self.bdv_mode = bdv_mode
        self.initial_map = be.initial_map
        self.statistics = stats
        self.total_statistic = float(be.total_statistic[0])
        self.map_pixels0 = int(be.map_pixels0[0])
        self.background_pixels0 = int(be.background_pixels0[0])
        self.mean_density0 = float(be.mean_density0[0])
        self.background_mass = float(be.background_mass[0])
        self.weights_px = be.weights_px[0]
        self._labels0 = be._labels0[0]

    @property
    def base(self):
        from .displacement import base_mapping

        return base_mapping(self.n)

    def run(self) -> RunResult:
        res = self._be.run_all()[0]
        if isinstance(res, Exception):
            raise res
        return res

    def evaluate(self, mapmodel, iteration: int, labels: LabelTexture | None = None) -> CartogramState:
        """Rasterise a map and measure its cartographic errors (engine.py:143-160)."""
        if labels is None:
            labels = rasterize_labels(mapmodel, self.k, check_collapse=False, device=self._be.device)
            self._be._token = None  # the shared context now holds another map
        counts = labels.pixel_counts()
        if (counts == 0).any():
            raise RegionCollapsedError(labels.region_ids[int(np.argmin(counts))], iteration)
        per_region, eps, xi = cartographic_error_arrays(counts.astype(float), self.weights_px)
        return CartogramState(mapmodel=mapmodel, iteration=iteration, labels=labels, pixel_counts=counts,
                              per_region_error=per_region, epsilon=eps, xi=xi)

    def current_bdv(self, labels: LabelTexture) -> float:
        """engine.py:162-168."""
        n_bg = labels.background_count()
        if n_bg == 0:
            return self.mean_density0 * self.bdv_multiplier
        if self.bdv_mode == "fixed-mass":
            return self.background_mass / n_bg
        return self.bdv_multiplier * self.total_statistic / labels.map_pixel_count()

    def step(self, state: CartogramState) -> CartogramState:
        """One deformation on the GPU (engine.py:170-180): one device iteration from state's vertices."""
        be = BatchEngine.__new__(BatchEngine)
        be.__dict__.update(self._be.__dict__)
        verts = np.asarray(state.mapmodel.vertex_array(), dtype=np.float64)
        be._start = verts[None]
        be._token = None
        try:
            be._ctx()
        except Exception:
            # vertex rows no longer share positions the way the initial map did: reload topology
            be._xy = verts
            be._token = None
            be._start = None
            be._ctx()
        res = be.run_all(StoppingCriteria(error_threshold=1e-300, stagnation_window=1 << 30, max_iterations=1),
                         iteration_offset=state.iteration, clamp_offset=state.clamp_events)[0]
        self._be._token = None
        if isinstance(res, Exception):
            raise res
        st = res.state
        return replace(st, mapmodel=rebuild(state.mapmodel, st.mapmodel.vertex_array()))


def run(mapmodel, criteria: StoppingCriteria | None = None, bdv_multiplier: float = 1.0, k: int = 10,
        **kwargs) -> RunResult:
    """Run the full iterative algorithm on a normalised map (engine.py:222-233)."""
    return CartogramEngine(mapmodel, criteria=criteria, k=k, bdv_multiplier=bdv_multiplier, **kwargs).run()
