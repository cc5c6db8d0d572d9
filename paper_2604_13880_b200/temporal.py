"""Time-varying cartogram sequences -- drop-in for cartomorph/temporal.py.

Transition modes (temporal.py:162-290):

* ``run_direct``: every frame starts from the densified base map.  Frames are
  independent, so all T frames run as ONE batch on the GPU (``BatchEngine``:
  every kernel launch covers all frames) -- the B200-native replacement for the
  reference's frame-by-frame loop.
* ``run_cumulative``: frame t starts from frame t-1's output; frames run one
  after another, each fully device-resident.

The background-mass schedule (temporal.py:83-102, 151-159) and the per-frame
error capture (temporal.py:231-244) follow the reference.  Every successful
frame carries its quality report (``full_report``, metrics.py:213-260,
temporal.py:203-209) computed on the GPU for all frames at once
(``metrics.frame_reports``), and the shape-distortion watchdog
(temporal.py:219-228) is evaluated from it.
"""

from __future__ import annotations

import functools
import logging
import time
from dataclasses import dataclass, field

import numpy as np

from ._context import get_context, region_ranks
from ._lib import DET_E_RASTER, STOP_BDV, STOP_COLLAPSED, STOP_NAMES, STOP_NEGINDEX
from .engine import DENSIFY_EDGE_PIXELS, BatchEngine, CartogramState, RunResult, StoppingCriteria, trace_records
from .errors import CartomorphError, IngestionError, RasterizationError, RegionCollapsedError
from .geomodel import deferred_rebuild, densify, ring_layout
from .metrics import frame_reports
from .raster import LabelTexture, _LazyLabels, rasterize_labels
from .shard import run_sharded

log = logging.getLogger(__name__)

DEFAULT_WATCHDOG_CEILING = 0.5
DEFAULT_FRAMES_PER_STEP = 10


@dataclass(frozen=True)
class TimeSeriesDataset:
    """A map plus one positive statistic vector per time step (temporal.py:36-63)."""

    mapmodel: object
    times: tuple
    statistics: np.ndarray

    def __post_init__(self):
        stats = np.asarray(self.statistics, dtype=float)
        if stats.ndim != 2 or stats.shape[0] != len(self.times):
            raise IngestionError("statistics must be (time, region) shaped")
        if stats.shape[1] != len(self.mapmodel.regions):
            raise IngestionError("statistics column count must match region count")
        if (stats <= 0).any() or not np.isfinite(stats).all():
            raise IngestionError("all statistics must be positive and finite")
        object.__setattr__(self, "statistics", stats)

    @property
    def step_count(self) -> int:
        return len(self.times)

    def totals(self) -> np.ndarray:
        return self.statistics.sum(axis=1)

    def map_at(self, t: int):
        return self.mapmodel.with_statistics(self.statistics[t])


@dataclass(frozen=True)
class AreaFractionPolicy:
    a_min: float
    a_max: float
    window: tuple | None = None

    def __post_init__(self):
        if not (0.0 < self.a_min < self.a_max < 1.0):
            raise ValueError("need 0 < a_min < a_max < 1")
        if self.window is not None and self.window[0] > self.window[1]:
            raise ValueError("window must be ordered")


def background_mass_schedule(dataset: TimeSeriesDataset, policy: AreaFractionPolicy):
    """Per-time (M_b, A_i) from the area-fraction schedule (temporal.py:83-102)."""
    totals = dataset.totals()
    t0, t1 = policy.window or (0, dataset.step_count - 1)
    if not (0 <= t0 <= t1 < dataset.step_count):
        raise ValueError("window outside dataset range")
    m_min = float(totals[t0 : t1 + 1].min())
    m_max = float(totals[t0 : t1 + 1].max())
    if m_max == m_min:
        log.info("constant mass over the window; using w = 1 for all time steps")
        w = np.ones_like(totals)
    else:
        w = np.clip((totals - m_min) / (m_max - m_min), 0.0, 1.0)
    area_fraction = (1.0 - w) * policy.a_min + w * policy.a_max
    return totals * (1.0 - area_fraction) / area_fraction, area_fraction


@dataclass
class Frame:
    time_index: int
    time: str
    mapmodel: object
    result: RunResult | None
    report: object
    background_mass: float
    area_fraction: float | None
    wall_ms: float
    watchdog: bool = False
    error: str | None = None


@dataclass
class FrameSequence:
    strategy: str
    dataset: TimeSeriesDataset
    base_map: object
    frames: list = field(default_factory=list)

    def series(self) -> dict:
        totals = self.dataset.totals()
        return {
            "times": list(self.dataset.times),
            "M_i": [float(v) for v in totals],
            "M_b": [f.background_mass for f in self.frames],
            "A_i": [f.area_fraction if f.area_fraction is not None else float(t / (t + f.background_mass))
                    for f, t in zip(self.frames, totals)],
            "epsilon": [f.report.epsilon if f.report else None for f in self.frames],
            "xi": [f.report.xi if f.report else None for f in self.frames],
            "hamming_avg": [f.report.hamming_avg if f.report else None for f in self.frames],
            "position_error": [f.report.position_error if f.report else None for f in self.frames],
            "wall_ms": [f.wall_ms for f in self.frames],
            "watchdog": [f.watchdog for f in self.frames],
            "errors": [f.error for f in self.frames],
        }


def _default_background_masses(dataset: TimeSeriesDataset, k: int, bdv_multiplier: float):
    """temporal.py:151-159: the original map's pixel split, for both strategies (GPU raster)."""
    labels = rasterize_labels(dataset.mapmodel, k)
    n_map = labels.map_pixel_count()
    n_bg = labels.background_count()
    return bdv_multiplier * dataset.totals() / n_map * n_bg


def _masses(dataset, policy, k, bdv_multiplier):
    if policy is None:
        return _default_background_masses(dataset, k, bdv_multiplier), [None] * dataset.step_count
    return background_mass_schedule(dataset, policy)


def run_direct(dataset: TimeSeriesDataset, criteria: StoppingCriteria | None = None,
               policy: AreaFractionPolicy | None = None, k: int = 10, bdv_multiplier: float = 1.0,
               watchdog_ceiling: float = DEFAULT_WATCHDOG_CEILING, report_raster_k: int = 7, *,
               device: int = 0, field_dtype: str = "float64", devices=None,
               distributed: bool = False) -> FrameSequence:
    """Every frame deformed independently from the original map -- all frames in one GPU batch.

    ``devices=[...]`` shards the frames over one worker process per GPU, ``distributed=True`` over
    the ranks of an initialised torch.distributed job (shard.run_sharded); the frames are
    independent, so the only exchange is the final gather."""
    criteria = criteria or StoppingCriteria()
    masses, fractions = _masses(dataset, policy, k, bdv_multiplier)
    base_map = densify(dataset.mapmodel, DENSIFY_EDGE_PIXELS / (1 << k))
    seq = FrameSequence(strategy="direct", dataset=dataset, base_map=base_map)
    task = functools.partial(_direct_block, base_map, dataset.times, dataset.statistics, criteria,
                             np.asarray(masses, dtype=float), fractions, k, watchdog_ceiling, report_raster_k,
                             field_dtype)
    if devices is None and not distributed:
        seq.frames.extend(task(0, dataset.step_count, device))
    else:
        seq.frames.extend(run_sharded(dataset.step_count, task, devices=devices, distributed=distributed))
    return seq


def _direct_block(base_map, times, statistics, criteria, masses, fractions, k, watchdog_ceiling, report_raster_k,
                  field_dtype, lo, hi, device):
    """Frames [lo, hi) of a direct-mode sequence as one device batch on `device`, with their
    reports (temporal.py:185-246 per frame)."""
    began = time.perf_counter()
    idx = list(range(lo, hi))
    try:
        # engines are built with the reference's per-frame arguments (temporal.py:190-196):
        # bdv_multiplier defaults to 1.0 there, the masses carry the user's multiplier
        be = BatchEngine(base_map, statistics[lo:hi], criteria=criteria, k=k, background_mass=masses[lo:hi],
                         apply_densify=False, device=device, field_dtype=field_dtype)
        results = be.run_all()
    except CartomorphError as exc:  # a start-map problem fails every frame alike
        results = [exc] * len(idx)
    wall_ms = (time.perf_counter() - began) * 1e3 / max(len(idx), 1)
    ok = [i for i, res in enumerate(results) if not isinstance(res, Exception)]
    reports = _reports(base_map, statistics, masses, [results[i].state.mapmodel for i in ok], [lo + i for i in ok],
                       report_raster_k, wall_ms, device)
    rep_of = dict(zip(ok, reports))
    frames = []
    for i, res in enumerate(results):
        t = lo + i
        frac = None if fractions[t] is None else float(fractions[t])
        if isinstance(res, CartomorphError):
            log.error("direct frame %d failed: %s", t, res)
            frames.append(Frame(t, times[t], None, None, None, float(masses[t]), frac, wall_ms, error=str(res)))
        elif isinstance(res, Exception):
            raise res
        else:
            frames.append(_frame("direct", t, times, res, rep_of[i], float(masses[t]), frac, wall_ms,
                                 watchdog_ceiling))
    return frames


def _reports(base_map, statistics, masses, cartos, times, raster_k, wall_ms, device):
    """full_report of each successful frame (temporal.py:200-209), all frames in one GPU pass."""
    if not times:
        return []
    _, rs, rr, ids, _ = ring_layout(base_map)
    xy = np.stack([c.vertex_array() for c in cartos])
    stats = statistics[times]
    weights = [statistics[t] / float(statistics[t].sum() + masses[t]) for t in times]
    return frame_reports(base_map, (None, rs, rr, len(ids)), xy, stats, weights, raster_k,
                         [wall_ms] * len(times), device=device)


def _frame(strategy, t, times, res, report, mb, frac, wall_ms, ceiling):
    """A successful deformation plus its report; a report error fails the frame (temporal.py:231-244)."""
    if isinstance(report, Exception):
        log.error("%s frame %d failed: %s", strategy, t, report)
        return Frame(t, times[t], None, None, None, mb, frac, wall_ms, error=str(report))
    fr = Frame(t, times[t], res.state.mapmodel, res, report, mb, frac, wall_ms,
               watchdog=report.hamming_avg > ceiling)
    if fr.watchdog:
        log.warning("%s frame %d: average shape distortion %.3f exceeds ceiling %.3f", strategy, t,
                    report.hamming_avg, ceiling)
    return fr


def run_cumulative(dataset: TimeSeriesDataset, criteria: StoppingCriteria | None = None,
                   policy: AreaFractionPolicy | None = None, k: int = 10, bdv_multiplier: float = 1.0,
                   watchdog_ceiling: float = DEFAULT_WATCHDOG_CEILING, report_raster_k: int = 7, *,
                   device: int = 0, field_dtype: str = "float64") -> FrameSequence:
    """Each frame starts from the previous frame's deformed map (temporal.py:271-290).

    The whole chain stays on the GPU (``det_run_chain``): frame t+1 starts from frame t's
    device-resident vertices; per frame only the results come back.
    """
    criteria = criteria or StoppingCriteria()
    masses, fractions = _masses(dataset, policy, k, bdv_multiplier)
    base_map = densify(dataset.mapmodel, DENSIFY_EDGE_PIXELS / (1 << k))
    seq = FrameSequence(strategy="cumulative", dataset=dataset, base_map=base_map)
    xy, rs, rr, ids, _ = ring_layout(base_map)
    ctx = get_context(k, device, field_dtype)
    ctx.load_map(xy, rs, rr, region_ranks(ids))
    totals = np.array([float(s.sum()) for s in dataset.statistics])  # engine.py:123 (numpy sum)
    masses = np.asarray(masses, dtype=float)
    n = 1 << k
    sizes = np.diff(rs).astype(np.int64)
    frames = [None] * dataset.step_count
    start, start_xy = 0, None
    while start < dataset.step_count:
        # the chain runs on the device from `start`; a frame whose report fails keeps the previous
        # geometry (temporal.py:229-230 is skipped), so the chain restarts after it
        ctx.set_batch(dataset.statistics[start : start + 1], xy=start_xy)
        began = time.perf_counter()
        out_xy, res, cnt, trace = ctx.run_chain(dataset.statistics[start:], totals[start:], masses[start:],
                                                criteria.error_threshold, criteria.stagnation_window,
                                                criteria.max_iterations)
        wall_ms = (time.perf_counter() - began) * 1e3 / max(dataset.step_count - start, 1)
        results = {}
        for i, r in enumerate(res):
            t = start + i
            err = None
            if r.status == DET_E_RASTER:
                empty = [rid for rid, c in zip(ids, cnt[i, :-1]) if c == 0]
                err = RasterizationError(f"zero-pixel region(s) at resolution {n}x{n}: {empty} (resolution too low)")
            elif r.stop_reason == STOP_COLLAPSED:
                err = RegionCollapsedError(ids[r.collapsed_region], r.iteration)
            elif r.stop_reason in (STOP_BDV, STOP_NEGINDEX):
                raise ValueError("bdv must be positive" if r.stop_reason == STOP_BDV
                                 else "'list' argument must have no negative elements")
            if err is not None:
                results[t] = err
                continue
            results[t] = _chain_result(ctx, base_map, ids, sizes, dataset.statistics[t], totals[t], masses[t],
                                       out_xy[i], r, cnt[i], trace[i], n, k, device)
        ok = [t for t in sorted(results) if not isinstance(results[t], Exception)]
        reports = _reports(base_map, dataset.statistics, masses, [results[t].state.mapmodel for t in ok], ok,
                           report_raster_k,
                           wall_ms, device)
        rep_of = dict(zip(ok, reports))
        restart = None
        for t in range(start, dataset.step_count):
            frac = None if fractions[t] is None else float(fractions[t])
            mb = float(masses[t])
            res_t = results[t]
            if isinstance(res_t, Exception):
                log.error("cumulative frame %d failed: %s", t, res_t)
                frames[t] = Frame(t, dataset.times[t], None, None, None, mb, frac, wall_ms, error=str(res_t))
                continue
            frames[t] = _frame("cumulative", t, dataset.times, res_t, rep_of[t], mb, frac, wall_ms, watchdog_ceiling)
            if frames[t].error is not None:
                restart = t
                break
            start_xy = out_xy[t - start]
        if restart is None:
            break
        start = restart + 1
    seq.frames.extend(frames)
    return seq


def _chain_result(ctx, base_map, ids, sizes, stats_t, total_t, mb, xy_t, r, counts, trace_t, n, k, device):
    carto = deferred_rebuild(base_map, xy_t, stats_t, sizes)
    total_mass = float(total_t) + float(mb)
    weights = stats_t / total_mass * (n * n)
    records = trace_records(trace_t[: r.trace_len])
    labels = LabelTexture(size=n, labels=_LazyLabels(ctx, 0, -1, carto, k, device),
                          region_ids=tuple(ids), _counts=counts)
    per_region = np.abs(counts[:-1] - weights) / np.maximum(counts[:-1].astype(float), weights)
    state = CartogramState(mapmodel=carto, iteration=int(r.iteration), labels=labels,
                           pixel_counts=counts[:-1].copy(), per_region_error=per_region,
                           epsilon=float(r.epsilon), xi=float(r.xi), clamp_events=int(r.clamp_events))
    return RunResult(state=state, trace=records, stop_reason=STOP_NAMES[r.stop_reason], weights_px=weights,
                     background_mass=float(mb))


def _blend(a, b, fracs, device=0):
    """Per-vertex + per-statistic linear blends of two frames on the GPU (k_interpolate)."""
    va, vb = a.vertex_array(), b.vertex_array()
    if va.shape != vb.shape:
        raise ValueError("vertex-count mismatch between frames")
    sa = np.array([r.statistic for r in a.regions], dtype=float)
    sb = np.array([r.statistic for r in b.regions], dtype=float)
    ctx = get_context(4, device)
    out = ctx.interpolate(np.concatenate([va.ravel(), sa]), np.concatenate([vb.ravel(), sb]), fracs)
    nv = va.size
    sizes = np.array([np.asarray(r).shape[0] for reg in a.regions for r in reg.rings], dtype=np.int64)
    return [deferred_rebuild(a, o[:nv].reshape(-1, 2), o[nv:], sizes) for o in out]


def interpolate_vertices(a, b, fraction: float, device: int = 0):
    """Linear per-vertex blend of two frames with identical vertex layout (temporal.py:293-302)."""
    return _blend(a, b, np.array([float(fraction)]), device)[0]


def interpolate_frames(seq: FrameSequence, frames_per_step: int = DEFAULT_FRAMES_PER_STEP, device: int = 0):
    """Dense animation frames (temporal.py:305-326); all blends of a step pair in one GPU launch."""
    if frames_per_step < 1:
        raise ValueError("frames_per_step must be >= 1")
    out = []
    frames = list(seq.frames)
    for idx, cur in enumerate(frames):
        if cur.mapmodel is None:
            continue
        out.append((cur.time, cur.mapmodel))
        if idx + 1 >= len(frames) or frames[idx + 1].mapmodel is None or frames_per_step == 1:
            continue
        nxt = frames[idx + 1]
        us = [sub / frames_per_step for sub in range(1, frames_per_step)]
        for u, mm in zip(us, _blend(cur.mapmodel, nxt.mapmodel, np.array(us), device)):
            out.append((f"{cur.time}+{u:.3f}", mm))
    return out
