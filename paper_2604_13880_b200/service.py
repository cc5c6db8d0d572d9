"""GPU frame computation for the steering service -- SURVEY.md §8f #4.

Drop-in for the body of ``cartomorph/service.py:_compute_frame`` (service.py:181-241): one
frame = engine run (the DET loop on the device) + quality report (device metric kernels) +
GeoJSON.  The HTTP layer, session cache and scheduling of the reference service are out of
scope; a maintainer swaps this call in for the frame body.

Per-session device state: the service runs one worker thread per session
(service.py:_worker_loop), and device contexts are cached per thread (``_context.py``: one
CUDA stream and one set of device buffers per thread, device and texture size), so every
session computes on its own stream without sharing buffers with another session.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

from .engine import CartogramEngine, StoppingCriteria
from .errors import CartomorphError
from .geomodel import to_geojson
from .metrics import full_report


@dataclass
class ComputedFrame:
    """service.py:73-82."""

    mapmodel: object
    geojson: dict | None
    report: dict | None
    background_mass: float
    area_fraction: float | None
    wall_ms: float
    stop_reason: str | None = None
    error: str | None = None


def compute_frame(start_geometry, base_map, stats_t, mass: float, fraction: float | None, params, *,
                  device: int = 0, field_dtype: str = "float64") -> ComputedFrame:
    """One session frame as service.py:202-236 computes it.

    ``params`` carries the session parameters the reference reads (``threshold``,
    ``stagnation``, ``max_iter``, ``texture_k``, ``hamming_k``); ``start_geometry`` is the
    base map (direct) or the previous frame's map (cumulative).
    """
    began = time.perf_counter()
    try:
        start_map = start_geometry.with_statistics(stats_t)
        engine = CartogramEngine(start_map, criteria=StoppingCriteria(params.threshold, params.stagnation,
                                                                      params.max_iter),
                                 k=params.texture_k, background_mass=mass, apply_densify=False, device=device,
                                 field_dtype=field_dtype)
        result = engine.run()
        wall_ms = (time.perf_counter() - began) * 1e3
        carto = result.state.mapmodel
        weights = stats_t / (float(stats_t.sum()) + mass)
        report = full_report(base_map.with_statistics(stats_t), carto, weights=weights, raster_k=params.hamming_k,
                             wall_ms=wall_ms, device=device)
        return ComputedFrame(mapmodel=carto, geojson=json.loads(to_geojson(carto, report.per_region)),
                             report=report.to_dict(), background_mass=mass, area_fraction=fraction,
                             wall_ms=wall_ms, stop_reason=result.stop_reason)
    except CartomorphError as exc:
        return ComputedFrame(None, None, None, mass, fraction, (time.perf_counter() - began) * 1e3, error=str(exc))
