"""Quality measures for (original map, cartogram) pairs -- drop-in for cartomorph/metrics.py.

The per-frame report of the temporal runs (temporal.py:203-209) on the GPU:

* shape distortion (metrics.py:82-135): ``k_shape`` rescales, rasterises and correlates every
  region of every frame in one launch (one CTA per (region, frame)); the best overlap is an exact
  integer correlation over bit rows, so the Hamming values equal the reference's bit for bit;
* region areas and barycenters (geomodel.py:63-77) come out of the same launch, with numpy's
  summation order, so the cartographic errors are bit-identical as well;
* adjacency detection (geomodel.py:380-415): ``k_adj_*`` (cell keys, radix sort, 3x3 probes);
* relative position error (metrics.py:138-162): ``k_poserr`` over all barycenter pairs of all
  frames (summation order differs from the reference's Python loop: agreement to ~1e-13 relative).

Cartographic errors and topology distortion are R-vector / set arithmetic and stay on the host,
written exactly as the reference writes them.  Error types and messages follow the reference.
"""

from __future__ import annotations

import json
import logging
from dataclasses import dataclass, field

import numpy as np

from ._context import get_context
from .errors import CartomorphError, NumericError, RasterizationError
from .geomodel import ring_layout

log = logging.getLogger(__name__)

DEFAULT_HAMMING_K = 7  # 128 x 128 shape rasters
DEFAULT_ADJACENCY_EPSILON = 0.5 / 1024

_ST_AREA_A, _ST_AREA_B, _ST_EMPTY, _ST_NEG_A, _ST_NEG_B = 1, 2, 3, 4, 5


def _ctx(device: int):
    return get_context(4, device)  # metric kernels carry their own layouts; no loaded map is used


def cartographic_errors(o: np.ndarray, w: np.ndarray):
    """Per-region |o - w| / max(o, w), its mean (epsilon) and max (xi) (metrics.py:29-37)."""
    o = np.asarray(o, dtype=float)
    w = np.asarray(w, dtype=float)
    if (o <= 0).any() or (w <= 0).any():
        raise NumericError("cartographic error needs positive actual and desired areas")
    per_region = np.abs(o - w) / np.maximum(o, w)
    return float(per_region.mean()), float(per_region.max()), per_region


def topology_distortion(edges_map, edges_carto) -> float:
    """1 - Jaccard similarity of two adjacency sets; 0 when both are empty (metrics.py:40-47)."""
    em = {tuple(sorted(e)) for e in edges_map}
    ec = {tuple(sorted(e)) for e in edges_carto}
    union = em | ec
    if not union:
        return 0.0
    return 1.0 - len(em & ec) / len(union)


def _check_same_regions(a, b) -> None:
    if [r.region_id for r in a.regions] != [r.region_id for r in b.regions]:
        raise ValueError("map and cartogram must list the same regions in the same order")


def _layout(mapmodel):
    xy, rs, rr, ids, _ = ring_layout(mapmodel)
    return (xy, rs, rr, len(ids)), ids


def _raise_status(code: int) -> None:
    if code in (_ST_AREA_A, _ST_AREA_B):
        raise NumericError("region with non-positive area")
    if code == _ST_EMPTY:
        raise RasterizationError("shape rasterized to zero pixels in Hamming grid")
    if code in (_ST_NEG_A, _ST_NEG_B):
        raise ValueError("'list' argument must have no negative elements")  # np.bincount, raster.py:86-89


def _shapes(layout_a, layout_b, raster_k: int, rescale: bool, device: int):
    return _ctx(device).shape_metrics(layout_a, layout_b, raster_k, rescale)


def hamming_distance(rings_m, rings_c, raster_k: int = DEFAULT_HAMMING_K, rescale: bool = True, *,
                     device: int = 0) -> float:
    """Normalized symmetric difference of two shapes minimised over shifts (metrics.py:80-118)."""
    def one(rings):
        rings = [np.asarray(r, dtype=float) for r in rings]
        rs = np.concatenate([[0], np.cumsum([r.shape[0] for r in rings])]).astype(np.int32)
        return np.vstack(rings), rs, np.zeros(len(rings), dtype=np.int32), 1

    ham, _, _, _, st = _shapes(one(rings_m), one(rings_c), raster_k, rescale, device)
    _raise_status(int(st[0, 0]))
    return float(ham[0, 0])


def shape_distortion(mapmodel, carto, raster_k: int = DEFAULT_HAMMING_K, rescale: bool = True, *, device: int = 0):
    """Per-region Hamming shape distortion plus (average, maximum) (metrics.py:121-135)."""
    _check_same_regions(mapmodel, carto)
    la, _ = _layout(mapmodel)
    lb, _ = _layout(carto)
    ham, _, _, _, st = _shapes(la, lb, raster_k, rescale, device)
    bad = np.flatnonzero(st[0])
    if bad.size:
        _raise_status(int(st[0, bad[0]]))
    values = ham[0]
    return values, float(values.mean()), float(values.max())


def _position_errors(cent_m, cent_c, device: int) -> np.ndarray:
    count = cent_m.shape[0]
    sums, degenerate = _ctx(device).position_error(cent_m, cent_c)
    for d in degenerate:
        if d:
            log.info("relative_position_error: %d degenerate barycenter pairs contributed 0", int(d))
    return sums / (np.pi * count * (count - 1))


def relative_position_error(mapmodel, carto, *, device: int = 0) -> float:
    """Mean |angle change| of pairwise barycenter vectors, normalized by pi (metrics.py:138-162)."""
    _check_same_regions(mapmodel, carto)
    if len(mapmodel.regions) < 2:
        raise NumericError("relative position error needs at least two regions")
    la, _ = _layout(mapmodel)
    lb, _ = _layout(carto)
    _, _, ca, cb, _ = _shapes(la, lb, 0, False, device)  # raster_k 0: barycenters only
    return float(_position_errors(ca, cb, device)[0])


def _adjacent_pairs(xy, ring_start, ring_region, n_regions, epsilon, device):
    """(frame, a, b) triples for one or more vertex sets of one layout."""
    if epsilon <= 0:
        raise ValueError("epsilon must be positive")
    row_region = np.repeat(np.asarray(ring_region, dtype=np.int32), np.diff(ring_start))
    return _ctx(device).adjacency(xy, row_region, n_regions, epsilon)


def detect_adjacencies(mapmodel, epsilon: float, *, device: int = 0) -> frozenset:
    """Region pairs sharing >= 2 epsilon-cells of vertices (geomodel.py:380-415), on the GPU."""
    (xy, rs, rr, r), ids = _layout(mapmodel)
    pairs = _adjacent_pairs(xy, rs, rr, r, epsilon, device)
    return frozenset(tuple(sorted((ids[a], ids[b]))) for _, a, b in pairs.tolist())


def _edge_keys(edges, ids):
    """Id-pair set -> sorted unique int64 keys min*R + max over region indices (None if an id is unknown)."""
    pos = {rid: i for i, rid in enumerate(ids)}
    try:
        idx = np.array([(pos[a], pos[b]) for a, b in edges], dtype=np.int64).reshape(-1, 2)
    except KeyError:
        return None
    r = len(ids)
    return np.unique(idx.min(axis=1) * r + idx.max(axis=1))


def _tau(keys_m, keys_c) -> float:
    """topology_distortion on key arrays: 1 - |em & ec| / |em | ec| (metrics.py:40-47)."""
    inter = np.intersect1d(keys_m, keys_c, assume_unique=True).size
    union = keys_m.size + keys_c.size - inter
    if not union:
        return 0.0
    return 1.0 - inter / union


@dataclass
class QualityReport:
    """All six measures of one map/cartogram pair (metrics.py:165-210)."""

    epsilon: float
    xi: float
    tau: float
    hamming_avg: float
    hamming_max: float
    position_error: float
    per_region: dict = field(default_factory=dict)
    wall_ms: float | None = None

    def to_dict(self) -> dict:
        return {
            "epsilon": self.epsilon,
            "xi": self.xi,
            "tau": self.tau,
            "hamming_avg": self.hamming_avg,
            "hamming_max": self.hamming_max,
            "position_error": self.position_error,
            "per_region": self.per_region,
            "wall_ms": self.wall_ms,
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2)

    @classmethod
    def from_dict(cls, data: dict) -> "QualityReport":
        return cls(**data)

    def to_csv(self) -> str:
        lines = ["region,cartographic_error,shape_distortion"]
        for rid, vals in self.per_region.items():
            lines.append(f"{rid},{vals['cartographic_error']:.9g},{vals['shape_distortion']:.9g}")
        lines.append(
            f"_aggregate,epsilon={self.epsilon:.9g};xi={self.xi:.9g};tau={self.tau:.9g},"
            f"avg={self.hamming_avg:.9g};max={self.hamming_max:.9g};R={self.position_error:.9g}"
        )
        return "\n".join(lines) + "\n"


class _FrameMetrics:
    """Device results for F cartogram frames that share one vertex layout."""

    def __init__(self, mapmodel, carto_layout, carto_xy, raster_k, rescale, epsilon, device):
        la, self.ids = _layout(mapmodel)
        xy_b, rs_b, rr_b, r = carto_layout
        self.carto_layout = carto_layout
        self.carto_xy = np.asarray(carto_xy, dtype=float).reshape(-1, int(rs_b[-1]), 2)
        self.ham, self.area, self.ca, self.cb, self.status = _shapes(
            la, (self.carto_xy, rs_b, rr_b, r), raster_k, rescale, device)
        self.pos = _position_errors(self.ca, self.cb, device) if r >= 2 else None
        self.mapmodel, self.map_layout, self.epsilon, self.device = mapmodel, la, epsilon, device
        self._adj = self._map_keys = None

    def carto_keys(self, f: int) -> np.ndarray:
        """Adjacency keys of frame f; all frames are detected in one device pass on first use."""
        if self._adj is None:
            _, rs_b, rr_b, r = self.carto_layout
            t = _adjacent_pairs(self.carto_xy, rs_b, rr_b, r, self.epsilon, self.device).astype(np.int64)
            keys = t[:, 1] * r + t[:, 2]
            cuts = np.searchsorted(t[:, 0], np.arange(self.carto_xy.shape[0] + 1))
            self._adj = [keys[cuts[i]:cuts[i + 1]] for i in range(self.carto_xy.shape[0])]
        return self._adj[f]

    def map_keys(self):
        """mapmodel.adjacency or detect_adjacencies(mapmodel) (metrics.py:231), as keys."""
        if self._map_keys is None:
            adj = self.mapmodel.adjacency
            keys = _edge_keys(adj, self.ids) if adj else None
            if keys is None and not adj:
                xy, rs, rr, r = self.map_layout
                t = _adjacent_pairs(xy, rs, rr, r, self.epsilon, self.device).astype(np.int64)
                keys = t[:, 1] * r + t[:, 2]
            self._map_keys = keys if keys is not None else adj
        return self._map_keys


def _assemble(mapmodel, fm: _FrameMetrics, f: int, weights, wall_ms):
    """Reference order (metrics.py:225-247): errors, topology, shapes, position; first raise wins."""
    o = fm.area[f]
    if weights is None:
        s = np.array([r.statistic for r in mapmodel.regions], dtype=float)
        weights = s / s.sum() * o.sum()
    eps, xi, per_cart = cartographic_errors(o, weights)
    km = fm.map_keys()
    kc = fm.carto_keys(f)
    if isinstance(km, np.ndarray):
        tau = _tau(km, kc)
    else:  # an adjacency set naming ids outside the map: set arithmetic on id pairs
        r = len(fm.ids)
        tau = topology_distortion(km, {(fm.ids[k // r], fm.ids[k % r]) for k in kc.tolist()})
    bad = np.flatnonzero(fm.status[f])
    if bad.size:
        _raise_status(int(fm.status[f, bad[0]]))
    per_shape = fm.ham[f]
    if fm.pos is None:
        raise NumericError("relative position error needs at least two regions")
    per_region = {rid: {"cartographic_error": ce, "shape_distortion": sd}
                  for rid, ce, sd in zip(fm.ids, per_cart.tolist(), per_shape.tolist())}
    return QualityReport(epsilon=eps, xi=xi, tau=tau, hamming_avg=float(per_shape.mean()),
                         hamming_max=float(per_shape.max()), position_error=float(fm.pos[f]),
                         per_region=per_region, wall_ms=wall_ms)


def full_report(mapmodel, carto, weights: np.ndarray | None = None, raster_k: int = DEFAULT_HAMMING_K,
                adjacency_epsilon: float = DEFAULT_ADJACENCY_EPSILON, rescale_shapes: bool = True,
                wall_ms: float | None = None, *, device: int = 0) -> QualityReport:
    """All six measures for a map/cartogram pair (metrics.py:213-260)."""
    _check_same_regions(mapmodel, carto)
    lb, _ = _layout(carto)
    fm = _FrameMetrics(mapmodel, lb, lb[0], raster_k, rescale_shapes, adjacency_epsilon, device)
    return _assemble(mapmodel, fm, 0, weights, wall_ms)


def frame_reports(base_map, carto_layout, carto_xy, statistics, weights, raster_k: int = DEFAULT_HAMMING_K,
                  wall_ms=None, adjacency_epsilon: float = DEFAULT_ADJACENCY_EPSILON, *, device: int = 0):
    """``full_report(base_map.with_statistics(s_t), carto_t, weights_t)`` for F frames in one pass.

    ``carto_xy`` is (F, rows, 2) in ``carto_layout``; one launch each for the shapes, the
    adjacencies and the position errors covers all frames.  Returns per frame a QualityReport, or
    the CartomorphError the reference would have raised for it.
    """
    carto_xy = np.asarray(carto_xy, dtype=float)
    n_frames = carto_xy.shape[0]
    if n_frames == 0:
        return []
    fm = _FrameMetrics(base_map, carto_layout, carto_xy, raster_k, True, adjacency_epsilon, device)
    out = []
    for f in range(n_frames):
        w = None
        if weights is not None:
            w = np.asarray(weights[f], dtype=float)
        else:
            s = np.asarray(statistics[f], dtype=float)
            w = s / s.sum() * fm.area[f].sum()
        try:
            out.append(_assemble(base_map, fm, f, w, None if wall_ms is None else wall_ms[f]))
        except CartomorphError as exc:
            out.append(exc)
    return out
