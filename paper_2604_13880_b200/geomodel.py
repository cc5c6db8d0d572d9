"""Host-side polygon map model for the DET path.

Mirrors the parts of ``cartomorph.geomodel`` that sit on or next to the hot
path (``/root/reference/pkg/src/cartomorph/geomodel.py``):

* :class:`Region` / :class:`MapModel` (geomodel.py:50-145) -- same field names,
  same region -> ring -> vertex flattening order in :meth:`MapModel.vertex_array`
  (geomodel.py:128-130), so vertex arrays are interchangeable with the
  reference's.  Any object exposing ``regions`` whose items expose
  ``region_id``, ``name``, ``rings`` and ``statistic`` (a reference
  ``cartomorph.MapModel`` included) is accepted by the engine.
* :func:`densify` (geomodel.py:353-377) -- one-time host pre-processing at
  engine construction, float64, same formula as the reference so the vertex
  rows fed to the GPU are identical.
* :func:`shoelace_area` (geomodel.py:24-31) -- host convenience; the engine's
  per-region area output is computed on the device (``det_get_areas``).

Coordinates are y-down in the unit square; rings are open (no repeated
closing vertex); outer rings have positive shoelace area.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


def shoelace_area(ring: np.ndarray) -> float:
    """Signed area of an open (V, 2) ring (geomodel.py:24-31)."""
    r = np.asarray(ring, dtype=float)
    if r.shape[0] < 3:
        return 0.0
    xs, ys = r[:, 0], r[:, 1]
    return 0.5 * float(np.sum(xs * np.roll(ys, -1) - np.roll(xs, -1) * ys))


def ring_centroid(ring: np.ndarray) -> np.ndarray:
    """Area-weighted centroid of one ring from its shoelace moments (geomodel.py:34-47); the
    vertex mean for a degenerate ring."""
    r = np.asarray(ring, dtype=float)
    xs, ys = r[:, 0], r[:, 1]
    xn, yn = np.roll(xs, -1), np.roll(ys, -1)
    cross = xs * yn - xn * ys
    a = 0.5 * float(np.sum(cross))
    if a == 0.0:
        return r.mean(axis=0)
    return np.array([float(np.sum((xs + xn) * cross)) / (6.0 * a), float(np.sum((ys + yn) * cross)) / (6.0 * a)])


@dataclass(frozen=True)
class Region:
    """One statistical region (geomodel.py:50-80)."""

    region_id: str
    name: str
    rings: tuple
    statistic: float

    def area(self) -> float:
        return sum(shoelace_area(r) for r in self.rings)

    def centroid(self) -> np.ndarray:
        """Area-weighted centroid over all rings, holes subtracting (geomodel.py:67-77)."""
        total, acc = 0.0, np.zeros(2)
        for ring in self.rings:
            a = shoelace_area(ring)
            acc += a * ring_centroid(ring)
            total += a
        if total == 0.0:
            return np.vstack(self.rings).mean(axis=0)
        return acc / total

    def vertex_count(self) -> int:
        return sum(int(np.asarray(r).shape[0]) for r in self.rings)

    @classmethod
    def _make(cls, region_id, name, rings, statistic):
        """Fast constructor (skips the frozen-dataclass __setattr__ path)."""
        obj = object.__new__(cls)
        obj.__dict__.update(region_id=region_id, name=name, rings=rings, statistic=statistic)
        return obj


@dataclass(frozen=True)
class MapModel:
    """Regions plus optional adjacency / normalisation metadata (geomodel.py:95-145)."""

    regions: tuple
    adjacency: frozenset = frozenset()
    normalization: object = None

    def region_ids(self) -> list:
        return [r.region_id for r in self.regions]

    def statistics(self) -> np.ndarray:
        return np.array([r.statistic for r in self.regions], dtype=float)

    def total_statistic(self) -> float:
        return float(self.statistics().sum())

    def bounds(self):
        pts = self.vertex_array()
        return (float(pts[:, 0].min()), float(pts[:, 1].min()),
                float(pts[:, 0].max()), float(pts[:, 1].max()))

    def with_statistics(self, values) -> "MapModel":
        vals = np.asarray(values, dtype=float)
        return replace(self, regions=tuple(replace(r, statistic=float(v))
                                           for r, v in zip(self.regions, vals)))

    def vertex_array(self) -> np.ndarray:
        return np.vstack([np.asarray(ring, dtype=float) for reg in self.regions for ring in reg.rings])

    def with_vertex_array(self, verts: np.ndarray) -> "MapModel":
        return rebuild(self, verts)


def ring_layout(mapmodel):
    """Flatten a (duck-typed) map into index arrays.

    Returns ``(xy, ring_start, ring_region, ids, stats)`` where ``xy`` is the
    (N_rows, 2) float64 vertex array in region/ring order, ``ring_start`` the
    (n_rings+1,) row offsets and ``ring_region`` the owning region index of
    each ring.
    """
    ids, stats, rings, owner = [], [], [], []
    for ridx, reg in enumerate(mapmodel.regions):
        ids.append(str(reg.region_id))
        stats.append(float(reg.statistic))
        for ring in reg.rings:
            rings.append(np.asarray(ring, dtype=float))
            owner.append(ridx)
    sizes = np.array([r.shape[0] for r in rings], dtype=np.int64)
    ring_start = np.zeros(len(rings) + 1, dtype=np.int32)
    ring_start[1:] = np.cumsum(sizes)
    xy = np.ascontiguousarray(np.vstack(rings), dtype=np.float64)
    return xy, ring_start, np.array(owner, dtype=np.int32), ids, np.array(stats, dtype=float)


def rebuild(mapmodel, verts: np.ndarray):
    """Rebuild a map (any dataclass-based MapModel) from stacked vertex rows."""
    verts = np.asarray(verts, dtype=float)
    out, pos = [], 0
    for reg in mapmodel.regions:
        rs = []
        for ring in reg.rings:
            q = np.asarray(ring).shape[0]
            rs.append(np.array(verts[pos : pos + q], dtype=float))
            pos += q
        out.append(replace(reg, rings=tuple(rs)))
    if pos != verts.shape[0]:
        raise ValueError("vertex array length mismatch")
    return replace(mapmodel, regions=tuple(out))


def ring_sizes(mapmodel) -> np.ndarray:
    """Number of vertex rows of every ring, region/ring order."""
    return np.array([np.asarray(r).shape[0] for reg in mapmodel.regions for r in reg.rings], dtype=np.int64)


class _DeferredMapModel(MapModel):
    """A MapModel whose Region objects are built from a host vertex array on first access.

    Result maps of batched runs are views of the vertices already copied back from the
    device; building 10^3-10^4 Region dataclasses per frame would cost more than the GPU
    run itself, so it happens on first access to ``regions`` (``vertex_array`` needs no
    Regions at all).  Everything else -- equality, ``dataclasses.replace``, ``with_*`` --
    behaves as for a MapModel (the first field access materialises the regions).
    """

    def __getattr__(self, name):
        if name == "regions":
            base, verts, stats, sizes = self.__dict__["_deferred"]
            regs = rebuild_fast(base, verts, stats, sizes).regions
            object.__setattr__(self, "regions", regs)
            return regs
        raise AttributeError(name)

    def vertex_array(self) -> np.ndarray:
        if "regions" not in self.__dict__:
            return np.array(self.__dict__["_deferred"][1], dtype=float)
        return super().vertex_array()

    def __eq__(self, other):  # compares as a MapModel (dataclass __eq__ requires the same class)
        if isinstance(other, MapModel):
            return (self.regions, self.adjacency, self.normalization) == (
                other.regions, other.adjacency, other.normalization)
        return NotImplemented

    __hash__ = MapModel.__hash__


def deferred_rebuild(mapmodel, verts: np.ndarray, statistics=None, sizes=None):
    """``rebuild_fast`` whose Region objects are built on first access (own MapModel only)."""
    if type(mapmodel) is not MapModel and not isinstance(mapmodel, _DeferredMapModel):
        return rebuild_fast(mapmodel, verts, statistics, sizes)
    verts = np.asarray(verts, dtype=float)
    if sizes is None:
        sizes = ring_sizes(mapmodel)
    if int(sizes.sum()) != verts.shape[0]:
        raise ValueError("vertex array length mismatch")
    obj = object.__new__(_DeferredMapModel)
    obj.__dict__.update(adjacency=mapmodel.adjacency, normalization=mapmodel.normalization,
                        _deferred=(mapmodel, verts, statistics, sizes))
    return obj


def rebuild_fast(mapmodel, verts: np.ndarray, statistics=None, sizes=None):
    """``rebuild`` (+ optional new statistics) in one pass; rings are views of ``verts``.

    For this package's own ``Region``/``MapModel`` the objects are constructed
    directly; other (reference) dataclasses go through ``dataclasses.replace``.
    """
    verts = np.asarray(verts, dtype=float)
    if sizes is None:
        sizes = ring_sizes(mapmodel)
    if int(sizes.sum()) != verts.shape[0]:
        raise ValueError("vertex array length mismatch")
    offs = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    pieces = [verts[a:e] for a, e in zip(offs[:-1], offs[1:])]
    out, q = [], 0
    own = isinstance(mapmodel, MapModel)
    stats_l = None if statistics is None else np.asarray(statistics, dtype=float).tolist()
    for i, reg in enumerate(mapmodel.regions):
        nr = len(reg.rings)
        rings = tuple(pieces[q : q + nr])
        q += nr
        stat = reg.statistic if statistics is None else stats_l[i]
        if own and type(reg) is Region:
            out.append(Region._make(reg.region_id, reg.name, rings, stat))
        else:
            out.append(replace(reg, rings=rings, statistic=stat))
    if own:
        return MapModel(tuple(out), mapmodel.adjacency, mapmodel.normalization)
    return replace(mapmodel, regions=tuple(out))


def densify(mapmodel, max_edge: float):
    """Split edges longer than ``max_edge`` into equal pieces (geomodel.py:353-377)."""
    if max_edge <= 0:
        raise ValueError("max_edge must be positive")
    new_regions = []
    for reg in mapmodel.regions:
        rs = []
        for ring in reg.rings:
            ring = np.asarray(ring, dtype=float)
            nxt = np.roll(ring, -1, axis=0)
            ln = np.hypot(*(nxt - ring).T)
            pieces = np.maximum(1, np.ceil(ln / max_edge).astype(int))
            if pieces.max() == 1:
                rs.append(ring)
                continue
            parts = [p0 + (np.arange(q) / q)[:, None] * (p1 - p0) for p0, p1, q in zip(ring, nxt, pieces)]
            rs.append(np.vstack(parts))
        new_regions.append(replace(reg, rings=tuple(rs)))
    return replace(mapmodel, regions=tuple(new_regions))


def detect_adjacencies(mapmodel, epsilon: float, *, device: int = 0) -> frozenset:
    """Region pairs sharing >= 2 coincident vertex cells (geomodel.py:380-415), on the GPU."""
    from .metrics import detect_adjacencies as _detect

    return _detect(mapmodel, epsilon, device=device)


def with_adjacency(mapmodel, epsilon: float, *, device: int = 0):
    """The map with its adjacency set filled in (geomodel.py:418-419)."""
    return replace(mapmodel, adjacency=detect_adjacencies(mapmodel, epsilon, device=device))


def _inside_ring(pt, ring) -> bool:
    """Even-odd point-in-ring test used to attach holes (geomodel.py:466-477)."""
    x, y = float(pt[0]), float(pt[1])
    inside = False
    r = np.asarray(ring, dtype=float)
    for (x0, y0), (x1, y1) in zip(r, np.roll(r, -1, axis=0)):
        if (y0 <= y) != (y1 <= y) and x0 + (y - y0) * (x1 - x0) / (y1 - y0) > x:
            inside = not inside
    return inside


def to_geojson(mapmodel, extra_properties: dict | None = None) -> bytes:
    """GeoJSON FeatureCollection of a (deformed) map, y-up (geomodel.py:422-463).

    Output format of cartogram runs: outer rings are the positively oriented ones, each
    hole goes to the first outer ring containing its first vertex, rings are closed and
    y is emitted as 1 - y; keys are sorted and separators compact, so the bytes match the
    reference's emitter.
    """
    import json

    feats = []
    for reg in mapmodel.regions:
        rings = [np.asarray(r, dtype=float) for r in reg.rings]
        outer = [r for r in rings if shoelace_area(r) >= 0]
        holes = [r for r in rings if shoelace_area(r) < 0]
        if not outer:
            raise ValueError(f"region {reg.region_id!r} has no positively oriented ring")
        polys = [[r] for r in outer]
        for h in holes:
            dest = next((i for i, o in enumerate(outer) if _inside_ring(h[0], o)), 0)
            polys[dest].append(h)
        coords = [[[[float(x), float(1.0 - y)] for x, y in np.vstack([r, r[:1]])] for r in poly] for poly in polys]
        geom = ({"type": "Polygon", "coordinates": coords[0]} if len(coords) == 1
                else {"type": "MultiPolygon", "coordinates": coords})
        props = {"name": reg.name, "statistic": reg.statistic}
        if extra_properties and reg.region_id in extra_properties:
            props.update(extra_properties[reg.region_id])
        feats.append({"type": "Feature", "id": reg.region_id, "properties": props, "geometry": geom})
    return json.dumps({"type": "FeatureCollection", "features": feats}, sort_keys=True,
                      separators=(",", ":")).encode()
