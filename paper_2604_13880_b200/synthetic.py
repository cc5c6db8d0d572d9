"""Seeded synthetic inputs standing in for the BASELINE configs.

The reference publishes no benchmark dataset for this path (BASELINE.md §1,
SURVEY.md §8d); its configs are described as Voronoi maps with lognormal
statistics.  This module builds them deterministically:

* cells of ``R`` uniform seeds in the central 80 % of the unit square
  (``[0.1, 0.9]^2``), optionally relaxed by Lloyd iterations;
* cells are clipped to that box exactly by mirroring the seeds across its four
  sides before the Voronoi construction (scipy/qhull);
* every Voronoi edge ("chain") is resampled once and reused (reversed) by the
  neighbouring cell, so shared vertices are bit-identical between rings;
* rings are open and counter-clockwise in the y-down frame (positive
  shoelace), the orientation ``cartomorph`` expects.

The vertex count is pinned through the per-chain resampling (SURVEY.md §0
note 6): ``target_unique`` is the number of unique vertex positions.
"""

from __future__ import annotations

import numpy as np

from .geomodel import MapModel, Region, shoelace_area

BOX = (0.1, 0.9)


def _voronoi_cells(seeds: np.ndarray, lo: float, hi: float):
    from scipy.spatial import Voronoi

    r = seeds.shape[0]
    mirrors = [
        np.column_stack([2 * lo - seeds[:, 0], seeds[:, 1]]),
        np.column_stack([2 * hi - seeds[:, 0], seeds[:, 1]]),
        np.column_stack([seeds[:, 0], 2 * lo - seeds[:, 1]]),
        np.column_stack([seeds[:, 0], 2 * hi - seeds[:, 1]]),
    ]
    vor = Voronoi(np.vstack([seeds] + mirrors))
    cells = []
    for i in range(r):
        reg = vor.regions[vor.point_region[i]]
        if -1 in reg or len(reg) < 3:
            raise RuntimeError("unbounded Voronoi cell for an interior seed")
        cells.append(list(reg))
    verts = np.clip(vor.vertices, lo, hi)
    return verts, cells


def _cell_centroids(verts, cells):
    out = np.empty((len(cells), 2))
    for c, idx in enumerate(cells):
        p = verts[idx]
        x, y = p[:, 0], p[:, 1]
        xn, yn = np.roll(x, -1), np.roll(y, -1)
        cr = x * yn - xn * y
        a = 0.5 * cr.sum()
        out[c] = [((x + xn) * cr).sum() / (6 * a), ((y + yn) * cr).sum() / (6 * a)]
    return out


def voronoi_map(n_regions: int, seed: int = 0, lloyd: int = 0, target_unique: int | None = None,
                spacing: float | None = None, sigma: float = 1.0, id_prefix: str = "R",
                shuffle_ids: bool = False) -> MapModel:
    """A seeded Voronoi map with lognormal(0, sigma) statistics.

    Either ``target_unique`` (number of unique vertices) or ``spacing``
    (maximum chain segment length in unit-square coordinates) fixes the
    resampling.  With neither, chains keep only their Voronoi end points.
    """
    lo, hi = BOX
    rng = np.random.default_rng(seed)
    seeds = rng.uniform(lo, hi, size=(n_regions, 2))
    for _ in range(lloyd):
        v, c = _voronoi_cells(seeds, lo, hi)
        seeds = _cell_centroids(v, c)
    verts, cells = _voronoi_cells(seeds, lo, hi)

    # unique chains (Voronoi edges) used by the cells
    chains = {}
    for idx in cells:
        for a, b in zip(idx, idx[1:] + idx[:1]):
            chains.setdefault((min(a, b), max(a, b)), None)
    keys = sorted(chains)
    lens = np.array([np.hypot(*(verts[b] - verts[a])) for a, b in keys])
    used = sorted({v for idx in cells for v in idx})
    if target_unique is not None:
        extra = max(target_unique - len(used), 0)
        spacing = float(lens.sum()) / max(extra + len(keys), 1)
        # refine once so that the rounding of per-chain piece counts hits the target
        for _ in range(3):
            pieces = np.maximum(1, np.round(lens / spacing).astype(np.int64))
            got = len(used) + int((pieces - 1).sum())
            if got == 0:
                break
            spacing *= got / max(target_unique, 1)
    if spacing is None:
        pieces = np.ones(len(keys), dtype=np.int64)
    else:
        pieces = np.maximum(1, np.round(lens / spacing).astype(np.int64))
    for (a, b), q in zip(keys, pieces):
        t = np.arange(1, q)[:, None] / q
        chains[(a, b)] = verts[a] + t * (verts[b] - verts[a])

    regions = []
    ids = [f"{id_prefix}{i:05d}" for i in range(n_regions)]
    if shuffle_ids:
        perm = rng.permutation(n_regions)
        ids = [f"{id_prefix}{int(p)}" for p in perm]  # string order != index order
    stats = np.exp(rng.normal(0.0, sigma, size=n_regions))
    for c, idx in enumerate(cells):
        parts = []
        for a, b in zip(idx, idx[1:] + idx[:1]):
            parts.append(verts[a][None, :])
            inner = chains[(min(a, b), max(a, b))]
            parts.append(inner if a < b else inner[::-1])
        ring = np.vstack(parts)
        if shoelace_area(ring) < 0:
            ring = ring[::-1].copy()
        regions.append(Region(ids[c], ids[c], (np.ascontiguousarray(ring),), float(stats[c])))
    return MapModel(regions=tuple(regions))


def unique_vertex_count(mapmodel) -> int:
    xy = mapmodel.vertex_array()
    return int(np.unique(xy.view(np.complex128).ravel()).shape[0])


def random_walk(stats0: np.ndarray, steps: int, sigma: float, seed: int) -> np.ndarray:
    """(T, R) multiplicative lognormal random walk starting at ``stats0``."""
    rng = np.random.default_rng(seed)
    out = np.empty((steps, stats0.shape[0]))
    cur = np.asarray(stats0, dtype=float).copy()
    for t in range(steps):
        if t > 0:
            cur = cur * np.exp(rng.normal(0.0, sigma, size=cur.shape[0]))
        out[t] = cur
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configs, seeded
# ---------------------------------------------------------------------------

def config_map(name: str) -> tuple[MapModel, dict]:
    """Return (map, run-parameters) for a named BASELINE config.

    ``headline`` is the metric's own workload: 1024^2 texture and ~200k unique
    vertices (3000 Voronoi regions).
    """
    if name == "c1":
        m = voronoi_map(64, seed=0, target_unique=2000, sigma=1.0)
        return m, dict(k=8, iterations=100, bdv_multiplier=0.5, steps=1)
    if name == "c2":
        m = voronoi_map(500, seed=1, lloyd=2, target_unique=40_000, sigma=1.5)
        return m, dict(k=10, iterations=100, bdv_multiplier=1.0, steps=12, walk_sigma=0.1,
                       mode="cumulative")
    if name == "c3":
        m = voronoi_map(3000, seed=3, target_unique=200_000, sigma=2.0)
        s = m.statistics()
        rng = np.random.default_rng(33)
        pick = rng.choice(s.shape[0], size=int(0.05 * s.shape[0]), replace=False)
        s[pick] = 1e-3 * np.median(s)
        m = m.with_statistics(s)
        return m, dict(k=11, iterations=200, bdv_multiplier=0.3, steps=50, walk_sigma=0.15,
                       mode="direct")
    if name == "c4":
        m = voronoi_map(500, seed=1, lloyd=2, target_unique=40_000, sigma=1.5)
        return m, dict(k=10, iterations=150, batch=64)
    if name == "headline":
        # values are unspecified by the metric; lognormal(0, 0.5) keeps every frame of the
        # 3000-cell map alive for >2000 iterations (sigma >= 1 collapses regions after ~100-500
        # iterations -- RegionCollapsedError, as in the reference -- ending frames mid-benchmark;
        # tools/collapse_scan.py)
        m = voronoi_map(3000, seed=3, target_unique=200_000, sigma=0.5)
        return m, dict(k=10, iterations=200, bdv_multiplier=1.0)
    if name == "c5":
        m = voronoi_map(10_000, seed=5, target_unique=1_000_000, sigma=2.5)
        rng = np.random.default_rng(55)
        mu = rng.uniform(0.1, 0.9, size=(20, 2))
        cen = np.array([np.asarray(r.rings[0]).mean(axis=0) for r in m.regions])
        bump = np.exp(-((cen[:, None, :] - mu[None]) ** 2).sum(-1) / (2 * 0.05 ** 2)).sum(1)
        m = m.with_statistics(m.statistics() * (1.0 + bump))
        return m, dict(k=12, iterations=100, steps=100)
    raise KeyError(name)


def batch_statistics(mapmodel, n_seeds: int, sigma: float, seed0: int = 100) -> np.ndarray:
    """(n_seeds, R) lognormal(0, sigma) statistic vectors, one per value seed."""
    r = len(mapmodel.regions)
    return np.stack([np.exp(np.random.default_rng(seed0 + i).normal(0.0, sigma, size=r))
                     for i in range(n_seeds)])
