"""Small hand-made maps exercising the raster edge cases the reference tests.

Shared by the golden generator and the tests.  They are built from our own
``MapModel``; coordinates are y-down in the unit square.
"""

from __future__ import annotations

import numpy as np

from paper_2604_13880_b200.geomodel import MapModel, Region
from paper_2604_13880_b200.synthetic import voronoi_map


def _sq(x0, y0, x1, y1):
    return np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], dtype=float)


def two_region(stats=(1.0, 3.0)) -> MapModel:
    """Vertical split of the 0.9-scaled unit square (cf. fixtures.two_region_map)."""
    a = _sq(0.05, 0.05, 0.5, 0.95)
    b = _sq(0.5, 0.05, 0.95, 0.95)
    return MapModel(regions=(Region("A", "A", (a,), float(stats[0])), Region("B", "B", (b,), float(stats[1]))))


def tie_partition() -> MapModel:
    """Shared edge exactly on a pixel-centre column at n=16 (test_raster.py:49-63)."""
    s = 8.5 / 16
    a = np.array([[0.0, 0.0], [s, 0.0], [s, 1.0], [0.0, 1.0]])
    b = np.array([[s, 0.0], [1.0, 0.0], [1.0, 1.0], [s, 1.0]])
    return MapModel(regions=(Region("A", "A", (a,), 1.0), Region("B", "B", (b,), 1.0)))


def overlap_holes_multi() -> MapModel:
    """Overlapping regions (min id wins), a region with a hole and a two-ring region.

    Region ids are chosen so that string order differs from index order.
    """
    outer = _sq(0.1, 0.1, 0.6, 0.6)
    hole = _sq(0.25, 0.25, 0.4, 0.4)[::-1].copy()
    r_hole = Region("R10", "holed", (outer, hole), 3.0)
    r_over = Region("R2", "overlap", (_sq(0.45, 0.3, 0.85, 0.75),), 2.0)
    tri = np.array([[0.62, 0.05], [0.95, 0.08], [0.7, 0.28]])
    r_multi = Region("R1", "multi", (_sq(0.05, 0.7, 0.3, 0.95), tri), 1.5)
    r_in_hole = Region("R3", "island", (_sq(0.28, 0.28, 0.37, 0.37),), 0.7)
    return MapModel(regions=(r_hole, r_over, r_multi, r_in_hole))


def sliver() -> MapModel:
    """Three strips, the middle one with a near-zero statistic (test_engine.py:92-108)."""
    left = _sq(0.05, 0.05, 0.482, 0.95)
    mid = _sq(0.482, 0.05, 0.518, 0.95)
    right = _sq(0.518, 0.05, 0.95, 0.95)
    return MapModel(regions=(Region("L", "L", (left,), 100.0), Region("M", "M", (mid,), 1e-4),
                             Region("R", "R", (right,), 100.0)))


def small_voronoi(seed=0, r=24, target=600, shuffle_ids=True) -> MapModel:
    return voronoi_map(r, seed=seed, target_unique=target, sigma=1.0, shuffle_ids=shuffle_ids)


def config1() -> MapModel:
    """BASELINE config 1: 64 Voronoi regions, seed 0, ~2k unique vertices, lognormal(0,1)."""
    return voronoi_map(64, seed=0, target_unique=2000, sigma=1.0)


def pack_map(m) -> dict:
    from paper_2604_13880_b200.geomodel import ring_layout

    xy, rs, rr, ids, stats = ring_layout(m)
    return dict(xy=xy, ring_start=rs, ring_region=rr, ids=np.array(ids), stats=stats,
                names=np.array([str(r.name) for r in m.regions]))


def unpack_map(z, prefix="") -> MapModel:
    xy = z[prefix + "xy"]
    rs = z[prefix + "ring_start"]
    rr = z[prefix + "ring_region"]
    ids = [str(s) for s in z[prefix + "ids"]]
    stats = z[prefix + "stats"]
    rings = [[] for _ in ids]
    for q in range(len(rr)):
        rings[int(rr[q])].append(np.array(xy[rs[q] : rs[q + 1]], dtype=float))
    names = [str(s) for s in z[prefix + "names"]] if (prefix + "names") in z else ids
    return MapModel(regions=tuple(Region(i, nm, tuple(rg), float(s)) for i, nm, rg, s in zip(ids, names, rings, stats)))


def many_holes(n_holes=200, y0=0.47, y1=0.53) -> MapModel:
    """A square region pierced by `n_holes` thin triangular holes along one horizontal band, so a
    scanline through the band crosses 2*n_holes + 2 of its edges (raster.py:80-89 has no limit
    on crossings per row); a second region beside it and an island inside one hole."""
    outer = _sq(0.05, 0.05, 0.9, 0.95)
    holes = []
    xs = np.linspace(0.07, 0.88, n_holes, endpoint=False)
    w = 0.45 * (xs[1] - xs[0])
    for x in xs:
        holes.append(np.array([[x, y0], [x + 0.5 * w, y1], [x + w, y0 + 0.002]]))  # CW in y-down: a hole
    a = Region("A", "holed", (outer, *holes), 5.0)
    b = Region("B", "side", (_sq(0.91, 0.3, 0.98, 0.7),), 1.0)
    x = xs[n_holes // 2]
    isl = Region("C", "island", (np.array([[x + 0.2 * w, y0 + 0.01], [x + 0.8 * w, y0 + 0.01],
                                           [x + 0.5 * w, y0 + 0.02]]),), 0.5)
    return MapModel(regions=(a, b, isl))


def needle_rings(n_rings=150) -> MapModel:
    """A square region with `n_rings` two-vertex rings crossing the same scanlines: each adds two
    coincident toggles per scanline (they cancel), so a row carries > 256 toggles while the
    region keeps <= 384 rows (the shared-memory path of k_region)."""
    outer = _sq(0.1, 0.1, 0.9, 0.9)
    xs = np.linspace(0.15, 0.85, n_rings)
    rings = [np.array([[x, 0.3], [x + 0.001, 0.7]]) for x in xs]
    return MapModel(regions=(Region("A", "needles", (outer, *rings), 2.0),
                             Region("B", "other", (_sq(0.91, 0.3, 0.98, 0.6),), 1.0)))
