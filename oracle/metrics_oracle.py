"""ORACLE -- CPU restatement of the reference's frame quality metrics.  TEST INFRASTRUCTURE ONLY.

Same rules as ``det_oracle``: only ``tests/`` may import this module, as the checker of the
GPU metric kernels (``paper_2604_13880_b200.metrics``); the product path never imports it.

Restates ``cartomorph/metrics.py`` and ``geomodel.py:24-77,380-415`` with the reference's numpy
operation order (so areas, barycenters, rescaled rings and shape masks are bit-identical; pinned by
``tests/test_metrics_golden.py`` against fixtures generated from the reference itself).  The best
shift overlap is the exact integer correlation; the reference recovers the same integers by
rounding an FFT correlation (metrics.py:96-97), which this oracle also does, so either route gives
the reference's values.  Rings are lists of (V, 2) float64 arrays; maps are lists of such lists.
"""

from __future__ import annotations

import numpy as np
from scipy.signal import fftconvolve

from .det_oracle import region_fill


class OracleNumericError(Exception):
    pass


class OracleMaskError(Exception):
    pass


def shoelace(ring) -> float:
    """geomodel.py:24-31."""
    r = np.asarray(ring, dtype=float)
    if r.shape[0] < 3:
        return 0.0
    xs, ys = r[:, 0], r[:, 1]
    return 0.5 * float(np.sum(xs * np.roll(ys, -1) - np.roll(xs, -1) * ys))


def ring_centroid(ring) -> np.ndarray:
    """geomodel.py:34-47."""
    ring = np.asarray(ring, dtype=float)
    x, y = ring[:, 0], ring[:, 1]
    xn, yn = np.roll(x, -1), np.roll(y, -1)
    cross = x * yn - xn * y
    area = 0.5 * float(np.sum(cross))
    if area == 0.0:
        return ring.mean(axis=0)
    return np.array([float(np.sum((x + xn) * cross)) / (6.0 * area), float(np.sum((y + yn) * cross)) / (6.0 * area)])


def region_area(rings) -> float:
    """Region.area (geomodel.py:63-65): Python sum of ring areas."""
    return sum(shoelace(r) for r in rings)


def region_centroid(rings) -> np.ndarray:
    """Region.centroid (geomodel.py:67-77)."""
    total = 0.0
    acc = np.zeros(2)
    for ring in rings:
        a = shoelace(ring)
        acc += a * ring_centroid(ring)
        total += a
    if total == 0.0:
        return np.vstack(rings).mean(axis=0)
    return acc / total


def rescaled(rings, target_area: float = 1.0):
    """metrics.py:48-59."""
    areas = [shoelace(r) for r in rings]
    total = sum(areas)
    if total <= 0:
        raise OracleNumericError("region with non-positive area")
    centroid = sum(a * ring_centroid(r) for a, r in zip(areas, rings)) / total
    factor = np.sqrt(target_area / total)
    return [(np.asarray(r, dtype=float) - centroid) * factor for r in rings]


def mask_pair(rings_a, rings_b, k: int):
    """Both ring sets on one square 2^k grid (metrics.py:62-77)."""
    n = 1 << k
    pts = np.vstack([np.vstack(rings_a), np.vstack(rings_b)])
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    center = 0.5 * (lo + hi)
    half = 0.55 * float(max(hi - lo)) + 1e-12
    corner = center - half
    ma = region_fill([(r - corner) / (2 * half) for r in rings_a], n)
    mb = region_fill([(r - corner) / (2 * half) for r in rings_b], n)
    if not ma.any() or not mb.any():
        raise OracleMaskError("shape rasterized to zero pixels in Hamming grid")
    return ma, mb


def best_overlap(ma, mb) -> int:
    """max over the +-extent shift window of |A & shift(B)| (metrics.py:96-112)."""
    corr = np.round(fftconvolve(ma.astype(float), mb[::-1, ::-1].astype(float), mode="full"))
    n = ma.shape[0]

    def extent(m):
        ys, xs = np.nonzero(m)
        return xs.max() - xs.min() + 1, ys.max() - ys.min() + 1

    wxa, wya = extent(ma)
    wxb, wyb = extent(mb)
    wx, wy = max(wxa, wxb), max(wya, wyb)
    shifts = np.arange(2 * n - 1) - (n - 1)
    win = (np.abs(shifts)[:, None] <= wy) & (np.abs(shifts)[None, :] <= wx)
    return int(corr.clip(0.0, min(ma.sum(), mb.sum()))[win].max())


def hamming(rings_a, rings_b, k: int = 7, rescale: bool = True) -> float:
    """metrics.py:80-118."""
    if rescale:
        rings_a, rings_b = rescaled(rings_a), rescaled(rings_b)
    ma, mb = mask_pair(rings_a, rings_b, k)
    na, nb = float(ma.sum()), float(mb.sum())
    best = float(best_overlap(ma, mb))
    union = na + nb - best
    return 0.0 if union <= 0 else (na + nb - 2.0 * best) / union


def adjacency(region_rings, epsilon: float) -> set:
    """geomodel.py:380-415 on region indices: pairs (a < b) with >= 2 shared cells."""
    cell_sets, owners = [], {}
    for ridx, rings in enumerate(region_rings):
        cs = set(map(tuple, np.round(np.vstack(rings) / epsilon).astype(np.int64)))
        cell_sets.append(cs)
        for c in cs:
            owners.setdefault(c, set()).add(ridx)
    shared = {}
    for a, cs in enumerate(cell_sets):
        for cx, cy in cs:
            partners = set()
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    partners.update(owners.get((cx + dx, cy + dy), ()))
            for b in partners:
                if b > a:
                    shared[(a, b)] = shared.get((a, b), 0) + 1
    return {p for p, c in shared.items() if c >= 2}


def position_error(cent_m, cent_c) -> float:
    """metrics.py:138-162 (sequential Python sum over ordered pairs)."""
    count = len(cent_m)
    total = 0.0
    for u in range(count):
        for v in range(count):
            if u == v:
                continue
            vm = cent_m[v] - cent_m[u]
            vc = cent_c[v] - cent_c[u]
            if np.allclose(vm, 0) or np.allclose(vc, 0):
                continue
            total += abs(np.arctan2(vm[0] * vc[1] - vm[1] * vc[0], vm[0] * vc[0] + vm[1] * vc[1]))
    return total / (np.pi * count * (count - 1))
