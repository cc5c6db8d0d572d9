"""ORACLE -- CPU restatement of the reference DET hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and there only as the checker
(or the timed CPU baseline) -- never as the product path.  The product path is
``paper_2604_13880_b200`` (CUDA kernels behind a C-ABI) and it never imports
anything under ``oracle/``.

Every function restates one piece of the reference package ``cartomorph``
(``/root/reference/pkg/src/cartomorph``) with the same float64 operation order,
so on the same inputs it reproduces the reference bit for bit (pinned by
``tests/test_oracle_golden.py`` against fixtures generated from the reference
itself by ``tests/golden/make_golden.py``).  The data model here is a flat one
(vertex rows + ring/region index arrays) instead of the reference's frozen
dataclasses; the arithmetic is the reference's.

Citations are ``file:line`` into ``/root/reference/pkg/src/cartomorph``.
"""

from __future__ import annotations

import ctypes
import functools
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

BACKGROUND = -1  # raster.py:20
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libdet_oracle.so")


class OracleError(Exception):
    """Base for oracle-raised errors (mirrors cartomorph.errors)."""


class OracleRasterizationError(OracleError):
    pass


class OracleCollapseError(OracleError):
    def __init__(self, region_id, iteration):
        super().__init__(f"region {region_id!r} collapsed to zero pixels at iteration {iteration}")
        self.region_id = region_id
        self.iteration = iteration


class OracleNumericError(OracleError):
    pass


# ---------------------------------------------------------------------------
# C helper for the tilted recurrences (integral.py:65-125)
# ---------------------------------------------------------------------------

def build_oracle_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


@functools.lru_cache(maxsize=1)
def _lib():
    build_oracle_lib()
    lib = ctypes.CDLL(_LIB_PATH)
    for name in ("det_oracle_closed_top_cone", "det_oracle_diag_up_left", "det_oracle_diag_up_right"):
        fn = getattr(lib, name)
        fn.restype = ctypes.c_int
        fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


def _run2d(name: str, d: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(d, dtype=np.float64)
    out = np.empty_like(d)
    rc = getattr(_lib(), name)(d.ctypes.data, d.shape[0], d.shape[1], out.ctypes.data)
    if rc != 0:
        raise MemoryError(name)
    return out


# ---------------------------------------------------------------------------
# Rasterisation (raster.py)
# ---------------------------------------------------------------------------

def ring_toggles(ring: np.ndarray, n: int):
    """Even-odd toggle positions (j, i0) of one ring; raster.py:23-61.

    The crossing abscissa is evaluated as x0 + (yc - y0) * slope with
    slope = (x1 - x0) / (y1 - y0), each an IEEE float64 op, in that order.
    """
    a = np.asarray(ring, dtype=float)
    b = np.roll(a, -1, axis=0)
    ya = a[:, 1] * n
    yb = b[:, 1] * n
    sel = ya != yb
    if not sel.any():
        return None
    xa = a[sel, 0] * n
    xb = b[sel, 0] * n
    ya = ya[sel]
    yb = yb[sel]
    top = np.minimum(ya, yb)
    bot = np.maximum(ya, yb)
    first = np.clip(np.ceil(top - 0.5).astype(np.int64), 0, n)
    last = np.clip(np.ceil(bot - 0.5).astype(np.int64), 0, n)
    cnt = last - first
    ok = cnt > 0
    if not ok.any():
        return None
    xa, xb, ya, yb, first, cnt = xa[ok], xb[ok], ya[ok], yb[ok], first[ok], cnt[ok]
    tot = int(cnt.sum())
    base = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    local = np.arange(tot) - np.repeat(base, cnt)
    rows = np.repeat(first, cnt) + local
    centre = rows + 0.5
    k = (xb - xa) / (yb - ya)
    xc = np.repeat(xa, cnt) + (centre - np.repeat(ya, cnt)) * np.repeat(k, cnt)
    cols = np.clip(np.ceil(xc - 0.5).astype(np.int64), 0, n)
    return rows, cols


def region_crop_mask(rings, n: int):
    """(j_off, i_off, mask) of a region's even-odd fill in its bbox crop; raster.py:64-91."""
    pts = np.vstack(rings)
    j0 = int(np.clip(np.ceil(pts[:, 1].min() * n - 0.5), 0, n))
    j1 = int(np.clip(np.ceil(pts[:, 1].max() * n - 0.5), 0, n))
    i0 = int(np.clip(np.ceil(pts[:, 0].min() * n - 0.5), 0, n))
    i1 = int(np.clip(np.ceil(pts[:, 0].max() * n - 0.5), 0, n))
    h = max(j1 - j0, 0)
    w = max(i1 - i0, 0)
    if h == 0 or w == 0:
        return j0, i0, np.zeros((h, w), dtype=bool)
    stride = w + 1  # absorber column for toggles at/after the crop edge (raster.py:79-80)
    acc = np.zeros(h * stride, dtype=np.int64)
    for ring in rings:
        tg = ring_toggles(np.asarray(ring, dtype=float), n)
        if tg is None:
            continue
        rows, cols = tg
        # a negative flat index raises ValueError inside bincount, as in the reference
        acc += np.bincount((rows - j0) * stride + np.minimum(cols - i0, w), minlength=h * stride)
    par = np.cumsum(acc.reshape(h, stride)[:, :w], axis=1) & 1
    return j0, i0, par.astype(bool)


def region_fill(rings, n: int) -> np.ndarray:
    """Full-texture even-odd mask of a ring set; raster.py:94-99."""
    j0, i0, sub = region_crop_mask(rings, n)
    out = np.zeros((n, n), dtype=bool)
    out[j0 : j0 + sub.shape[0], i0 : i0 + sub.shape[1]] = sub
    return out


def paint_labels(region_rings, region_ids, k: int) -> np.ndarray:
    """Label texture, lowest id wins on overlaps; raster.py:136-147."""
    if not (4 <= k <= 13):
        raise ValueError("texture exponent k must be in [4, 13]")
    n = 1 << k
    lab = np.full((n, n), BACKGROUND, dtype=np.int32)
    for idx in sorted(range(len(region_ids)), key=lambda q: region_ids[q]):
        j0, i0, sub = region_crop_mask(region_rings[idx], n)
        view = lab[j0 : j0 + sub.shape[0], i0 : i0 + sub.shape[1]]
        np.copyto(view, idx, where=sub & (view == BACKGROUND))
    return lab


def label_counts(lab: np.ndarray, n_regions: int) -> np.ndarray:
    """Per-region pixel counts; raster.py:110-112."""
    return np.bincount(lab[lab >= 0], minlength=n_regions).astype(np.int64)


def background_pixels(lab: np.ndarray) -> int:
    """raster.py:114-115."""
    return int((lab == BACKGROUND).sum())


def density_texture(stats: np.ndarray, lab: np.ndarray, bdv: float) -> np.ndarray:
    """d = s/o inside regions, bdv on background; raster.py:166-184."""
    if bdv <= 0:
        raise ValueError("bdv must be positive")
    cnt = label_counts(lab, len(stats))
    if (cnt == 0).any():
        raise OracleRasterizationError("cannot build density with zero-pixel regions")
    lut = np.concatenate([np.asarray(stats, dtype=float) / cnt, [float(bdv)]])
    return lut[np.where(lab >= 0, lab, len(stats))]


# ---------------------------------------------------------------------------
# Integral images (integral.py)
# ---------------------------------------------------------------------------

def straight_channels(d: np.ndarray):
    """alpha, beta, gamma, delta, total; integral.py:47-62."""
    d = np.asarray(d, dtype=np.float64)
    al = d.cumsum(axis=0).cumsum(axis=1)
    colt = al[-1:, :]
    rowt = al[:, -1:]
    tot = float(al[-1, -1])
    return al, colt - al, tot - colt - rowt + al, rowt - al, tot


def tilted_channels(d: np.ndarray):
    """alpha_t (top), beta_t (left), gamma_t (bottom), delta_t (right); integral.py:128-152."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    fv = np.ascontiguousarray(d[::-1])
    at = _run2d("det_oracle_closed_top_cone", d)
    at -= _run2d("det_oracle_diag_up_right", d)
    at += d
    bt = _run2d("det_oracle_closed_top_cone", np.ascontiguousarray(d.T)).T.copy()
    bt -= _run2d("det_oracle_diag_up_left", d)
    gt = _run2d("det_oracle_closed_top_cone", fv)[::-1].copy()
    gt -= _run2d("det_oracle_diag_up_left", fv)[::-1]
    dt = _run2d("det_oracle_closed_top_cone", np.ascontiguousarray(d[:, ::-1].T)).T[:, ::-1].copy()
    dt -= _run2d("det_oracle_diag_up_right", fv)[::-1]
    return at, bt, gt, dt


def all_channels(d: np.ndarray):
    """(alpha, beta, gamma, delta, alpha_t, beta_t, gamma_t, delta_t, total); integral.py:155-169."""
    a, b, g, dl, tot = straight_channels(d)
    return (a, b, g, dl) + tilted_channels(d) + (tot,)


# ---------------------------------------------------------------------------
# Anchor mapping / displacement (displacement.py)
# ---------------------------------------------------------------------------

@functools.lru_cache(maxsize=8)
def anchor_grid(n: int):
    """q1..q4 and the pixel-centre coordinates; displacement.py:56-74."""
    c = (np.arange(n) + 0.5) / n
    x = c[None, :]
    y = c[:, None]
    lower = y < x
    q1x = np.where(lower, 1.0, 1.0 - y + x)
    q1y = np.where(lower, 1.0 + y - x, 1.0)
    q3x = np.where(lower, x - y, 0.0)
    q3y = np.where(lower, 0.0, y - x)
    near = x + y < 1.0
    q2x = np.where(near, x + y, 1.0)
    q2y = np.where(near, 0.0, x + y - 1.0)
    q4x = np.where(near, 0.0, x + y - 1.0)
    q4y = np.where(near, x + y, 1.0)
    return (q1x, q1y, q2x, q2y, q3x, q3y, q4x, q4y,
            np.broadcast_to(x, (n, n)), np.broadcast_to(y, (n, n)))


def target_field(ch) -> np.ndarray:
    """Anchor-combination target at every pixel centre, (n,n,2); displacement.py:102-131."""
    al, _b, _g, _d, at, bt, gt, dt, tot = ch
    if tot <= 0:
        raise OracleNumericError("mapping undefined for zero total density")
    n = al.shape[0]
    q1x, q1y, q2x, q2y, q3x, q3y, q4x, q4y, x, y = anchor_grid(n)
    inv = 1.0 / (2.0 * tot)
    ext = np.zeros((n + 1, n + 1))
    ext[1:, 1:] = al
    a = 0.25 * (ext[:-1, :-1] + ext[:-1, 1:] + ext[1:, :-1] + ext[1:, 1:])
    cf = ext[-1, :]
    rf = ext[:, -1]
    cavg = (0.5 * (cf[:-1] + cf[1:]))[None, :]
    ravg = (0.5 * (rf[:-1] + rf[1:]))[:, None]
    b = cavg - a
    dd = ravg - a
    g = tot - cavg - ravg + a
    tx = (a * q1x + b * q2x + g * q3x + dd * q4x + at * x + bt + gt * x) * inv
    ty = (a * q1y + b * q2y + g * q3y + dd * q4y + at + bt * y + dt * y) * inv
    return np.stack([tx, ty], axis=-1)


@functools.lru_cache(maxsize=8)
def base_target(n: int) -> np.ndarray:
    """Mapping of a constant texture; displacement.py:173-183."""
    g = target_field(all_channels(np.ones((n, n))))
    g.setflags(write=False)
    return g


def displacement(d: np.ndarray) -> np.ndarray:
    """u = t(d) - t(const) at pixel centres; displacement.py:198-206."""
    return target_field(all_channels(d)) - base_target(d.shape[0])


def bilinear(u: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """displacement.py:209-226."""
    n = u.shape[0]
    g = np.asarray(pts, dtype=float) * n - 0.5
    ix = np.clip(np.floor(g[:, 0]).astype(np.int64), 0, n - 2)
    iy = np.clip(np.floor(g[:, 1]).astype(np.int64), 0, n - 2)
    fx = np.clip(g[:, 0] - ix, 0.0, 1.0)[:, None]
    fy = np.clip(g[:, 1] - iy, 0.0, 1.0)[:, None]
    return (u[iy, ix] * (1 - fx) * (1 - fy) + u[iy, ix + 1] * fx * (1 - fy)
            + u[iy + 1, ix] * (1 - fx) * fy + u[iy + 1, ix + 1] * fx * fy)


def move_vertices(pts: np.ndarray, u: np.ndarray):
    """Advect + clamp + clamp count; displacement.py:229-238."""
    p = np.asarray(pts, dtype=float)
    moved = p + bilinear(u, p)
    cl = np.clip(moved, 0.0, 1.0)
    return cl, int(np.count_nonzero(cl != moved))


# ---------------------------------------------------------------------------
# Geometry helpers (geomodel.py)
# ---------------------------------------------------------------------------

def ring_area(ring) -> float:
    """Signed shoelace area; geomodel.py:24-31."""
    r = np.asarray(ring, dtype=float)
    if r.shape[0] < 3:
        return 0.0
    return 0.5 * float(np.sum(r[:, 0] * np.roll(r[:, 1], -1) - np.roll(r[:, 0], -1) * r[:, 1]))


def densify_ring(ring: np.ndarray, max_edge: float) -> np.ndarray:
    """Equidistant subdivision of long edges; geomodel.py:353-377 (one ring)."""
    nxt = np.roll(ring, -1, axis=0)
    ln = np.hypot(*(nxt - ring).T)
    pieces = np.maximum(1, np.ceil(ln / max_edge).astype(int))
    if pieces.max() == 1:
        return ring
    out = []
    for p0, p1, q in zip(ring, nxt, pieces):
        t = np.arange(q) / q
        out.append(p0 + t[:, None] * (p1 - p0))
    return np.vstack(out)


# ---------------------------------------------------------------------------
# Flat map + engine (engine.py, temporal.py)
# ---------------------------------------------------------------------------

@dataclass
class FlatMap:
    """Region -> ring -> vertex rows, the order of MapModel.vertex_array (geomodel.py:128-130)."""

    region_ids: list
    region_rings: list  # list (per region) of list of (V,2) float arrays
    stats: np.ndarray

    @classmethod
    def from_mapmodel(cls, m):
        return cls([r.region_id for r in m.regions],
                   [[np.asarray(x, dtype=float) for x in r.rings] for r in m.regions],
                   np.array([r.statistic for r in m.regions], dtype=float))

    def rows(self) -> np.ndarray:
        return np.vstack([ring for rr in self.region_rings for ring in rr])

    def with_rows(self, xy: np.ndarray) -> "FlatMap":
        out, pos = [], 0
        for rr in self.region_rings:
            cur = []
            for ring in rr:
                q = ring.shape[0]
                cur.append(np.array(xy[pos : pos + q], dtype=float))
                pos += q
            out.append(cur)
        if pos != xy.shape[0]:
            raise ValueError("vertex array length mismatch")
        return FlatMap(self.region_ids, out, self.stats)

    def with_stats(self, s) -> "FlatMap":
        return FlatMap(self.region_ids, self.region_rings, np.asarray(s, dtype=float))

    def densified(self, max_edge: float) -> "FlatMap":
        return FlatMap(self.region_ids,
                       [[densify_ring(r, max_edge) for r in rr] for rr in self.region_rings],
                       self.stats)

    def areas(self) -> np.ndarray:
        return np.array([sum(ring_area(r) for r in rr) for rr in self.region_rings])

    def labels(self, k: int) -> np.ndarray:
        return paint_labels(self.region_rings, self.region_ids, k)


@dataclass
class OracleResult:
    rows: np.ndarray
    labels: np.ndarray
    counts: np.ndarray
    region_error: np.ndarray
    epsilon: float
    xi: float
    iteration: int
    clamp_events: int
    stop_reason: str
    trace: list = field(default_factory=list)  # (iteration, epsilon, xi, millis)
    weights_px: np.ndarray | None = None
    background_mass: float = 0.0


class OracleEngine:
    """Restatement of CartogramEngine (engine.py:87-219) on a FlatMap."""

    def __init__(self, fmap: FlatMap, k: int = 10, bdv_multiplier: float = 1.0,
                 background_mass: float | None = None, bdv_mode: str = "fixed-mass",
                 apply_densify: bool = True):
        if bdv_mode not in ("fixed-mass", "rederive"):
            raise ValueError("bdv_mode must be 'fixed-mass' or 'rederive'")
        if bdv_multiplier <= 0:
            raise ValueError("bdv multiplier must be positive")
        self.k, self.n = k, 1 << k
        self.m = self.n * self.n
        self.mult, self.mode = bdv_multiplier, bdv_mode
        if apply_densify:
            fmap = fmap.densified(4.0 / self.n)  # engine.py:24,119-120
        self.fmap = fmap
        self.s = fmap.stats
        self.S = float(self.s.sum())
        if self.S <= 0:
            raise OracleNumericError("total statistic mass must be positive")
        lab0 = fmap.labels(k)
        cnt0 = label_counts(lab0, len(self.s))
        empty = [rid for rid, c in zip(fmap.region_ids, cnt0) if c == 0]
        if empty:  # raster.py:148-154
            raise OracleRasterizationError(
                f"zero-pixel region(s) at resolution {self.n}x{self.n}: {empty} (resolution too low)")
        nbg0 = background_pixels(lab0)
        self.map_pixels0 = self.m - nbg0
        self.background_pixels0 = nbg0
        self.mean_density0 = self.S / self.map_pixels0
        self.background_mass = (float(background_mass) if background_mass is not None
                                else bdv_multiplier * self.mean_density0 * nbg0)
        self.weights_px = self.s / (self.S + self.background_mass) * self.m
        self._lab0 = lab0

    def evaluate(self, fmap: FlatMap, it: int, lab=None):
        """engine.py:143-160."""
        if lab is None:
            lab = fmap.labels(self.k)
        o = label_counts(lab, len(self.s))
        if (o == 0).any():
            raise OracleCollapseError(fmap.region_ids[int(np.argmin(o))], it)
        e = np.abs(o.astype(float) - self.weights_px) / np.maximum(o.astype(float), self.weights_px)
        return dict(fmap=fmap, it=it, lab=lab, o=o, e=e, eps=float(e.mean()), xi=float(e.max()), clamps=0)

    def bdv(self, lab) -> float:
        """engine.py:162-168."""
        nbg = background_pixels(lab)
        if nbg == 0:
            return self.mean_density0 * self.mult
        if self.mode == "fixed-mass":
            return self.background_mass / nbg
        return self.mult * self.S / (self.m - nbg)

    def step(self, st):
        """engine.py:170-180."""
        d = density_texture(self.s, st["lab"], self.bdv(st["lab"]))
        u = displacement(d)
        moved, cl = move_vertices(st["fmap"].rows(), u)
        nxt = self.evaluate(st["fmap"].with_rows(moved), st["it"] + 1)
        nxt["clamps"] = st["clamps"] + cl
        return nxt

    def run(self, error_threshold=0.01, stagnation_window=32, max_iterations=512) -> OracleResult:
        """engine.py:182-219 (fixed-iteration parity runs use threshold 1e-300)."""
        st = self.evaluate(self.fmap, 0, lab=self._lab0)
        trace = []
        best_xi, best_it = np.inf, 0
        best_rows = self.fmap.rows().copy()
        reason = "max-iterations"
        t_prev = time.perf_counter()
        while True:
            now = time.perf_counter()
            trace.append((st["it"], st["eps"], st["xi"], (now - t_prev) * 1e3))
            t_prev = now
            if st["xi"] < best_xi:
                best_xi, best_it = st["xi"], st["it"]
                best_rows = st["fmap"].rows().copy()
            if st["xi"] < error_threshold:
                reason = "converged"
                break
            if st["it"] - best_it >= stagnation_window:
                reason = "stagnation"
                st = self.evaluate(st["fmap"].with_rows(best_rows), best_it)
                break
            if st["it"] >= max_iterations:
                break
            st = self.step(st)
        return OracleResult(rows=st["fmap"].rows(), labels=st["lab"], counts=st["o"],
                            region_error=st["e"], epsilon=st["eps"], xi=st["xi"], iteration=st["it"],
                            clamp_events=st["clamps"], stop_reason=reason, trace=trace,
                            weights_px=self.weights_px, background_mass=self.background_mass)


def default_background_masses(fmap: FlatMap, totals: np.ndarray, k: int, mult: float) -> np.ndarray:
    """temporal.py:151-159 (original map's pixel split)."""
    lab = fmap.labels(k)
    nbg = background_pixels(lab)
    return mult * totals / ((1 << k) ** 2 - nbg) * nbg


def area_fraction_schedule(totals: np.ndarray, a_min: float, a_max: float, window=None):
    """temporal.py:83-102."""
    t0, t1 = window or (0, len(totals) - 1)
    lo = float(totals[t0 : t1 + 1].min())
    hi = float(totals[t0 : t1 + 1].max())
    w = np.ones_like(totals) if hi == lo else np.clip((totals - lo) / (hi - lo), 0.0, 1.0)
    af = (1.0 - w) * a_min + w * a_max
    return totals * (1.0 - af) / af, af


def run_frames(fmap: FlatMap, stats_t: np.ndarray, k: int, cumulative: bool, mult: float = 1.0,
               masses=None, **criteria):
    """Transition modes of temporal.py:162-246 (engine part only, no quality report)."""
    if masses is None:
        masses = default_background_masses(fmap, stats_t.sum(axis=1), k, mult)
    base = fmap.densified(4.0 / (1 << k))
    prev = base
    out = []
    for t in range(stats_t.shape[0]):
        start = (prev if cumulative else base).with_stats(stats_t[t])
        try:
            eng = OracleEngine(start, k=k, background_mass=float(masses[t]), apply_densify=False)
            res = eng.run(**criteria)
            out.append(res)
            if cumulative:
                prev = start.with_rows(res.rows)
        except OracleError as exc:
            out.append(exc)
    return out
