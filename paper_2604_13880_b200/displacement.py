"""Displacement field and advection -- drop-in for cartomorph/displacement.py on the GPU.

``residual_field`` (displacement.py:198-206) evaluates u = t(d) - t(const) at
every pixel centre with the band kernels (residual-density form, float64);
``advect`` (displacement.py:229-238) runs ``k_advect_points``.  Inside the
engine both are fused into k_sat3 / k_region and never leave the device.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field

import numpy as np

from ._context import get_context
from .errors import NumericError
from .integral import IntegralImageSet, _k_of


@dataclass(frozen=True)
class AnchorSet:
    q1: tuple
    q2: tuple
    q3: tuple
    q4: tuple
    e1: tuple
    e2: tuple
    e3: tuple
    e4: tuple


def anchors(x: float, y: float) -> AnchorSet:
    """Border anchors of (x, y), y-down (displacement.py:35-53)."""
    if y < x:
        q1, q3 = (1.0, 1.0 + y - x), (x - y, 0.0)
    else:
        q1, q3 = (1.0 - y + x, 1.0), (0.0, y - x)
    if x + y < 1.0:
        q2, q4 = (x + y, 0.0), (0.0, x + y)
    else:
        q2, q4 = (1.0, x + y - 1.0), (x + y - 1.0, 1.0)
    return AnchorSet(q1, q2, q3, q4, (x, 1.0), (1.0, y), (x, 0.0), (0.0, y))


@dataclass
class DisplacementField:
    """Per-pixel displacement u = t(d) - t(d0) at pixel centres (displacement.py:186-195)."""

    size: int
    u: np.ndarray
    base: np.ndarray = field(repr=False, default=None)

    def max_magnitude(self) -> float:
        return float(np.hypot(self.u[..., 0], self.u[..., 1]).max())


def _channel_stack(ii: IntegralImageSet) -> np.ndarray:
    return np.stack(ii.straight_channels() + ii.tilted_channels())


def mapping_grid(ii: IntegralImageSet, device: int = 0) -> np.ndarray:
    """t(d) at every pixel centre, (n, n, 2), from the set's eight channels (displacement.py:102-131).

    ``k_map_grid`` evaluates the reference's corner-lattice average and anchor combination with
    its float64 op order, so any IntegralImageSet -- a hand-built one included -- maps exactly as
    the reference maps it."""
    if ii.total <= 0:
        raise NumericError("mapping undefined for zero total density")
    return get_context(_k_of(ii.size), device).mapping_channels(_channel_stack(ii), ii.total)


def mapping_point(x: float, y: float, ii: IntegralImageSet, device: int = 0) -> np.ndarray:
    """The anchor mapping at one continuous location (displacement.py:150-170): straight channels
    sampled on the corner lattice, tilted channels between pixel centres (``k_map_points``)."""
    if ii.total <= 0:
        raise NumericError("mapping undefined for zero total density")
    ctx = get_context(_k_of(ii.size), device)
    return ctx.mapping_points(_channel_stack(ii), ii.total, np.array([[x, y]], dtype=np.float64))[0]


@functools.lru_cache(maxsize=8)
def base_mapping(n: int) -> np.ndarray:
    """Mapping of a constant texture, cached per resolution (displacement.py:173-183)."""
    grid = get_context(_k_of(n)).mapping(np.ones((n, n)))
    grid.setflags(write=False)
    return grid


def residual_field(ii_d: IntegralImageSet, base: np.ndarray | None = None, device: int = 0) -> DisplacementField:
    """u = t(d) - base at every pixel centre (displacement.py:198-206).

    With ``base=None`` and a set built by :func:`integral_images` (which keeps its texture), u is
    evaluated by the engine's band kernels in residual-density form, which avoids the cancellation
    of t(d) - t(1) (agrees with the reference's subtraction to ~1e-13).  Otherwise u is the
    channel mapping minus ``base`` (``base_mapping(n)`` when None), exactly the reference's
    expression."""
    n = ii_d.size
    if base is not None and base.shape[0] != n:
        raise ValueError(f"base grid size {base.shape[0]} does not match texture size {n}")
    if ii_d.total <= 0:
        raise NumericError("mapping undefined for zero total density")
    ctx = get_context(_k_of(n), device)
    if base is None and ii_d.source is not None:
        u, _, _ = ctx.field(ii_d.source)
        return DisplacementField(size=n, u=u, base=base_mapping(n))
    if base is None:
        base = base_mapping(n)
    u = ctx.mapping_channels(_channel_stack(ii_d), ii_d.total, base)
    return DisplacementField(size=n, u=u, base=base)


def advect(vertices: np.ndarray, fld: DisplacementField, device: int = 0):
    """Move vertices by the bilinearly sampled field, clamp to [0,1]^2; returns (moved, clamp count)."""
    verts = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 2)
    return get_context(_k_of(fld.size), device).advect(fld.u, verts)
