"""Integral images -- drop-in for cartomorph/integral.py, computed on the GPU.

``integral_images(d)`` (integral.py:155-169) returns the eight straight and
45-degree-tilted channels of a dense texture from the sm_100a band kernels
(``k_sat1..3`` in csrc/det_sat.cuh, debug output mode); the engine itself never
materialises them and goes straight to the displacement field.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._context import get_context


@dataclass(frozen=True)
class IntegralImageSet:
    alpha: np.ndarray
    beta: np.ndarray
    gamma: np.ndarray
    delta: np.ndarray
    alpha_t: np.ndarray
    beta_t: np.ndarray
    gamma_t: np.ndarray
    delta_t: np.ndarray
    total: float
    source: np.ndarray | None = field(default=None, repr=False, compare=False)

    @property
    def size(self) -> int:
        return self.alpha.shape[0]

    def straight_channels(self):
        return (self.alpha, self.beta, self.gamma, self.delta)

    def tilted_channels(self):
        return (self.alpha_t, self.beta_t, self.gamma_t, self.delta_t)


def _k_of(n: int) -> int:
    if n < 16 or n & (n - 1):
        raise ValueError("texture size must be a power of two >= 16 (k in [4, 13])")
    return n.bit_length() - 1


def integral_images(d: np.ndarray, device: int = 0) -> IntegralImageSet:
    d = np.ascontiguousarray(d, dtype=np.float64)
    if d.ndim != 2 or d.shape[0] != d.shape[1]:
        raise ValueError("density texture must be square")
    ctx = get_context(_k_of(d.shape[0]), device)
    ch, tot = ctx.channels(d)
    return IntegralImageSet(*[ch[i] for i in range(8)], total=float(tot), source=d)


def straight_inims(d: np.ndarray, device: int = 0):
    ii = integral_images(d, device)
    return ii.alpha, ii.beta, ii.gamma, ii.delta, ii.total


def tilted_inims(d: np.ndarray, device: int = 0):
    return integral_images(d, device).tilted_channels()
