"""Test-only helper: import the reference ``cartomorph`` package in THIS container.

The reference lives read-only at ``/root/reference/pkg/src`` and is absent on
the GPU box, so nothing under ``-m gpu``, ``smoke()`` or ``bench.py`` may use
this module.  It is used by ``tests/golden/make_golden.py`` (to generate the
committed golden fixtures) and by the optional ``live_reference`` tests that
skip when the reference is missing.

``shapely`` is not installed; the reference imports it only for the ingestion
check ``_validate_ring`` (geomodel.py:148-153), which synthetic ``MapModel``
objects never reach.  A stand-in ``shapely.geometry.LineString`` satisfies the
import.  ``NUMBA_CACHE_DIR`` is pointed at a writable directory because the
reference's ``@njit(cache=True)`` would otherwise try to write into the
read-only source tree.
"""

from __future__ import annotations

import os
import sys
import tempfile
import types

REF_SRC = os.environ.get("CARTOMORPH_REF_SRC", "/root/reference/pkg/src")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "cartomorph"))


def import_reference():
    if not reference_available():
        raise ImportError(f"reference not found at {REF_SRC}")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_ref"))
    if "shapely" not in sys.modules:
        shp = types.ModuleType("shapely")
        geo = types.ModuleType("shapely.geometry")

        class LineString:  # minimal stand-in: synthetic maps never hit _validate_ring
            def __init__(self, coords):
                self.coords = coords

            @property
            def is_simple(self):
                return True

        geo.LineString = LineString
        shp.geometry = geo
        sys.modules["shapely"] = shp
        sys.modules["shapely.geometry"] = geo
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import cartomorph  # noqa: E402

    return cartomorph


def to_reference_map(cm, mapmodel):
    """Convert any duck-typed map into a reference ``cartomorph.MapModel``."""
    import numpy as np

    regs = tuple(
        cm.Region(str(r.region_id), str(r.name), tuple(np.asarray(x, dtype=float) for x in r.rings),
                  float(r.statistic))
        for r in mapmodel.regions
    )
    return cm.MapModel(regions=regs)
