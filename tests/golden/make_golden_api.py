"""Golden fixtures for the stage API members added in round 2, from the REAL reference.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden_api.py      -> tests/golden/api.npz

Covers ``mapping_grid`` / ``mapping_point`` / ``residual_field(ii, base)`` on the channel set of
``stage_k6.npz`` and on a hand-built IntegralImageSet (no texture behind it), and
``Region.centroid`` of a holed / multi-ring map.  Only reference outputs and their seeded inputs
are written.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from refshim import import_reference, to_reference_map  # noqa: E402
import fixture_maps as fm  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    cm = import_reference()
    from cartomorph import displacement, integral

    st = np.load(os.path.join(OUT, "stage_k6.npz"))
    ch, total = st["channels"], float(st["total"])
    ii = integral.IntegralImageSet(*[ch[i] for i in range(8)], total=total)
    rng = np.random.default_rng(77)
    # points: random, the four corners, edge midpoints, both diagonals, pixel centres and corners
    pts = [rng.uniform(0, 1, 2) for _ in range(40)]
    pts += [np.array(p, float) for p in [(0, 0), (1, 1), (0, 1), (1, 0), (0.5, 0), (0, 0.5), (1, 0.5), (0.5, 1),
                                         (0.25, 0.25), (0.3, 0.7), (0.7, 0.3), (0.5, 0.5),
                                         (0.5 / 64, 0.5 / 64), (3 / 64, 17 / 64), (63.5 / 64, 0.5 / 64)]]
    pts = np.array(pts)
    mp = np.array([displacement.mapping_point(float(x), float(y), ii) for x, y in pts])
    grid = displacement.mapping_grid(ii)
    base = displacement.base_mapping(64)
    # a non-default base: the residual against a shifted base grid
    base2 = base + rng.normal(0, 1e-3, base.shape)
    u_base2 = displacement.residual_field(ii, base2).u
    u_none = displacement.residual_field(ii).u

    # a hand-built set: random positive channels that are not the channels of any texture
    hch = rng.uniform(0.1, 2.0, (8, 16, 16))
    htot = 37.5
    hii = integral.IntegralImageSet(*[hch[i] for i in range(8)], total=htot)
    hgrid = displacement.mapping_grid(hii)
    hpts = rng.uniform(0, 1, (12, 2))
    hmp = np.array([displacement.mapping_point(float(x), float(y), hii) for x, y in hpts])

    m = fm.overlap_holes_multi()
    rm = to_reference_map(cm, m)
    cents = np.array([r.centroid() for r in rm.regions])
    vor = to_reference_map(cm, fm.small_voronoi(seed=0, r=24, target=600, shuffle_ids=True))
    vcents = np.array([r.centroid() for r in vor.regions])

    np.savez_compressed(os.path.join(OUT, "api.npz"), pts=pts, mapping_point=mp, mapping_grid=grid, base2=base2,
                        u_base2=u_base2, u_none=u_none, h_channels=hch, h_total=htot, h_grid=hgrid, h_pts=hpts,
                        h_mapping_point=hmp, centroids_overlap=cents, centroids_vor=vcents)
    print("written", os.path.join(OUT, "api.npz"))


if __name__ == "__main__":
    main()
