"""Time the GPU frame-report path at the headline map size (3000 regions, ~400k rows).

python tools/metrics_time.py [frames] -- prints one JSON line: ms per frame for the whole
report (frame_reports), the shape kernel alone, adjacency and position error, plus the oracle's
time for one frame's shape distortion on a 200-region sample (CPU, 1 core).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13880_b200 import metrics as M  # noqa: E402
from paper_2604_13880_b200.geomodel import densify, ring_layout  # noqa: E402
from paper_2604_13880_b200.synthetic import config_map  # noqa: E402


def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    base, _ = config_map("headline")
    base = densify(base, 4.0 / 1024)
    xy, rs, rr, ids, stats = ring_layout(base)
    rng = np.random.default_rng(0)
    cart = np.stack([np.clip(xy + rng.normal(0, 0.0003, xy.shape), 0, 1) for _ in range(F)])
    lay = (None, rs, rr, len(ids))
    w = [stats / stats.sum()] * F
    M.frame_reports(base, lay, cart[:1], [stats], w[:1], 7)  # warm-up
    out = {"regions": len(ids), "rows": int(xy.shape[0]), "frames": F}
    t0 = time.perf_counter()
    reps = M.frame_reports(base, lay, cart, [stats] * F, w, 7)
    out["report_ms_per_frame"] = (time.perf_counter() - t0) * 1e3 / F
    assert all(not isinstance(r, Exception) for r in reps), reps[0]
    la, _ = M._layout(base)
    t0 = time.perf_counter()
    M._shapes(la, (cart, rs, rr, len(ids)), 7, True, 0)
    out["shape_ms_per_frame"] = (time.perf_counter() - t0) * 1e3 / F
    row_region = np.repeat(rr, np.diff(rs))
    t0 = time.perf_counter()
    for f in range(F):
        M._ctx(0).adjacency(cart[f], row_region, len(ids), M.DEFAULT_ADJACENCY_EPSILON)
    out["adjacency_ms_per_frame"] = (time.perf_counter() - t0) * 1e3 / F
    cm = np.array(rng.random((len(ids), 2)))
    cc = np.stack([cm + rng.normal(0, 0.01, cm.shape) for _ in range(F)])
    t0 = time.perf_counter()
    M._ctx(0).position_error(cm, cc)
    out["poserr_ms_per_frame"] = (time.perf_counter() - t0) * 1e3 / F
    out["hamming_avg"] = reps[0].hamming_avg
    try:
        from oracle import metrics_oracle as MO

        regs = [[np.asarray(r) for r in reg.rings] for reg in base.regions]
        cb = base.with_vertex_array(cart[0])
        regc = [[np.asarray(r) for r in reg.rings] for reg in cb.regions]
        t0 = time.perf_counter()
        for a, b in zip(regs[:200], regc[:200]):
            MO.hamming(a, b, 7)
        out["oracle_shape_ms_per_frame_est"] = (time.perf_counter() - t0) * 1e3 / 200 * len(ids)
    except Exception as exc:  # noqa: BLE001
        out["oracle_error"] = str(exc)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
