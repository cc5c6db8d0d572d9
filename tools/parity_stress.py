"""Randomised parity stress of the CUDA path against the oracle (diagnostics, not a CI test).

python tools/parity_stress.py [seconds] -- loops over random maps (Voronoi with shuffled ids,
2-60 regions, random vertex jitter that creates overlaps/self-touching rings) and texture sizes
k = 4..9:
  * raster: GPU labels vs oracle labels (bit-exact) for the jittered geometry;
  * engine: 4 float64-field iterations vs the oracle engine (counts and trace bit-exact,
    vertices within 1e-9).
Prints one JSON line with the case counts and the first mismatch (if any).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import fixture_maps as fm  # noqa: E402
import paper_2604_13880_b200 as P  # noqa: E402
from oracle import det_oracle as O  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(time.time()) % 100000)
    seed0 = int(rng.integers(1 << 30))
    t0 = time.perf_counter()
    stats = {"seed0": seed0, "raster_cases": 0, "engine_cases": 0, "mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and stats["mismatch"] is None:
        r = np.random.default_rng(seed0 + i)
        i += 1
        nreg = int(r.integers(2, 60))
        m = fm.small_voronoi(seed=int(r.integers(1 << 20)), r=nreg, target=int(r.integers(100, 1500)))
        k = int(r.integers(4, 10))
        jit = float(r.choice([0.0, 0.001, 0.004, 0.01]))
        xy = np.clip(m.vertex_array() + r.normal(0, jit, m.vertex_array().shape), 0, 1)
        mj = m.with_vertex_array(xy)
        try:
            lab = P.rasterize_labels(mj, k, check_collapse=False).labels
        except Exception as exc:  # noqa: BLE001
            f = O.FlatMap.from_mapmodel(mj)
            try:
                f.labels(k)
                stats["mismatch"] = {"case": i, "kind": "gpu raised", "err": str(exc)[:200]}
            except Exception:  # noqa: BLE001 -- both raise: consistent
                pass
            continue
        ref = O.FlatMap.from_mapmodel(mj).labels(k)
        stats["raster_cases"] += 1
        if not np.array_equal(np.asarray(lab), ref):
            stats["mismatch"] = {"case": i, "kind": "raster", "k": k, "regions": nreg, "jitter": jit,
                                 "pixels": int((np.asarray(lab) != ref).sum())}
            break
        if jit == 0.0 and k >= 5:  # engine trajectories on clean partitions
            crit = P.StoppingCriteria(1e-300, 10**9, 4)
            try:
                res = P.CartogramEngine(m, criteria=crit, k=k, field_dtype="float64").run()
            except P.CartomorphError:
                continue
            eng = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=k)
            ores = eng.run(error_threshold=1e-300, stagnation_window=10**9, max_iterations=4)
            stats["engine_cases"] += 1
            ok = (np.array_equal(res.state.pixel_counts, ores.counts) and
                  np.abs(res.state.mapmodel.vertex_array() - ores.rows).max() <= 1e-9)
            if not ok:
                stats["mismatch"] = {"case": i, "kind": "engine", "k": k, "regions": nreg}
    stats["seconds"] = time.perf_counter() - t0
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
