"""Randomised parity stress of the CUDA path against the oracle (diagnostics, not a CI test).

python tools/parity_stress.py [seconds] -- loops over random maps (Voronoi with shuffled ids,
2-60 regions, random vertex jitter that creates overlaps/self-touching rings) and texture sizes
k = 4..9:
  * raster: GPU labels vs oracle labels (bit-exact) for the jittered geometry;
  * engine: 4 float64-field iterations vs the oracle engine (counts and trace bit-exact,
    vertices within 1e-9).
Prints one JSON line with the case counts and the first mismatch (if any).

PARITY_FIELD=float32 (or mixed) runs the engine / temporal sections in that field mode and holds
them to the north-star bars instead of trajectory identity: vertices within 1e-4, per-region
shoelace areas within 1e-3 relative (runs whose stop reason or collapse differs from the oracle's
are counted, not failed -- a float32 trajectory may cross a threshold one iteration apart).
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

FIELD = os.environ.get("PARITY_FIELD", "float64")
# STRESS_K="lo,hi": texture exponents of the raster/engine and random-criteria sections (default 4..9 and
# 5..7); "9,11" puts every engine case on the float64 band kernels of n >= 512 (k_sat1x, k_sat3x)
_KR = [int(v) for v in os.environ["STRESS_K"].split(",")] if os.environ.get("STRESS_K") else None


def _k(r, lo, hi):
    return int(r.integers(_KR[0], _KR[1])) if _KR else int(r.integers(lo, hi))


def _areas(rows, m):
    from paper_2604_13880_b200.geomodel import ring_layout

    _, rs, rr, ids, _ = ring_layout(m)
    out = np.zeros(len(ids))
    for q in range(len(rs) - 1):
        p = rows[rs[q] : rs[q + 1]]
        if p.shape[0] >= 3:
            nx = np.roll(p, -1, axis=0)
            out[rr[q]] += 0.5 * float(np.sum(p[:, 0] * nx[:, 1] - nx[:, 0] * p[:, 1]))
    return out


def _within_bars(rows, ref_rows, m, out):
    """float32/mixed: the north-star bars on one final state; tracks the worst deviations."""
    dv = float(np.abs(rows - ref_rows).max())
    a, ar = _areas(rows, m), _areas(ref_rows, m)
    da = float((np.abs(a - ar) / np.maximum(np.abs(ar), 1e-300)).max())
    out["max_vertex_dev"] = max(out.get("max_vertex_dev", 0.0), dv)
    out["max_area_rel"] = max(out.get("max_area_rel", 0.0), da)
    return dv <= 1e-4 and da <= 1e-3
import paper_2604_13880_b200 as P  # noqa: E402
from oracle import det_oracle as O  # noqa: E402


def metrics_stress(budget, seed0):
    """Random map pairs: GPU Hamming values (k 3..8, rescale on/off) and adjacency sets vs the oracle."""
    from oracle import metrics_oracle as MO
    from paper_2604_13880_b200 import detect_adjacencies, shape_distortion

    t0 = time.perf_counter()
    out = {"metric_cases": 0, "metric_regions": 0, "metric_mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and out["metric_mismatch"] is None:
        r = np.random.default_rng(seed0 + 7919 * i)
        i += 1
        m = fm.small_voronoi(seed=int(r.integers(1 << 20)), r=int(r.integers(2, 40)), target=int(r.integers(100, 1200)))
        c = m.with_vertex_array(np.clip(m.vertex_array() + r.normal(0, float(r.choice([0.001, 0.005, 0.02])),
                                                                     m.vertex_array().shape), 0, 1))
        k, resc = int(r.integers(3, 9)), bool(r.integers(2))
        rm = [[np.asarray(x) for x in reg.rings] for reg in m.regions]
        rc = [[np.asarray(x) for x in reg.rings] for reg in c.regions]
        try:
            want = np.array([MO.hamming(a, b, k, resc) for a, b in zip(rm, rc)])
        except Exception:  # noqa: BLE001 -- degenerate shape: the GPU must raise as well
            try:
                shape_distortion(m, c, raster_k=k, rescale=resc)
                out["metric_mismatch"] = {"case": i, "kind": "oracle raised, gpu did not"}
            except Exception:  # noqa: BLE001
                pass
            continue
        got, _, _ = shape_distortion(m, c, raster_k=k, rescale=resc)
        out["metric_cases"] += 1
        out["metric_regions"] += len(rm)
        if not np.array_equal(got, want):
            out["metric_mismatch"] = {"case": i, "kind": "hamming", "k": k, "rescale": resc,
                                      "regions": int((got != want).sum())}
            break
        pos = {rid: q for q, rid in enumerate(c.region_ids())}
        adj = {tuple(sorted((pos[a], pos[b]))) for a, b in detect_adjacencies(c, 0.5 / 1024)}
        if adj != MO.adjacency(rc, 0.5 / 1024):
            out["metric_mismatch"] = {"case": i, "kind": "adjacency"}
    return out


def engine_stress(budget, seed0):
    """Random stopping criteria, bdv modes and multipliers (float64 field): stop reason, stop
    iteration, counts and collapse region equal the oracle engine's; vertices within 1e-9."""
    t0 = time.perf_counter()
    out = {"engine_runs": 0, "stops": {}, "engine_mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and out["engine_mismatch"] is None:
        r = np.random.default_rng(seed0 + 104729 * i)
        i += 1
        m = fm.small_voronoi(seed=int(r.integers(1 << 20)), r=int(r.integers(2, 30)), target=int(r.integers(100, 900)))
        m = m.with_statistics(np.exp(r.normal(0, float(r.choice([0.5, 1.5, 3.0])), len(m.regions))))
        k = _k(r, 5, 8)
        mode = str(r.choice(["fixed-mass", "rederive"]))
        mult = float(r.choice([0.3, 1.0, 2.0]))
        thr = float(r.choice([1e-300, 0.05, 0.2]))
        win = int(r.choice([3, 8, 10**9]))
        its = int(r.integers(5, 40))
        crit = P.StoppingCriteria(thr, win, its)
        try:
            res = P.CartogramEngine(m, criteria=crit, k=k, bdv_multiplier=mult, bdv_mode=mode,
                                    field_dtype=FIELD).run()
            got = ("ok", res.stop_reason, res.state.iteration, res.state.pixel_counts, res.state.mapmodel.vertex_array())
        except P.RegionCollapsedError as exc:
            got = ("collapse", exc.region_id, exc.iteration, None, None)
        except Exception as exc:  # noqa: BLE001
            got = ("error", type(exc).__name__, str(exc), None, None)
        f = O.FlatMap.from_mapmodel(m)
        try:
            ores = O.OracleEngine(f, k=k, bdv_multiplier=mult, bdv_mode=mode).run(thr, win, its)
            want = ("ok", ores.stop_reason, ores.iteration, ores.counts, ores.rows)
        except O.OracleCollapseError as exc:
            want = ("collapse", exc.region_id, exc.iteration, None, None)
        except Exception as exc:  # noqa: BLE001 -- the oracle's error types carry an "Oracle" prefix
            want = ("error", type(exc).__name__.replace("Oracle", "", 1), str(exc), None, None)
        out["engine_runs"] += 1
        key = got[0] + ":" + str(got[1])
        out["stops"][key] = out["stops"].get(key, 0) + 1
        if FIELD != "float64":
            if got[0] == "ok" and want[0] == "ok" and got[1:3] == want[1:3]:
                same = _within_bars(got[4], want[4], m, out)
            else:
                out["divergent_stops"] = out.get("divergent_stops", 0) + (got[:3] != want[:3])
                same = True
        else:
            same = got[:3] == want[:3] if got[0] != "ok" else (
                got[:3] == want[:3] and np.array_equal(got[3], want[3]) and np.abs(got[4] - want[4]).max() <= 1e-9)
        if not same:
            out["engine_mismatch"] = {"case": i, "got": [str(x)[:80] for x in got[:3]],
                                      "want": [str(x)[:80] for x in want[:3]], "k": k, "mode": mode,
                                      "mult": mult, "thr": thr, "win": win, "its": its}
    return out


def temporal_stress(budget, seed0):
    """Direct / cumulative frame sequences (float64 field) vs the oracle's run_frames: per frame the
    same success/failure, counts equal, vertices within 1e-9 (a frame failing only in its quality
    report -- outside the oracle's engine-only restatement -- ends the comparison of that sequence)."""
    t0 = time.perf_counter()
    out = {"sequences": 0, "frames": 0, "failed_frames": 0, "report_failures": 0, "temporal_mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and out["temporal_mismatch"] is None:
        r = np.random.default_rng(seed0 + 15485863 * i)
        i += 1
        m = fm.small_voronoi(seed=int(r.integers(1 << 20)), r=int(r.integers(3, 25)), target=int(r.integers(150, 700)))
        T, k = 4, int(r.integers(5, 7))
        sig = float(r.choice([0.1, 0.5, 1.5]))
        s0 = m.statistics()
        walk = np.stack([s0 * np.exp(r.normal(0, sig, s0.shape)) for _ in range(T)])
        cumulative = bool(r.integers(2))
        crit = P.StoppingCriteria(1e-300, 10**9, 6)
        ds = P.TimeSeriesDataset(m, tuple(f"t{q}" for q in range(T)), walk)
        fn = P.run_cumulative if cumulative else P.run_direct
        try:
            seq = fn(ds, crit, k=k, field_dtype=FIELD)
        except P.RasterizationError:
            # the original map has a zero-pixel region at this resolution: the reference raises the same
            # error while deriving the background masses (temporal.py:151-159); the oracle's split must agree
            if (O.FlatMap.from_mapmodel(m).labels(k) >= 0).sum() and len(np.unique(O.FlatMap.from_mapmodel(m).labels(k))) - 1 == len(m.regions):
                out["temporal_mismatch"] = {"case": i, "kind": "gpu raised RasterizationError, oracle has every region"}
            out["setup_raster_errors"] = out.get("setup_raster_errors", 0) + 1
            continue
        ref = O.run_frames(O.FlatMap.from_mapmodel(m), walk, k, cumulative, error_threshold=1e-300,
                           stagnation_window=10**9, max_iterations=6)
        out["sequences"] += 1
        for t, (fr, rf) in enumerate(zip(seq.frames, ref)):
            out["frames"] += 1
            if isinstance(rf, Exception):
                out["failed_frames"] += 1
                if fr.error != str(rf):
                    out["temporal_mismatch"] = {"case": i, "t": t, "ours": str(fr.error)[:120], "oracle": str(rf)[:120]}
                    break
                continue
            if fr.error is not None:
                if any(w in fr.error for w in ("Hamming", "non-positive area", "cartographic error", "position error")):
                    out["report_failures"] += 1
                    break
                out["temporal_mismatch"] = {"case": i, "t": t, "ours": fr.error[:120], "oracle": "ok"}
                break
            if FIELD != "float64":
                ok = _within_bars(fr.mapmodel.vertex_array(), rf.rows, m, out)
            else:
                ok = (np.array_equal(fr.result.state.pixel_counts, rf.counts) and
                      np.abs(fr.mapmodel.vertex_array() - rf.rows).max() <= 1e-9)
            if not ok:
                out["temporal_mismatch"] = {"case": i, "t": t, "kind": "state", "cumulative": cumulative, "k": k}
                break
    return out


def polygon_stress(budget, seed0):
    """Random star / self-intersecting rings, holes, overlapping regions, shuffled ids, k 4..9:
    GPU labels vs oracle labels (bit-exact), or the same ValueError."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_live_reference import _random_map

    t0 = time.perf_counter()
    out = {"polygon_cases": 0, "raised_both": 0, "polygon_mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and out["polygon_mismatch"] is None:
        r = np.random.default_rng(seed0 + 31337 * i)
        i += 1
        m = _random_map(r, int(r.integers(1, 12)))
        k = int(r.integers(4, 10))
        try:
            want = O.FlatMap.from_mapmodel(m).labels(k)
        except ValueError:
            try:
                P.rasterize_labels(m, k, check_collapse=False)
                out["polygon_mismatch"] = {"case": i, "kind": "oracle raised, gpu did not"}
            except ValueError:
                out["raised_both"] += 1
            continue
        got = np.asarray(P.rasterize_labels(m, k, check_collapse=False).labels)
        out["polygon_cases"] += 1
        if not np.array_equal(got, want):
            out["polygon_mismatch"] = {"case": i, "k": k, "pixels": int((got != want).sum())}
    return out


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    if len(sys.argv) > 2 and sys.argv[2] == "polygons":
        print(json.dumps(polygon_stress(budget, int(time.time()) % 100000)))
        return
    if len(sys.argv) > 2 and sys.argv[2] == "temporal":
        print(json.dumps(temporal_stress(budget, int(time.time()) % 100000)))
        return
    if len(sys.argv) > 2 and sys.argv[2] == "engine":
        print(json.dumps(engine_stress(budget, int(time.time()) % 100000)))
        return
    if len(sys.argv) > 2 and sys.argv[2] == "metrics":
        print(json.dumps(metrics_stress(budget, int(time.time()) % 100000)))
        return
    rng = np.random.default_rng(int(time.time()) % 100000)
    seed0 = int(rng.integers(1 << 30))
    t0 = time.perf_counter()
    stats = {"seed0": seed0, "field": FIELD, "raster_cases": 0, "engine_cases": 0, "mismatch": None}
    i = 0
    while time.perf_counter() - t0 < budget and stats["mismatch"] is None:
        r = np.random.default_rng(seed0 + i)
        i += 1
        nreg = int(r.integers(2, 60))
        m = fm.small_voronoi(seed=int(r.integers(1 << 20)), r=nreg, target=int(r.integers(100, 1500)))
        k = _k(r, 4, 10)
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
                res = P.CartogramEngine(m, criteria=crit, k=k, field_dtype=FIELD).run()
            except P.CartomorphError:
                continue
            eng = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=k)
            ores = eng.run(error_threshold=1e-300, stagnation_window=10**9, max_iterations=4)
            stats["engine_cases"] += 1
            if FIELD != "float64":
                ok = _within_bars(res.state.mapmodel.vertex_array(), ores.rows, m, stats)
            else:
                ok = (np.array_equal(res.state.pixel_counts, ores.counts) and
                      np.abs(res.state.mapmodel.vertex_array() - ores.rows).max() <= 1e-9)
            if not ok:
                stats["mismatch"] = {"case": i, "kind": "engine", "k": k, "regions": nreg}
    stats["seconds"] = time.perf_counter() - t0
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
