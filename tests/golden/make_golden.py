"""Generate the committed golden fixtures from the REAL reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

Everything written here is an *output* of the reference (``cartomorph``,
imported through ``tests/refshim.py``) on seeded inputs, plus those inputs.
No reference source is copied.  The fixtures pin the oracle
(``tests/test_oracle_golden.py``) and the CUDA path (``tests/test_gpu_parity.py``).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from refshim import import_reference, to_reference_map  # noqa: E402
import fixture_maps as fm  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _criteria(cm, iters, thr=1e-300, window=10**9):
    return cm.StoppingCriteria(error_threshold=thr, stagnation_window=window, max_iterations=iters)


def _run_case(cm, m, k, iters, **kw):
    eng = cm.CartogramEngine(to_reference_map(cm, m), criteria=kw.pop("criteria", None) or _criteria(cm, iters), k=k, **kw)
    res = eng.run()
    st = res.state
    tr = np.array([[t.iteration, t.epsilon, t.xi] for t in res.trace])
    return dict(
        init_xy=eng.initial_map.vertex_array(),
        final_xy=st.mapmodel.vertex_array(),
        labels=st.labels.labels.astype(np.int32),
        counts=st.pixel_counts.astype(np.int64),
        region_error=st.per_region_error,
        trace=tr,
        stop=np.array(res.stop_reason),
        iteration=np.array(st.iteration),
        clamps=np.array(st.clamp_events),
        weights_px=res.weights_px,
        background_mass=np.array(res.background_mass),
        areas=np.array([r.area() for r in st.mapmodel.regions]),
    )


def main():
    cm = import_reference()
    from cartomorph import displacement, integral, raster

    rng = np.random.default_rng(1234)

    # 1. stage fixtures at k=6 on a small Voronoi map with shuffled ids
    m = fm.small_voronoi(seed=0, r=24, target=600, shuffle_ids=True)
    rm = to_reference_map(cm, m)
    lab = raster.rasterize_labels(rm, 6)
    dens = raster.build_density(rm.statistics(), lab, 0.8 * raster.default_bdv(rm.statistics(), lab))
    ii = integral.integral_images(dens.d)
    u = displacement.residual_field(ii).u
    rows = rm.vertex_array()
    moved, clamps = displacement.advect(rows, displacement.residual_field(ii))
    np.savez_compressed(
        os.path.join(OUT, "stage_k6.npz"), **fm.pack_map(m), labels=lab.labels, counts=lab.pixel_counts(),
        d=dens.d, channels=np.stack(list(ii.straight_channels()) + list(ii.tilted_channels())), total=ii.total,
        u=u, moved=moved, clamps=clamps, base=displacement.base_mapping(64))

    # 2. raster parity on perturbed vertex sets (k=7), incl. overlaps/holes/multi-ring and ties
    cases = {}
    for name, mm, k in [("overlap", fm.overlap_holes_multi(), 7), ("tie", fm.tie_partition(), 4),
                        ("vor", fm.small_voronoi(seed=3, r=40, target=900), 7)]:
        base = mm.vertex_array()
        for q in range(3):
            xy = base if q == 0 else np.clip(base + rng.normal(0, 0.004, base.shape), 0, 1)
            mq = mm.with_vertex_array(xy)
            lab = raster.rasterize_labels(to_reference_map(cm, mq), k, check_collapse=False)
            for key, val in fm.pack_map(mq).items():
                cases[f"{name}{q}_{key}"] = val
            cases[f"{name}{q}_labels"] = lab.labels
            cases[f"{name}{q}_k"] = np.array(k)
    np.savez_compressed(os.path.join(OUT, "raster_cases.npz"), **cases)

    # 3. engine runs (fixed iteration counts) -- config 1 at k=8, two-region, rederive, stagnation
    runs = {}
    c1 = fm.config1()
    for name, mm, k, iters, kw in [
        ("c1", c1, 8, 20, dict(bdv_multiplier=0.5)),
        ("two", fm.two_region(), 6, 12, {}),
        ("two_rederive", fm.two_region(), 6, 12, dict(bdv_mode="rederive")),
        ("vor_stag", fm.small_voronoi(seed=5, r=16, target=300, shuffle_ids=False), 6, 60,
         dict(criteria=cm.StoppingCriteria(error_threshold=1e-9, stagnation_window=5, max_iterations=200))),
        ("overlap", fm.overlap_holes_multi(), 7, 15, dict(bdv_multiplier=1.3)),
    ]:
        out = _run_case(cm, mm, k, iters, **kw)
        for key, val in fm.pack_map(mm).items():
            runs[f"{name}_in_{key}"] = val
        runs[f"{name}_k"] = np.array(k)
        for key, val in out.items():
            runs[f"{name}_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "engine_runs.npz"), **runs)

    # 4. collapse: the sliver region must collapse at a definite iteration
    try:
        cm.run(to_reference_map(cm, fm.sliver()), cm.StoppingCriteria(error_threshold=1e-6, max_iterations=400), k=5)
        raise SystemExit("expected a collapse")
    except cm.RegionCollapsedError as exc:
        np.savez_compressed(os.path.join(OUT, "collapse.npz"), region=np.array(exc.region_id),
                            iteration=np.array(exc.iteration), message=np.array(str(exc)))

    # 5. temporal: direct + cumulative on a small Voronoi map
    mt = fm.small_voronoi(seed=7, r=12, target=300, shuffle_ids=False)
    s0 = mt.statistics()
    walk = np.stack([s0 * np.exp(np.random.default_rng(70 + t).normal(0, 0.2, s0.shape)) for t in range(3)])
    ds = cm.TimeSeriesDataset(to_reference_map(cm, mt), ("t0", "t1", "t2"), walk)
    tem = dict(fm.pack_map(mt), walk=walk)
    for strat, fn in [("direct", cm.run_direct), ("cumulative", cm.run_cumulative)]:
        seq = fn(ds, _criteria(cm, 8), k=6, bdv_multiplier=1.0)
        for t, fr in enumerate(seq.frames):
            tem[f"{strat}_{t}_xy"] = fr.mapmodel.vertex_array()
            tem[f"{strat}_{t}_counts"] = fr.result.state.pixel_counts
            tem[f"{strat}_{t}_mb"] = np.array(fr.background_mass)
    np.savez_compressed(os.path.join(OUT, "temporal.npz"), **tem)
    # 6. output format: GeoJSON bytes of a holed/multi-ring map and of a deformed config-1 frame
    from cartomorph.geomodel import to_geojson

    gj = {}
    for name, mm in [("overlap", fm.overlap_holes_multi()), ("c1", fm.config1())]:
        rm = to_reference_map(cm, mm)
        if name == "c1":
            rm = rm.with_vertex_array(runs["c1_final_xy"])
        gj[name] = np.frombuffer(to_geojson(rm, extra_properties={rm.regions[0].region_id: {"x": 1}}), dtype=np.uint8)
        for key, val in fm.pack_map(mm).items():
            gj[f"{name}_{key}"] = val
    gj["c1_final_xy"] = runs["c1_final_xy"]
    np.savez_compressed(os.path.join(OUT, "geojson.npz"), **gj)
    # 7. frame quality metrics (metrics.py:29-260, geomodel.py:380-415): full reports of map/cartogram pairs
    from cartomorph import metrics as cmet
    from cartomorph.geomodel import detect_adjacencies

    met = {}
    eps_adj = cmet.DEFAULT_ADJACENCY_EPSILON

    def idx_pairs(edges, ids):
        pos = {rid: i for i, rid in enumerate(ids)}
        out = sorted(tuple(sorted((pos[a], pos[b]))) for a, b in edges)
        return np.array(out, dtype=np.int32).reshape(-1, 2)

    def save_pair(name, mm, cxy, k, rescale=True):
        rm = to_reference_map(cm, mm)
        rc = rm.with_vertex_array(cxy)
        for key, val in fm.pack_map(mm).items():
            met[f"{name}_m_{key}"] = val
        met[f"{name}_c_xy"] = np.asarray(cxy, dtype=float)
        met[f"{name}_k"] = np.array(k)
        met[f"{name}_rescale"] = np.array(rescale)
        vals, avg, mx = cmet.shape_distortion(rm, rc, raster_k=k, rescale=rescale)
        met[f"{name}_hamming"] = vals
        rep = cmet.full_report(rm, rc, raster_k=k, rescale_shapes=rescale)
        met[f"{name}_json"] = np.array(rep.to_json())
        met[f"{name}_csv"] = np.array(rep.to_csv())
        met[f"{name}_areas"] = np.array([r.area() for r in rc.regions])
        met[f"{name}_cent_m"] = np.array([r.centroid() for r in rm.regions])
        met[f"{name}_cent_c"] = np.array([r.centroid() for r in rc.regions])
        ids = rm.region_ids()
        met[f"{name}_adj_m"] = idx_pairs(detect_adjacencies(rm, eps_adj), ids)
        met[f"{name}_adj_c"] = idx_pairs(detect_adjacencies(rc, eps_adj), ids)
        met[f"{name}_poserr"] = np.array(cmet.relative_position_error(rm, rc))

    save_pair("c1", c1, runs["c1_final_xy"], 7)
    save_pair("c1_k6_raw", c1, runs["c1_final_xy"], 6, rescale=False)
    mo = fm.overlap_holes_multi()
    save_pair("overlap", mo, np.clip(mo.vertex_array() + rng.normal(0, 0.003, mo.vertex_array().shape), 0, 1), 7)
    mv = fm.small_voronoi(seed=11, r=40, target=900)
    save_pair("vor_k8", mv, np.clip(mv.vertex_array() + rng.normal(0, 0.002, mv.vertex_array().shape), 0, 1), 8)
    mt2 = fm.two_region()
    save_pair("two", mt2, mt2.vertex_array() * np.array([1.0, 0.9]) + np.array([0.02, 0.03]), 5)
    # square vs disk (test_metrics.py:103-117) at k=6
    theta = np.linspace(0.0, 2 * np.pi, 96, endpoint=False)
    radius = 0.4 / np.sqrt(np.pi)
    sq = [np.array([[0.3, 0.3], [0.7, 0.3], [0.7, 0.7], [0.3, 0.7]])]
    disk = [np.stack([0.5 + radius * np.cos(theta), 0.5 + radius * np.sin(theta)], axis=1)]
    met["sqdisk_a"], met["sqdisk_b"] = sq[0], disk[0]
    met["sqdisk_hamming"] = np.array(cmet.hamming_distance(sq, disk, raster_k=6))
    met["sqdisk_hamming_raw"] = np.array(cmet.hamming_distance(sq, disk, raster_k=6, rescale=False))
    # a clockwise (negative-area) region: NumericError from the rescale
    try:
        cmet.hamming_distance([sq[0][::-1]], disk, raster_k=6)
        raise SystemExit("expected NumericError")
    except cm.NumericError as exc:
        met["neg_area_message"] = np.array(str(exc))
    np.savez_compressed(os.path.join(OUT, "metrics.npz"), **met)

    # 8. temporal frames with their reports and watchdog flags (temporal.py:200-228)
    tr = dict(fm.pack_map(mt), walk=walk)
    for strat, fn in [("direct", cm.run_direct), ("cumulative", cm.run_cumulative)]:
        seq = fn(ds, _criteria(cm, 8), k=6, bdv_multiplier=1.0, watchdog_ceiling=0.02, report_raster_k=6)
        for t, fr in enumerate(seq.frames):
            tr[f"{strat}_{t}_report"] = np.array(fr.report.to_json())
            tr[f"{strat}_{t}_watchdog"] = np.array(fr.watchdog)
        tr[f"{strat}_series"] = np.array(json.dumps(seq.series(), sort_keys=True))
    np.savez_compressed(os.path.join(OUT, "temporal_reports.npz"), **tr)
    # 9. one steering-service frame (service.py:202-236 composition): engine + report + GeoJSON
    from cartomorph.geomodel import to_geojson as ref_geojson

    ms = fm.small_voronoi(seed=13, r=14, target=400, shuffle_ids=False)
    rbase = to_reference_map(cm, ms)
    sv = {}
    for key, val in fm.pack_map(ms).items():
        sv[f"m_{key}"] = val
    for t, (mass, k, hk, strat) in enumerate([(0.3, 6, 6, "direct"), (0.6, 7, 5, "direct")]):
        stats_t = ms.statistics() * np.exp(np.random.default_rng(90 + t).normal(0, 0.3, len(ms.regions)))
        eng = cm.CartogramEngine(rbase.with_statistics(stats_t),
                                 criteria=cm.StoppingCriteria(1e-300, 10**9, 12), k=k,
                                 background_mass=mass, apply_densify=False)
        res = eng.run()
        carto = res.state.mapmodel
        weights = stats_t / (float(stats_t.sum()) + mass)
        rep = cmet.full_report(rbase.with_statistics(stats_t), carto, weights=weights, raster_k=hk, wall_ms=1.0)
        sv[f"f{t}_stats"] = stats_t
        sv[f"f{t}_cfg"] = np.array([mass, k, hk])
        sv[f"f{t}_report"] = np.array(json.dumps(rep.to_dict(), sort_keys=True))
        sv[f"f{t}_geojson"] = np.array(ref_geojson(carto, rep.per_region).decode())
        sv[f"f{t}_xy"] = carto.vertex_array()
        sv[f"f{t}_stop"] = np.array(res.stop_reason)
    np.savez_compressed(os.path.join(OUT, "service_frames.npz"), **sv)

    # 10. the bdv multiplier sweep of cli.py:265-300 (engine + report per multiplier, CSV rows)
    msw = fm.small_voronoi(seed=21, r=12, target=500, shuffle_ids=False)
    rsw = to_reference_map(cm, msw)
    sw = dict(fm.pack_map(msw))
    rows = []
    for mult in [0.5, 1.0, 1.7]:
        eng = cm.CartogramEngine(rsw, criteria=cm.StoppingCriteria(0.01, 32, 15), k=6, bdv_multiplier=mult)
        res = eng.run()
        weights = rsw.statistics() / (eng.total_statistic + eng.background_mass)
        rep = cmet.full_report(eng.initial_map, res.state.mapmodel, weights=weights, raster_k=6, wall_ms=0.0)
        rows.append(f"{mult:.6g},{res.stop_reason},{res.state.iteration},{res.state.xi:.9g},{res.state.epsilon:.9g},"
                    f"{rep.tau:.9g},{rep.hamming_avg:.9g},{rep.hamming_max:.9g},{rep.position_error:.9g}")
    sw["rows"] = np.array(rows)
    np.savez_compressed(os.path.join(OUT, "sweep.npz"), **sw)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
