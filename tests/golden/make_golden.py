"""Generate the committed golden fixtures from the REAL reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

Everything written here is an *output* of the reference (``cartomorph``,
imported through ``tests/refshim.py``) on seeded inputs, plus those inputs.
No reference source is copied.  The fixtures pin the oracle
(``tests/test_oracle_golden.py``) and the CUDA path (``tests/test_gpu_parity.py``).
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
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
