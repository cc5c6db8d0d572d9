"""Pin the CPU oracle against fixtures produced by the real reference.

These run without a GPU.  The oracle restates the reference's float64
arithmetic op-for-op, so labels/counts are compared bit-exactly and the
float fields at 1e-12 (the reference's own mapping-vs-brute-force bar,
test_displacement.py:88-92).
"""

import os

import numpy as np
import pytest

import fixture_maps as fm
from oracle import det_oracle as O


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def test_stage_labels_counts(golden_dir):
    z = _load(golden_dir, "stage_k6.npz")
    m = fm.unpack_map(z)
    f = O.FlatMap.from_mapmodel(m)
    lab = f.labels(6)
    assert np.array_equal(lab, z["labels"])
    assert np.array_equal(O.label_counts(lab, len(f.stats)), z["counts"])


def test_stage_channels_and_field(golden_dir):
    z = _load(golden_dir, "stage_k6.npz")
    ch = O.all_channels(z["d"])
    got = np.stack(ch[:8])
    assert np.array_equal(got, z["channels"])  # bit-identical restatement
    assert ch[8] == float(z["total"])
    u = O.displacement(z["d"])
    np.testing.assert_allclose(u, z["u"], atol=1e-15)
    np.testing.assert_array_equal(O.base_target(64), z["base"])
    m = fm.unpack_map(z)
    moved, cl = O.move_vertices(m.vertex_array(), u)
    np.testing.assert_allclose(moved, z["moved"], atol=1e-15)
    assert cl == int(z["clamps"])


@pytest.mark.parametrize("case", ["overlap", "tie", "vor"])
@pytest.mark.parametrize("q", [0, 1, 2])
def test_raster_cases(golden_dir, case, q):
    z = _load(golden_dir, "raster_cases.npz")
    m = fm.unpack_map(z, prefix=f"{case}{q}_")
    f = O.FlatMap.from_mapmodel(m)
    lab = f.labels(int(z[f"{case}{q}_k"]))
    assert np.array_equal(lab, z[f"{case}{q}_labels"])


@pytest.mark.parametrize("name", ["c1", "two", "two_rederive", "vor_stag", "overlap"])
def test_engine_runs(golden_dir, name):
    z = _load(golden_dir, "engine_runs.npz")
    m = fm.unpack_map(z, prefix=f"{name}_in_")
    k = int(z[f"{name}_k"])
    kw = {}
    crit = dict(error_threshold=1e-300, stagnation_window=10**9, max_iterations=int(z[f"{name}_trace"][-1, 0]))
    if name == "c1":
        kw = dict(bdv_multiplier=0.5)
    elif name == "two_rederive":
        kw = dict(bdv_mode="rederive")
    elif name == "overlap":
        kw = dict(bdv_multiplier=1.3)
    elif name == "vor_stag":
        crit = dict(error_threshold=1e-9, stagnation_window=5, max_iterations=200)
    eng = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=k, **kw)
    res = eng.run(**crit)
    assert res.stop_reason == str(z[f"{name}_stop"])
    assert res.iteration == int(z[f"{name}_iteration"])
    assert np.array_equal(res.rows, z[f"{name}_final_xy"])  # bit-identical trajectory
    assert np.array_equal(res.labels, z[f"{name}_labels"])
    assert np.array_equal(res.counts, z[f"{name}_counts"])
    assert res.clamp_events == int(z[f"{name}_clamps"])
    tr = np.array([t[:3] for t in res.trace])
    np.testing.assert_array_equal(tr, z[f"{name}_trace"])
    np.testing.assert_array_equal(res.weights_px, z[f"{name}_weights_px"])


def test_collapse(golden_dir):
    z = _load(golden_dir, "collapse.npz")
    eng = O.OracleEngine(O.FlatMap.from_mapmodel(fm.sliver()), k=5)
    with pytest.raises(O.OracleCollapseError) as err:
        eng.run(error_threshold=1e-6, stagnation_window=32, max_iterations=400)
    assert err.value.region_id == str(z["region"])
    assert err.value.iteration == int(z["iteration"])
    assert str(err.value) == str(z["message"])


def test_temporal(golden_dir):
    z = _load(golden_dir, "temporal.npz")
    m = fm.unpack_map(z)
    f = O.FlatMap.from_mapmodel(m)
    crit = dict(error_threshold=1e-300, stagnation_window=10**9, max_iterations=8)
    for strat in ("direct", "cumulative"):
        out = O.run_frames(f, z["walk"], 6, cumulative=(strat == "cumulative"), **crit)
        for t, res in enumerate(out):
            assert np.array_equal(res.rows, z[f"{strat}_{t}_xy"])
            assert np.array_equal(res.counts, z[f"{strat}_{t}_counts"])
            assert res.background_mass == float(z[f"{strat}_{t}_mb"])


@pytest.mark.parametrize("name", ["overlap", "c1"])
def test_geojson_output_matches_reference_bytes(golden_dir, name):
    from paper_2604_13880_b200.geomodel import to_geojson

    z = _load(golden_dir, "geojson.npz")
    m = fm.unpack_map(z, prefix=f"{name}_")
    if name == "c1":
        m = m.with_vertex_array(z["c1_final_xy"])
    got = to_geojson(m, extra_properties={m.regions[0].region_id: {"x": 1}})
    assert got == z[name].tobytes()
