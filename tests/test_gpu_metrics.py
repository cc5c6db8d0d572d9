"""GPU parity of the frame quality metrics (k_shape, k_adj_*, k_poserr) -- SURVEY.md §8f #2.

Against the reference's own outputs (tests/golden/metrics.npz, temporal_reports.npz) and against
the pinned oracle (oracle/metrics_oracle.py) on seeded random map pairs.  Bars: Hamming values,
areas, barycenters, epsilon/xi/tau and adjacency sets bit-exact; the position error, whose device
reduction order differs from the reference's sequential loop, within 1e-12 relative.
"""

import json
import os

import numpy as np
import pytest

import fixture_maps as fm

pytestmark = pytest.mark.gpu

CASES = ["c1", "c1_k6_raw", "overlap", "vor_k8", "two"]


@pytest.fixture(scope="module")
def met(golden_dir):
    return np.load(os.path.join(golden_dir, "metrics.npz"))


def pair(z, case):
    m = fm.unpack_map(z, prefix=f"{case}_m_")
    return m, m.with_vertex_array(z[f"{case}_c_xy"])


@pytest.mark.parametrize("case", CASES)
def test_shape_distortion_matches_reference(met, case):
    from paper_2604_13880_b200 import shape_distortion

    m, c = pair(met, case)
    vals, avg, mx = shape_distortion(m, c, raster_k=int(met[f"{case}_k"]), rescale=bool(met[f"{case}_rescale"]))
    np.testing.assert_array_equal(vals, met[f"{case}_hamming"])
    assert avg == float(met[f"{case}_hamming"].mean()) and mx == float(met[f"{case}_hamming"].max())


@pytest.mark.parametrize("case", CASES)
def test_full_report_matches_reference(met, case):
    from paper_2604_13880_b200 import full_report

    m, c = pair(met, case)
    rep = full_report(m, c, raster_k=int(met[f"{case}_k"]), rescale_shapes=bool(met[f"{case}_rescale"]))
    ref = json.loads(str(met[f"{case}_json"]))
    got = json.loads(rep.to_json())
    for key in ("epsilon", "xi", "tau", "hamming_avg", "hamming_max", "per_region", "wall_ms"):
        assert got[key] == ref[key], key
    assert got["position_error"] == pytest.approx(ref["position_error"], rel=1e-12, abs=1e-15)
    # CSV: region lines byte-identical; the aggregate line up to the position error's last digits
    gl, rl = rep.to_csv().splitlines(), str(met[f"{case}_csv"]).splitlines()
    assert gl[:-1] == rl[:-1]
    assert gl[-1].split(";R=")[0] == rl[-1].split(";R=")[0]


@pytest.mark.parametrize("case", CASES)
def test_adjacency_and_position_error(met, case):
    from paper_2604_13880_b200 import detect_adjacencies, relative_position_error

    m, c = pair(met, case)
    ids = m.region_ids()
    for mm, key in ((m, "adj_m"), (c, "adj_c")):
        want = {tuple(sorted((ids[a], ids[b]))) for a, b in met[f"{case}_{key}"].tolist()}
        assert detect_adjacencies(mm, 0.5 / 1024) == want
    assert relative_position_error(m, c) == pytest.approx(float(met[f"{case}_poserr"]), rel=1e-12, abs=1e-15)


def test_hamming_distance_square_disk_and_errors(met):
    from paper_2604_13880_b200 import NumericError, hamming_distance

    a, b = [met["sqdisk_a"]], [met["sqdisk_b"]]
    assert hamming_distance(a, b, raster_k=6) == float(met["sqdisk_hamming"])
    assert hamming_distance(a, b, raster_k=6, rescale=False) == float(met["sqdisk_hamming_raw"])
    with pytest.raises(NumericError, match=str(met["neg_area_message"])):
        hamming_distance([a[0][::-1]], b, raster_k=6)
    # reference test_metrics.py cases: identity and pure translation give 0
    sq = np.array([[0.1, 0.1], [0.4, 0.1], [0.4, 0.4], [0.1, 0.4]])
    assert hamming_distance([sq], [sq], raster_k=6) == 0.0
    assert hamming_distance([sq], [sq + np.array([0.3, 0.4])], raster_k=6) == 0.0


def test_metric_argument_errors():
    from paper_2604_13880_b200 import NumericError, detect_adjacencies, full_report, relative_position_error
    from paper_2604_13880_b200.geomodel import MapModel, Region

    a = fm.two_region()
    b = MapModel(regions=a.regions[:1])
    with pytest.raises(ValueError):
        full_report(a, b)
    with pytest.raises(NumericError):
        relative_position_error(b, b)
    with pytest.raises(ValueError):
        detect_adjacencies(a, 0.0)
    with pytest.raises(NumericError, match="positive actual and desired"):
        full_report(a, a, weights=np.array([1.0, 0.0]))
    corner = MapModel(regions=(Region("A", "A", (np.array([[0.0, 0.0], [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]]),), 1.0),
                               Region("B", "B", (np.array([[0.5, 0.5], [1.0, 0.5], [1.0, 1.0], [0.5, 1.0]]),), 1.0)))
    assert detect_adjacencies(corner, 0.5 / 1024) == frozenset()  # one shared corner is not adjacency


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("k", [4, 7, 8])
def test_random_pairs_match_oracle(seed, k):
    from oracle import metrics_oracle as MO
    from paper_2604_13880_b200 import detect_adjacencies, shape_distortion

    rng = np.random.default_rng(100 + seed)
    m = fm.small_voronoi(seed=20 + seed, r=30, target=700)
    c = m.with_vertex_array(np.clip(m.vertex_array() + rng.normal(0, 0.01, m.vertex_array().shape), 0, 1))
    rm = [[np.asarray(r) for r in reg.rings] for reg in m.regions]
    rc = [[np.asarray(r) for r in reg.rings] for reg in c.regions]
    for resc in (True, False):
        want = np.array([MO.hamming(a, b, k, resc) for a, b in zip(rm, rc)])
        got, _, _ = shape_distortion(m, c, raster_k=k, rescale=resc)
        np.testing.assert_array_equal(got, want)
    pos = {rid: i for i, rid in enumerate(c.region_ids())}
    got_adj = {tuple(sorted((pos[a], pos[b]))) for a, b in detect_adjacencies(c, 0.5 / 1024)}
    assert got_adj == MO.adjacency(rc, 0.5 / 1024)


def test_temporal_reports_and_watchdog(golden_dir):
    from paper_2604_13880_b200 import StoppingCriteria, TimeSeriesDataset, run_cumulative, run_direct

    z = np.load(os.path.join(golden_dir, "temporal_reports.npz"))
    m = fm.unpack_map(z)
    ds = TimeSeriesDataset(m, ("t0", "t1", "t2"), z["walk"])
    crit = StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=8)
    for strat, fn in (("direct", run_direct), ("cumulative", run_cumulative)):
        seq = fn(ds, crit, k=6, bdv_multiplier=1.0, watchdog_ceiling=0.02, report_raster_k=6, field_dtype="float64")
        for t, fr in enumerate(seq.frames):
            ref = json.loads(str(z[f"{strat}_{t}_report"]))
            got = json.loads(fr.report.to_json())
            # the device fp64 field sums in another order than the reference, so frame vertices agree
            # to ~1e-12 (test_gpu_parity.py::test_temporal_vs_golden), not bit for bit: areas and the
            # cartographic errors follow at 1e-9; masks, adjacency and Hamming values stay exact
            for key in ("tau", "hamming_avg", "hamming_max"):
                assert got[key] == ref[key], (strat, t, key)
            for key in ("epsilon", "xi", "position_error"):
                assert got[key] == pytest.approx(ref[key], rel=1e-9, abs=1e-12), (strat, t, key)
            for rid, vals in ref["per_region"].items():
                assert got["per_region"][rid]["shape_distortion"] == vals["shape_distortion"]
                assert got["per_region"][rid]["cartographic_error"] == pytest.approx(vals["cartographic_error"],
                                                                                     rel=1e-9, abs=1e-12)
            assert fr.watchdog == bool(z[f"{strat}_{t}_watchdog"])
        ser = seq.series()
        ref_ser = json.loads(str(z[f"{strat}_series"]))
        for key in ("hamming_avg", "watchdog", "errors", "M_b", "A_i"):
            assert ser[key] == ref_ser[key], key
        np.testing.assert_allclose(ser["epsilon"], ref_ser["epsilon"], rtol=1e-9)


def test_headline_scale_shapes_and_adjacency_match_oracle():
    """3000-region map, ~400k rows: every 97th region's Hamming value (k=7) and the full adjacency
    set of a deformed copy equal the oracle's."""
    from oracle import metrics_oracle as MO
    from paper_2604_13880_b200 import detect_adjacencies, shape_distortion
    from paper_2604_13880_b200.geomodel import densify
    from paper_2604_13880_b200.synthetic import config_map

    m, _ = config_map("headline")
    m = densify(m, 4.0 / 1024)
    rng = np.random.default_rng(77)
    c = m.with_vertex_array(np.clip(m.vertex_array() + rng.normal(0, 3e-4, m.vertex_array().shape), 0, 1))
    vals, _, _ = shape_distortion(m, c, raster_k=7)
    for r in range(0, len(m.regions), 97):
        ra = [np.asarray(x) for x in m.regions[r].rings]
        rc = [np.asarray(x) for x in c.regions[r].rings]
        assert vals[r] == MO.hamming(ra, rc, 7), r
    pos = {rid: i for i, rid in enumerate(c.region_ids())}
    got = {tuple(sorted((pos[a], pos[b]))) for a, b in detect_adjacencies(c, 0.5 / 1024)}
    assert got == MO.adjacency([[np.asarray(x) for x in reg.rings] for reg in c.regions], 0.5 / 1024)


def test_long_rings_shape_distortion_matches_oracle():
    """Rings of ~5000 vertices: the pairwise moment sums walk a deep split tree (regression: a
    recursive version overflowed the per-thread stack)."""
    from oracle import metrics_oracle as MO
    from paper_2604_13880_b200 import shape_distortion
    from paper_2604_13880_b200.geomodel import densify

    m = densify(fm.two_region(), 0.0005)
    assert max(np.asarray(r).shape[0] for reg in m.regions for r in reg.rings) > 4000
    rng = np.random.default_rng(3)
    c = m.with_vertex_array(np.clip(m.vertex_array() + rng.normal(0, 0.002, m.vertex_array().shape), 0, 1))
    got, _, _ = shape_distortion(m, c, raster_k=6)
    want = [MO.hamming([np.asarray(x) for x in a.rings], [np.asarray(x) for x in b.rings], 6)
            for a, b in zip(m.regions, c.regions)]
    np.testing.assert_array_equal(got, want)
