"""CPU-only tests: C-ABI exports, host-side logic, input generators, API validation."""

import os
import re

import numpy as np
import pytest

import fixture_maps as fm
from oracle import det_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2604_13880_b200 import _lib

    lib = _lib.load_library()
    header = open(os.path.join(ROOT, "include", "det_api.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?(det_\w+)\s*\(", header, re.M))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == declared
    assert lib.det_abi_version() == 1


def test_context_fails_loudly_without_gpu():
    from conftest import cuda_available
    from paper_2604_13880_b200 import _lib

    if cuda_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.DetError):
        _lib.Context(8)


def test_vertex_array_roundtrip_and_rebuild():
    from paper_2604_13880_b200.geomodel import rebuild, ring_layout

    m = fm.overlap_holes_multi()
    xy, rs, rr, ids, stats = ring_layout(m)
    assert xy.shape[0] == rs[-1] and len(rr) == len(rs) - 1
    assert ids == [r.region_id for r in m.regions]
    m2 = rebuild(m, xy * 0.5)
    np.testing.assert_array_equal(m2.vertex_array(), xy * 0.5)
    with pytest.raises(ValueError):
        rebuild(m, xy[:-1])


def test_densify_matches_oracle():
    from paper_2604_13880_b200.geomodel import densify

    m = fm.two_region()
    d = densify(m, 4.0 / 64)
    f = O.FlatMap.from_mapmodel(m).densified(4.0 / 64)
    np.testing.assert_array_equal(d.vertex_array(), f.rows())


def test_region_ranks_string_order():
    from paper_2604_13880_b200._context import region_ranks

    ids = ["R10", "R2", "R1", "R3"]
    rk = region_ranks(ids)
    assert [ids[i] for i in np.argsort(rk)] == sorted(ids)


def test_synthetic_voronoi_properties():
    from paper_2604_13880_b200.synthetic import unique_vertex_count, voronoi_map

    a = voronoi_map(64, seed=0, target_unique=2000)
    b = voronoi_map(64, seed=0, target_unique=2000)
    np.testing.assert_array_equal(a.vertex_array(), b.vertex_array())
    nu = unique_vertex_count(a)
    assert abs(nu - 2000) <= 40
    assert a.vertex_array().shape[0] > 1.5 * nu  # shared chains stored once per ring
    assert all(r.area() > 0 for r in a.regions)
    xy = a.vertex_array()
    assert xy.min() >= 0.1 and xy.max() <= 0.9
    total = sum(r.area() for r in a.regions)
    assert total == pytest.approx(0.64, rel=1e-9)  # exact tiling of the central box


def test_api_validation_without_gpu():
    import paper_2604_13880_b200 as P

    with pytest.raises(ValueError):
        P.StoppingCriteria(error_threshold=0.0)
    with pytest.raises(ValueError):
        P.StoppingCriteria(stagnation_window=0)
    with pytest.raises(ValueError):
        P.CartogramEngine(fm.two_region(), bdv_mode="bogus")
    with pytest.raises(ValueError):
        P.CartogramEngine(fm.two_region(), bdv_multiplier=0.0)
    with pytest.raises(ValueError):
        P.BatchEngine(fm.two_region(), np.ones((1, 2)), k=3)
    with pytest.raises(P.IngestionError):
        P.TimeSeriesDataset(fm.two_region(), ("a",), np.ones((2, 2)))


def test_background_mass_schedule_matches_oracle():
    import paper_2604_13880_b200 as P

    m = fm.small_voronoi(seed=1, r=10, target=200)
    stats = np.abs(np.random.default_rng(0).normal(5, 2, (6, 10))) + 0.1
    ds = P.TimeSeriesDataset(m, tuple(f"t{i}" for i in range(6)), stats)
    pol = P.AreaFractionPolicy(0.3, 0.7, window=(1, 4))
    mb, af = P.background_mass_schedule(ds, pol)
    mb2, af2 = O.area_fraction_schedule(ds.totals(), 0.3, 0.7, (1, 4))
    np.testing.assert_array_equal(mb, mb2)
    np.testing.assert_array_equal(af, af2)


@pytest.mark.gpu
def test_interpolate_vertices():
    import paper_2604_13880_b200 as P
    from conftest import cuda_available

    if not cuda_available():
        pytest.skip("needs a CUDA device")

    a = fm.two_region((1.0, 3.0))
    b = a.with_vertex_array(a.vertex_array() * 0.9).with_statistics([2.0, 2.0])
    mid = P.interpolate_vertices(a, b, 0.5)
    va, vb = a.vertex_array(), b.vertex_array()
    np.testing.assert_array_equal(mid.vertex_array(), va + 0.5 * (vb - va))  # bit-exact, reference op order
    np.testing.assert_array_equal(mid.statistics(), np.array([1.0, 3.0]) + 0.5 * (np.array([2.0, 2.0]) - [1.0, 3.0]))


def test_shard_bounds_cover():
    from paper_2604_13880_b200.shard import shard_bounds

    for n in (1, 7, 64):
        for w in (1, 2, 3, 8):
            cov = [shard_bounds(n, r, w) for r in range(w)]
            assert cov[0][0] == 0 and cov[-1][1] == n
            assert all(cov[i][1] == cov[i + 1][0] for i in range(w - 1))


def test_region_centroid_matches_reference(golden_dir):
    import numpy as np
    import fixture_maps as fm

    z = np.load(os.path.join(golden_dir, "api.npz"))
    m = fm.overlap_holes_multi()
    assert np.array_equal(np.array([r.centroid() for r in m.regions]), z["centroids_overlap"])
    v = fm.small_voronoi(seed=0, r=24, target=600, shuffle_ids=True)
    assert np.array_equal(np.array([r.centroid() for r in v.regions]), z["centroids_vor"])


def test_raster_debug_dumps(tmp_path):
    import numpy as np
    from paper_2604_13880_b200.raster import write_pgm16, write_raw_f32, write_raw_f64

    a = np.arange(12, dtype=float).reshape(3, 4)
    write_pgm16(tmp_path / "a.pgm", a)
    data = (tmp_path / "a.pgm").read_bytes()
    assert data.startswith(b"P5\n4 3\n65535\n") and len(data) == len(b"P5\n4 3\n65535\n") + 24
    assert np.frombuffer(data[-24:], dtype=">u2")[-1] == 65535
    write_raw_f32(tmp_path / "a.f32", a)
    write_raw_f64(tmp_path / "a.f64", a)
    assert np.array_equal(np.fromfile(tmp_path / "a.f32", dtype="<f4"), a.ravel().astype(np.float32))
    assert np.array_equal(np.fromfile(tmp_path / "a.f64", dtype="<f8"), a.ravel())


def test_trace_view_is_a_lazy_tuple_of_records():
    """RunResult.trace builds its IterationRecord objects on first access (engine.py:38-43 records,
    :189-195 bookkeeping): same length, items, equality and pickle as the plain tuple."""
    import pickle

    from paper_2604_13880_b200.engine import TraceView, trace_records

    tr = np.random.default_rng(0).random((7, 4))
    tr[:, 0] = np.arange(7)
    ref = trace_records(tr, 5)
    v = TraceView(tr.copy(), 5)
    assert len(v) == 7 and v._recs is None            # the length needs no records
    assert v[0] == ref[0] and v[-1].iteration == 11
    assert v == ref and list(v) == list(ref) and v == TraceView(tr.copy(), 5)
    w = pickle.loads(pickle.dumps(v))
    assert isinstance(w, tuple) and w == ref
    assert [t.xi for t in v] == [t.xi for t in ref]
