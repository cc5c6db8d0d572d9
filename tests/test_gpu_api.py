"""Stage API members on reference-typed inputs, against fixtures made by the real reference
(tests/golden/make_golden_api.py): mapping_grid / mapping_point / residual_field(ii, base) of a
channel set (including a hand-built IntegralImageSet with no texture behind it), and the
float32-field step == run identity."""

import os

import numpy as np
import pytest

import fixture_maps as fm
from conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def P():
    import paper_2604_13880_b200 as P

    return P


@pytest.fixture(scope="module")
def api(golden_dir):
    return np.load(os.path.join(golden_dir, "api.npz"))


@pytest.fixture(scope="module")
def stage(golden_dir):
    return np.load(os.path.join(golden_dir, "stage_k6.npz"))


def _ii(P, ch, total, source=None):
    return P.IntegralImageSet(*[np.asarray(ch[i]) for i in range(8)], total=float(total), source=source)


def test_mapping_grid_of_channels_bit_exact(P, api, stage):
    # k_map_grid follows displacement.py:102-131's float64 op order: bit-identical
    g = P.mapping_grid(_ii(P, stage["channels"], stage["total"]))
    assert np.array_equal(g, api["mapping_grid"])


def test_mapping_grid_hand_built_set(P, api):
    g = P.mapping_grid(_ii(P, api["h_channels"], api["h_total"]))
    assert np.array_equal(g, api["h_grid"])


def test_mapping_point_bit_exact(P, api, stage):
    ii = _ii(P, stage["channels"], stage["total"])
    got = np.array([P.mapping_point(float(x), float(y), ii) for x, y in api["pts"]])
    np.testing.assert_allclose(got, api["mapping_point"], rtol=0, atol=1e-15)
    hii = _ii(P, api["h_channels"], api["h_total"])
    got = np.array([P.mapping_point(float(x), float(y), hii) for x, y in api["h_pts"]])
    np.testing.assert_allclose(got, api["h_mapping_point"], rtol=0, atol=1e-15)


def test_residual_field_honours_base(P, api, stage):
    ii = _ii(P, stage["channels"], stage["total"])
    fld = P.residual_field(ii, api["base2"])
    assert np.array_equal(fld.u, api["u_base2"])
    assert fld.base is not None and np.array_equal(fld.base, api["base2"])


def test_residual_field_without_source(P, api, stage):
    # no texture behind the set: the reference's t(d) - base_mapping(n) from the channels
    fld = P.residual_field(_ii(P, stage["channels"], stage["total"]))
    np.testing.assert_allclose(fld.u, api["u_none"], rtol=0, atol=1e-13)


def test_residual_field_fused_path_matches(P, api, stage):
    # set built from the texture: band kernels in residual-density form (no t(d) - t(1) cancellation)
    ii = P.integral_images(stage["d"])
    fld = P.residual_field(ii)
    np.testing.assert_allclose(fld.u, api["u_none"], rtol=0, atol=1e-12)


def test_mapping_rejects_zero_total(P, api):
    ii = _ii(P, np.zeros((8, 16, 16)), 0.0)
    with pytest.raises(P.NumericError):
        P.mapping_grid(ii)
    with pytest.raises(P.NumericError):
        P.mapping_point(0.5, 0.5, ii)


def test_residual_field_base_size_mismatch(P, stage):
    with pytest.raises(ValueError):
        P.residual_field(_ii(P, stage["channels"], stage["total"]), np.zeros((32, 32, 2)))


@pytest.mark.parametrize("field", ["float64", "mixed", "float32"])
def test_step_equals_run(P, field):
    # CartogramEngine.step from the returned state reproduces run() iteration by iteration in every
    # precision mode (the float32 state is exactly representable after the first step)
    m = fm.config1()
    crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=6)
    eng = P.CartogramEngine(m, criteria=crit, k=8, bdv_multiplier=0.5, field_dtype=field)
    full = eng.run()
    st = eng.evaluate(eng.initial_map, 0)
    for _ in range(6):
        st = eng.step(st)
    assert st.iteration == full.state.iteration
    assert np.array_equal(st.pixel_counts, full.state.pixel_counts)
    assert np.array_equal(st.mapmodel.vertex_array(), full.state.mapmodel.vertex_array())


# ---------------------------------------------------------------- crossings per scanline
@pytest.mark.parametrize("maker,k", [("many_holes", 12), ("many_holes", 10), ("needle_rings", 9),
                                     ("needle_rings", 12)])
def test_many_crossings_per_scanline_bit_exact(P, maker, k):
    # > 256 toggles on one scanline of one region (the parity-bitmap window of k_region)
    from oracle import det_oracle as O

    m = getattr(fm, maker)()
    tex = P.rasterize_labels(m, k, check_collapse=False)
    ref = O.FlatMap.from_mapmodel(m).labels(k)
    assert np.array_equal(tex.labels, ref), f"{(tex.labels != ref).sum()} pixels differ"
    assert np.array_equal(tex.pixel_counts(), np.bincount(ref[ref >= 0], minlength=len(m.regions)))


def test_many_holes_engine_vs_oracle(P):
    from oracle import det_oracle as O

    m = fm.many_holes()
    crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=3)
    res = P.CartogramEngine(m, criteria=crit, k=10).run()
    ref = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=10).run(1e-300, 10**9, 3)
    assert np.array_equal(res.state.pixel_counts, ref.counts)
    np.testing.assert_allclose(res.state.mapmodel.vertex_array(), ref.rows, rtol=0, atol=1e-9)


# ---------------------------------------------------------------- multi-GPU drop-in (1 GPU here)
def test_run_direct_sharded_equals_single(P):
    # devices=[0, 0]: two blocks through the per-GPU worker process, gathered in frame order
    from paper_2604_13880_b200.shard import shutdown_workers

    m = fm.small_voronoi(seed=5, r=16, target=400, shuffle_ids=True)
    walk = np.stack([m.statistics() * np.exp(0.1 * t * np.sin(np.arange(16))) for t in range(5)])
    ds = P.TimeSeriesDataset(m, tuple(f"t{t}" for t in range(5)), walk)
    crit = P.StoppingCriteria(1e-300, 10**9, 6)
    one = P.run_direct(ds, crit, k=7)
    try:
        two = P.run_direct(ds, crit, k=7, devices=[0, 0])
        csv1, res1 = P.sweep_bdv(m, [0.5, 0.8, 1.1, 1.4, 1.7], crit, k=7)
        csv2, res2 = P.sweep_bdv(m, [0.5, 0.8, 1.1, 1.4, 1.7], crit, k=7, devices=[0, 0])
        be = P.BatchEngine(m, walk, criteria=crit, k=7, devices=[0, 0])
        bres = be.run_all()
    finally:
        shutdown_workers()
    assert len(two.frames) == len(one.frames) == 5
    for a, b in zip(one.frames, two.frames):
        assert a.time_index == b.time_index and a.error == b.error
        assert np.array_equal(a.mapmodel.vertex_array(), b.mapmodel.vertex_array())
        assert np.array_equal(a.result.state.pixel_counts, b.result.state.pixel_counts)
        assert a.report.hamming_avg == b.report.hamming_avg
    strip = lambda c: [",".join(r.split(",")[:-2]) for r in c.splitlines()]  # drop wall_ms, error
    assert strip(csv1) == strip(csv2)
    for a, b, r in zip(one.frames, bres, range(5)):
        assert np.array_equal(a.mapmodel.vertex_array(), b.state.mapmodel.vertex_array())
        assert np.array_equal(b.state.labels.labels, a.result.state.labels.labels)  # re-rasterised after pickling


@pytest.mark.parametrize("field", ["float64", "float32"])
def test_run_is_deterministic_and_prefix_stable(P, field):
    # the same run twice is bit-identical, and a shorter run's trace is a prefix of a longer one's
    m = fm.config1()
    runs = []
    for T in (5, 9, 9):
        crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=T)
        runs.append(P.CartogramEngine(m, criteria=crit, k=8, bdv_multiplier=0.5, field_dtype=field).run())
    a, b, c = runs
    assert [t.xi for t in b.trace] == [t.xi for t in c.trace]
    assert np.array_equal(b.state.mapmodel.vertex_array(), c.state.mapmodel.vertex_array())
    assert [t.xi for t in a.trace] == [t.xi for t in b.trace][:6]


def test_bitmap_raster_engine_deterministic(P):
    # the parity-bitmap k_region instantiation (switched to on toggle overflow) is deterministic
    m = fm.many_holes()
    crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=4)
    r1 = P.CartogramEngine(m, criteria=crit, k=10).run()
    r2 = P.CartogramEngine(m, criteria=crit, k=10).run()
    assert np.array_equal(r1.state.mapmodel.vertex_array(), r2.state.mapmodel.vertex_array())
    assert np.array_equal(r1.state.pixel_counts, r2.state.pixel_counts)


# ---------------------------------------------------------------- float64 advect variants
_ADV_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import voronoi_map
m = voronoi_map(200, seed=7, target_unique=20000, sigma=0.8)
res = P.run(m, P.StoppingCriteria(1e-300, 10**9, 25), k=10)
np.save({out!r}, np.concatenate([res.state.mapmodel.vertex_array().ravel(),
                                 res.state.pixel_counts.astype(np.float64), [res.state.clamp_events]]))
"""


def test_unique_vertex_advect_equals_per_row(tmp_path):
    # k_advect_uniq64 + raster-only k_region (default) vs the fused per-row advect (DET_UNIQ_ADVECT=0):
    # the same float64 arithmetic per vertex, so the trajectories are bit-identical
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for i, e in enumerate([{}, {"DET_UNIQ_ADVECT": "0"}]):
        out = str(tmp_path / f"a{i}.npy")
        r = subprocess.run([sys.executable, "-c", _ADV_SCRIPT.format(root=root, out=out)],
                           env=dict(os.environ, **e), capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])


def test_start_rows_breaking_shared_vertices(P):
    # caller-given start rows where one copy of a shared vertex differs from the other: the batch
    # falls back to the per-row advect, and the run still equals the oracle's
    from oracle import det_oracle as O

    m = fm.small_voronoi(seed=11, r=16, target=500, shuffle_ids=False)
    xy = m.vertex_array().copy()
    rounded = np.round(xy, 12)
    _, first, counts = np.unique(rounded.view(np.complex128).ravel(), return_index=True, return_counts=True)
    dup = first[np.argmax(counts >= 2)]  # a row whose vertex is shared
    xy[dup] += 1e-4
    crit = P.StoppingCriteria(1e-300, 10**9, 5)
    be = P.BatchEngine(m, m.statistics()[None], criteria=crit, k=7, start_vertices=xy[None], apply_densify=False)
    res = be.run_all()[0]
    ref = O.OracleEngine(O.FlatMap.from_mapmodel(m.with_vertex_array(xy)), k=7, apply_densify=False).run(1e-300, 10**9, 5)
    assert np.array_equal(res.state.pixel_counts, ref.counts)
    np.testing.assert_allclose(res.state.mapmodel.vertex_array(), ref.rows, rtol=0, atol=1e-9)
