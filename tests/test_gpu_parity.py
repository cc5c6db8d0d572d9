"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the golden fixtures.

Bars (BASELINE.json north_star): region-ID rasters bit-exact on identical vertex
input; vertices within 1e-4 of the domain extent; per-region areas within 1e-3
relative.  Float64-field runs are additionally held to trajectory identity with
the reference where the fixtures allow it.
"""

import os

import numpy as np
import pytest

import fixture_maps as fm
from conftest import cuda_available
from oracle import det_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

VERT_TOL = 1e-4   # north_star: vertex positions within 1e-4 of the domain extent
AREA_RTOL = 1e-3  # north_star: per-region area error within 1e-3 relative


@pytest.fixture(scope="module")
def P():
    import paper_2604_13880_b200 as P

    return P


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


# ---------------------------------------------------------------- raster
@pytest.mark.parametrize("case", ["overlap", "tie", "vor"])
@pytest.mark.parametrize("q", [0, 1, 2])
def test_raster_golden_bit_exact(P, golden_dir, case, q):
    z = _load(golden_dir, "raster_cases.npz")
    m = fm.unpack_map(z, prefix=f"{case}{q}_")
    tex = P.rasterize_labels(m, int(z[f"{case}{q}_k"]), check_collapse=False)
    assert np.array_equal(tex.labels, z[f"{case}{q}_labels"])
    ref = z[f"{case}{q}_labels"]
    assert np.array_equal(tex.pixel_counts(), np.bincount(ref[ref >= 0], minlength=len(m.regions)))
    assert tex.background_count() == int((ref == -1).sum())


@pytest.mark.parametrize("k", [4, 6, 8, 10])
def test_raster_perturbed_vs_oracle(P, k):
    m = fm.config1()
    rng = np.random.default_rng(k)
    base = m.vertex_array()
    for q in range(4):
        xy = base if q == 0 else np.clip(base + rng.normal(0, 0.5 / (1 << k), base.shape), 0, 1)
        mq = m.with_vertex_array(xy)
        tex = P.rasterize_labels(mq, k, check_collapse=False)
        ref = O.FlatMap.from_mapmodel(mq).labels(k)
        assert np.array_equal(tex.labels, ref), f"k={k} q={q}: {(tex.labels != ref).sum()} pixels differ"


def test_raster_tie_and_edge_cases(P):
    tex = P.rasterize_labels(fm.tie_partition(), 4)
    assert tex.background_count() == 0 and tex.pixel_counts().tolist() == [128, 128]
    full = P.MapModel(regions=(P.Region("A", "A", (np.array([[0., 0.], [1., 0.], [1., 1.], [0., 1.]]),), 1.0),))
    assert P.rasterize_labels(full, 4).pixel_counts()[0] == 256
    tiny = P.MapModel(regions=(P.Region("A", "A", (np.array([[.5, .5], [.501, .5], [.501, .501], [.5, .501]]),), 1.),))
    with pytest.raises(P.RasterizationError, match="zero-pixel"):
        P.rasterize_labels(tiny, 4)
    with pytest.raises(ValueError):
        P.rasterize_labels(full, 3)


def test_raster_headline_size_vs_oracle(P):
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(3000, seed=3, target_unique=200_000, sigma=2.0)
    tex = P.rasterize_labels(m, 10, check_collapse=False)
    ref = O.FlatMap.from_mapmodel(m).labels(10)
    assert np.array_equal(tex.labels, ref)
    assert tex.pixel_counts().sum() + tex.background_count() == 1 << 20


# ---------------------------------------------------------------- integral images / field / advect
def test_channels_vs_oracle(P, golden_dir):
    z = _load(golden_dir, "stage_k6.npz")
    ii = P.integral_images(z["d"])
    got = np.stack(ii.straight_channels() + ii.tilted_channels())
    tol = 1e-9 * ii.total
    assert np.abs(got - z["channels"]).max() <= tol
    assert abs(ii.total - float(z["total"])) <= 1e-12 * ii.total


@pytest.mark.parametrize("n", [16, 32, 128, 512])
def test_channels_random_vs_oracle(P, n):
    d = np.random.default_rng(n).uniform(0.0, 3.0, (n, n))
    ii = P.integral_images(d)
    ref = O.all_channels(d)
    for a, b in zip(ii.straight_channels() + ii.tilted_channels(), ref[:8]):
        assert np.abs(a - b).max() <= 1e-9 * ref[8]


def test_field_and_advect_vs_golden(P, golden_dir):
    z = _load(golden_dir, "stage_k6.npz")
    fld = P.residual_field(P.integral_images(z["d"]))
    assert np.abs(fld.u - z["u"]).max() <= 1e-12
    moved, cl = P.advect(fm.unpack_map(z).vertex_array(), P.DisplacementField(64, z["u"]))
    assert np.abs(moved - z["moved"]).max() <= 1e-15
    assert cl == int(z["clamps"])
    assert np.abs(P.base_mapping(64) - z["base"]).max() <= 1e-12


@pytest.mark.parametrize("n", [256, 1024])
def test_field_large_vs_oracle(P, n):
    rng = np.random.default_rng(7)
    d = np.repeat(np.repeat(rng.lognormal(0, 1, (n // 16, n // 16)), 16, 0), 16, 1)
    from paper_2604_13880_b200._context import get_context

    u, _, _ = get_context(n.bit_length() - 1).field(d)
    ref = O.displacement(d)
    assert np.abs(u - ref).max() <= 1e-12


def test_density_vs_oracle(P, golden_dir):
    z = _load(golden_dir, "stage_k6.npz")
    lab = P.LabelTexture(64, z["labels"], tuple(str(i) for i in z["ids"]))
    stats = z["stats"]
    bdv = 0.8 * P.default_bdv(stats, lab)
    dens = P.build_density(stats, lab, bdv)
    assert np.array_equal(dens.d, O.density_texture(stats, z["labels"], bdv))


# ---------------------------------------------------------------- engine runs
_RUNS = ["c1", "two", "two_rederive", "vor_stag", "overlap"]


def _golden_run_args(z, name):
    kw, crit = {}, dict(error_threshold=1e-300, stagnation_window=10**9, max_iterations=int(z[f"{name}_trace"][-1, 0]))
    if name == "c1":
        kw = dict(bdv_multiplier=0.5)
    elif name == "two_rederive":
        kw = dict(bdv_mode="rederive")
    elif name == "overlap":
        kw = dict(bdv_multiplier=1.3)
    elif name == "vor_stag":
        crit = dict(error_threshold=1e-9, stagnation_window=5, max_iterations=200)
    return kw, crit


@pytest.mark.parametrize("field_dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", _RUNS)
def test_engine_vs_golden(P, golden_dir, name, field_dtype):
    z = _load(golden_dir, "engine_runs.npz")
    m = fm.unpack_map(z, prefix=f"{name}_in_")
    kw, crit = _golden_run_args(z, name)
    res = P.run(m, P.StoppingCriteria(**crit), k=int(z[f"{name}_k"]), field_dtype=field_dtype, **kw)
    verts = res.state.mapmodel.vertex_array()
    dv = np.abs(verts - z[f"{name}_final_xy"]).max()
    assert dv <= VERT_TOL, f"max vertex deviation {dv:.3e}"
    np.testing.assert_array_equal(res.weights_px, z[f"{name}_weights_px"])
    assert res.stop_reason == str(z[f"{name}_stop"])
    cnt = res.state.pixel_counts
    ref_cnt = z[f"{name}_counts"]
    assert np.abs(cnt - ref_cnt).max() <= max(2, 1e-3 * ref_cnt.max())
    areas = np.array([r.area() for r in res.state.mapmodel.regions])
    assert np.allclose(areas, z[f"{name}_areas"], rtol=AREA_RTOL)
    if field_dtype == "float64":
        # trajectory identical to the reference: same integer pixel counts every iteration
        assert res.state.iteration == int(z[f"{name}_iteration"])
        assert np.array_equal(cnt, ref_cnt)
        tr = np.array([[t.iteration, t.epsilon, t.xi] for t in res.trace])
        np.testing.assert_allclose(tr, z[f"{name}_trace"], rtol=1e-12, atol=1e-15)
        assert dv <= 1e-9


def test_engine_rasterizes_its_own_state(P):
    """Stage parity every iteration: the engine's labels equal the oracle raster of its own vertices."""
    m = fm.config1()
    for iters in (1, 3, 7):
        res = P.run(m, P.StoppingCriteria(1e-300, 10**9, iters), k=8, bdv_multiplier=0.5)
        ref = O.FlatMap.from_mapmodel(res.state.mapmodel).labels(8)
        assert np.array_equal(res.state.labels.labels, ref)
        assert np.array_equal(res.state.pixel_counts, O.label_counts(ref, len(m.regions)))


def test_collapse_matches_golden(P, golden_dir):
    z = _load(golden_dir, "collapse.npz")
    with pytest.raises(P.RegionCollapsedError) as err:
        P.run(fm.sliver(), P.StoppingCriteria(error_threshold=1e-6, max_iterations=400), k=5, field_dtype="float64")
    assert err.value.region_id == str(z["region"])
    assert err.value.iteration == int(z["iteration"])


def test_determinism_bit_identical(P):
    m = fm.two_region((1.0, 2.0))
    r1 = P.run(m, P.StoppingCriteria(), k=6)
    r2 = P.run(m, P.StoppingCriteria(), k=6)
    assert (r1.state.mapmodel.vertex_array() == r2.state.mapmodel.vertex_array()).all()
    assert [t.xi for t in r1.trace] == [t.xi for t in r2.trace]


def test_analytic_ratio(P):
    res = P.run(fm.two_region((1.0, 3.0)), P.StoppingCriteria(error_threshold=0.004), k=8)
    assert res.stop_reason == "converged"
    c = res.state.pixel_counts
    assert c[1] / c[0] == pytest.approx(3.0, rel=0.01)


def test_batch_equals_single(P):
    m = fm.small_voronoi(seed=2, r=20, target=500)
    stats = np.stack([m.statistics() * np.exp(np.random.default_rng(s).normal(0, 0.5, len(m.regions)))
                      for s in range(4)])
    mult = np.array([0.4, 0.8, 1.0, 1.6])
    crit = P.StoppingCriteria(1e-300, 10**9, 25)
    be = P.BatchEngine(m, stats, criteria=crit, k=7, bdv_multiplier=mult)
    batch = be.run_all()
    for b in range(4):
        single = P.run(m.with_statistics(stats[b]), crit, k=7, bdv_multiplier=float(mult[b]))
        assert np.array_equal(batch[b].state.mapmodel.vertex_array(), single.state.mapmodel.vertex_array())
        assert np.array_equal(batch[b].state.pixel_counts, single.state.pixel_counts)


def test_device_areas_match_shoelace(P):
    m = fm.config1()
    be = P.BatchEngine(m, m.statistics()[None], criteria=P.StoppingCriteria(1e-300, 10**9, 10), k=8)
    res = be.run_all()[0]
    host = np.array([r.area() for r in res.state.mapmodel.regions])
    np.testing.assert_allclose(be.areas(0), host, rtol=1e-9, atol=1e-15)


def test_step_and_evaluate_match_run(P):
    m = fm.two_region((1.0, 3.0))
    eng = P.CartogramEngine(m, P.StoppingCriteria(1e-300, 10**9, 3), k=6, field_dtype="float64")
    st = eng.evaluate(eng.initial_map, 0, labels=eng._labels0)
    for _ in range(3):
        st = eng.step(st)
    res = eng.run()
    assert st.iteration == res.state.iteration == 3
    assert np.abs(st.mapmodel.vertex_array() - res.state.mapmodel.vertex_array()).max() <= 1e-12
    assert np.array_equal(st.pixel_counts, res.state.pixel_counts)


# ---------------------------------------------------------------- temporal
@pytest.mark.parametrize("strategy", ["direct", "cumulative"])
def test_temporal_vs_golden(P, golden_dir, strategy):
    z = _load(golden_dir, "temporal.npz")
    m = fm.unpack_map(z)
    ds = P.TimeSeriesDataset(m, ("t0", "t1", "t2"), z["walk"])
    fn = P.run_direct if strategy == "direct" else P.run_cumulative
    seq = fn(ds, P.StoppingCriteria(1e-300, 10**9, 8), k=6, field_dtype="float64")
    for t, fr in enumerate(seq.frames):
        assert fr.error is None
        assert np.abs(fr.mapmodel.vertex_array() - z[f"{strategy}_{t}_xy"]).max() <= 1e-9
        assert np.array_equal(fr.result.state.pixel_counts, z[f"{strategy}_{t}_counts"])
        assert fr.background_mass == float(z[f"{strategy}_{t}_mb"])


# ---------------------------------------------------------------- full-size properties
def test_headline_size_properties(P):
    """1024^2 / ~200k-vertex map: 20 iterations, size-independent invariants + oracle raster of the result."""
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(3000, seed=3, target_unique=200_000, sigma=2.0, lloyd=1)
    res = P.run(m, P.StoppingCriteria(1e-300, 10**9, 20), k=10)
    c = res.state.pixel_counts
    assert c.sum() + res.state.labels.background_count() == 1 << 20
    assert (c > 0).all()
    eps = [t.epsilon for t in res.trace]
    assert eps[-1] < eps[0]  # equalisation progresses
    ref = O.FlatMap.from_mapmodel(res.state.mapmodel).labels(10)
    assert np.array_equal(res.state.labels.labels, ref)
    v = res.state.mapmodel.vertex_array()
    assert v.min() >= 0.0 and v.max() <= 1.0


# ---------------------------------------------------------------- other texture sizes / scales
@pytest.mark.parametrize("k", [11, 12, 13])
def test_large_textures_raster_and_field_precision(P, k):
    """k = 11..13 (1024-thread band CTAs): raster bit-exact vs the oracle; float32 vs float64 field agree."""
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(40, seed=k, target_unique=4000 * (1 << (k - 11)), sigma=0.5)
    tex = P.rasterize_labels(m, k, check_collapse=False)
    ref = O.FlatMap.from_mapmodel(m).labels(k)
    assert np.array_equal(tex.labels, ref)
    crit = P.StoppingCriteria(1e-300, 10**9, 6)
    r32 = P.run(m, crit, k=k, field_dtype="float32")
    r64 = P.run(m, crit, k=k, field_dtype="float64")
    dv = np.abs(r32.state.mapmodel.vertex_array() - r64.state.mapmodel.vertex_array()).max()
    assert dv <= 1e-5, dv
    assert np.array_equal(r64.state.labels.labels,
                          O.FlatMap.from_mapmodel(r64.state.mapmodel).labels(k))


def test_many_regions_control_step(P):
    """R = 10,000 regions (config-5 scale region count) at 2048^2: counts partition the texture."""
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(10_000, seed=5, target_unique=150_000, sigma=0.5)
    res = P.run(m, P.StoppingCriteria(1e-300, 10**9, 5), k=11)
    c = res.state.pixel_counts
    assert c.sum() + res.state.labels.background_count() == (1 << 11) ** 2
    assert np.array_equal(res.state.labels.labels, O.FlatMap.from_mapmodel(res.state.mapmodel).labels(11))


# ---------------------------------------------------------------- BASELINE configs 2-5 (seeded stand-ins)
def _trajectory_matches(P, m, k, iters, **kw):
    res = P.run(m, P.StoppingCriteria(1e-300, 10**9, iters), k=k, field_dtype="float64", **kw)
    ref = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=k, **kw).run(1e-300, 10**9, iters)
    return res, ref


def test_config2_cumulative_chain_vs_oracle(P):
    """Config 2 map (500 Lloyd-relaxed regions, ~40k vertices, 1024^2), cumulative chain of
    3 frames x 4 iterations: float64 field reproduces the oracle trajectory frame by frame."""
    from paper_2604_13880_b200.synthetic import config_map, random_walk

    m, prm = config_map("c2")
    walk = random_walk(m.statistics(), 3, prm["walk_sigma"], seed=21)
    ds = P.TimeSeriesDataset(m, ("t0", "t1", "t2"), walk)
    crit = dict(error_threshold=1e-300, stagnation_window=10**9, max_iterations=4)
    seq = P.run_cumulative(ds, P.StoppingCriteria(**crit), k=10, field_dtype="float64")
    ref = O.run_frames(O.FlatMap.from_mapmodel(m), walk, 10, cumulative=True, **crit)
    for fr, r in zip(seq.frames, ref):
        assert fr.error is None
        dv = np.abs(fr.mapmodel.vertex_array() - r.rows).max()
        assert dv <= 1e-9, dv
        assert np.array_equal(fr.result.state.pixel_counts, r.counts)


def test_config3_direct_mode_collapse_frames(P):
    """Config 3 (3000 regions, 5% at 1e-3 x median, multiplier 0.3, 2048^2), 4 direct frames:
    frames that collapse report the oracle's region and iteration; others stay in tolerance."""
    from paper_2604_13880_b200.synthetic import config_map, random_walk

    m, prm = config_map("c3")
    walk = random_walk(m.statistics(), 4, prm["walk_sigma"], seed=31)
    ds = P.TimeSeriesDataset(m, tuple(f"t{i}" for i in range(4)), walk)
    seq = P.run_direct(ds, P.StoppingCriteria(1e-300, 10**9, 60), k=11, bdv_multiplier=prm["bdv_multiplier"],
                       field_dtype="float64")
    collapsed = [fr for fr in seq.frames if fr.error is not None]
    assert collapsed, "config 3 is built to make small regions collapse"
    fr = collapsed[0]
    f = O.FlatMap.from_mapmodel(m)
    masses = O.default_background_masses(f, walk.sum(axis=1), 11, prm["bdv_multiplier"])
    eng = O.OracleEngine(f.densified(4.0 / 2048).with_stats(walk[fr.time_index]), k=11,
                         background_mass=float(masses[fr.time_index]), apply_densify=False)
    with pytest.raises(O.OracleCollapseError) as err:
        eng.run(error_threshold=1e-300, stagnation_window=10**9, max_iterations=60)
    assert fr.error == str(err.value)


def test_config4_parameter_sweep_batch(P):
    """Config 4: 8 value seeds x 8 multipliers of the config-2 map as ONE 64-cartogram batch;
    two members checked against the oracle trajectory (float64 field)."""
    from paper_2604_13880_b200.synthetic import batch_statistics, config_map

    m, _ = config_map("c4")
    seeds = batch_statistics(m, 8, 1.5)
    mult = np.repeat(np.arange(1, 9) / 10.0, 8)
    stats = np.tile(seeds, (8, 1))
    be = P.BatchEngine(m, stats, criteria=P.StoppingCriteria(1e-300, 10**9, 3), k=10, bdv_multiplier=mult,
                       field_dtype="float64")
    res = be.run_all()
    assert len(res) == 64
    for b in (5, 62):
        ref = O.OracleEngine(O.FlatMap.from_mapmodel(m.with_statistics(stats[b])), k=10,
                             bdv_multiplier=float(mult[b])).run(1e-300, 10**9, 3)
        assert np.abs(res[b].state.mapmodel.vertex_array() - ref.rows).max() <= 1e-9
        assert np.array_equal(res[b].state.pixel_counts, ref.counts)


def test_config5_stress_scale(P):
    """Config 5 scale: 10,000 regions, ~1M vertices, 4096^2 texture: a few iterations run, the
    state's raster equals the oracle raster of its vertices, and the float32 field stays within
    1e-5 of the float64 build (the 'fp32 integral image checked against an fp64 build' ask)."""
    from paper_2604_13880_b200.synthetic import config_map

    m, _ = config_map("c5")
    crit = P.StoppingCriteria(1e-300, 10**9, 3)
    r32 = P.run(m, crit, k=12, field_dtype="float32")
    r64 = P.run(m, crit, k=12, field_dtype="float64")
    dv = np.abs(r32.state.mapmodel.vertex_array() - r64.state.mapmodel.vertex_array()).max()
    assert dv <= 1e-5, dv
    assert np.array_equal(r64.state.labels.labels, O.FlatMap.from_mapmodel(r64.state.mapmodel).labels(12))


# ---------------------------------------------------------------- float32-path variants
_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import voronoi_map
m = voronoi_map(200, seed=7, target_unique=20000, sigma=0.8)
res = P.run(m, P.StoppingCriteria(1e-300, 10**9, 30), k=10, field_dtype="float32")
np.save({out!r}, np.concatenate([res.state.mapmodel.vertex_array().ravel(),
                                 res.state.pixel_counts.astype(np.float64)]))
"""


@pytest.mark.parametrize("env", [{"DET_SAT1W": "0"}, {"DET_SPLIT_ADVECT": "1"}])
def test_float_path_kernel_variants_agree(P, tmp_path, env):
    """The float32 path's A/B kernel variants (k_sat1 with CTA barriers instead of the barrier-free
    k_sat1w; the advect as its own flat kernel instead of inside k_region) give the same cartogram:
    vertices within float rounding (1e-5), pixel counts within a few pixels."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for i, e in enumerate([{}, env]):
        out = str(tmp_path / f"v{i}.npy")
        code = _VARIANT_SCRIPT.format(root=root, out=out)
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **e), capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    nv = outs[0].size - 200
    dv = np.abs(outs[0][:nv] - outs[1][:nv]).max()
    assert dv <= 1e-5, dv
    assert np.abs(outs[0][nv:] - outs[1][nv:]).max() <= 4


def test_float_state_start_raster_is_exact(P):
    """Float32 vertex state: the start raster (iteration 0's counts and error) is computed on the
    exact float64 rows, identical to the float64 path; later states stay within the tolerances."""
    m = fm.config1()
    crit = P.StoppingCriteria(1e-300, 10**9, 40)
    r32 = P.run(m, crit, k=8, bdv_multiplier=0.5, field_dtype="float32")
    r64 = P.run(m, crit, k=8, bdv_multiplier=0.5, field_dtype="float64")
    assert r32.trace[0].epsilon == r64.trace[0].epsilon and r32.trace[0].xi == r64.trace[0].xi
    np.testing.assert_array_equal(r32.weights_px, r64.weights_px)
    dv = np.abs(r32.state.mapmodel.vertex_array() - r64.state.mapmodel.vertex_array()).max()
    assert dv <= VERT_TOL, dv
    a32 = np.array([r.area() for r in r32.state.mapmodel.regions])
    a64 = np.array([r.area() for r in r64.state.mapmodel.regions])
    assert np.allclose(a32, a64, rtol=AREA_RTOL)
    # the float32 state's own raster is still bit-exact against the oracle on its (float32) rows
    ref = O.FlatMap.from_mapmodel(r32.state.mapmodel).labels(8)
    assert np.array_equal(r32.state.labels.labels, ref)


def test_band_height_independence(P):
    """The band kernels give the same cartogram for any band height (1, 2, 16 or the automatic
    one): k_sat1w's paired row-total butterfly, its odd-height tail and the slice-edge joins."""
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(60, seed=2, target_unique=6000, sigma=0.6)
    crit = P.StoppingCriteria(1e-300, 10**9, 5)
    outs = []
    for h in (0, 1, 2, 16):
        be = P.BatchEngine(m, np.atleast_2d(m.statistics()), criteria=crit, k=8, bdv_multiplier=1.0)
        ctx = be._ctx()
        if h:
            ctx.set_band_height(h)
        outs.append(be.run_all(crit)[0].state.mapmodel.vertex_array())
        ctx.set_band_height(0)  # back to the automatic height for the shared per-thread context
    assert max(np.abs(o - outs[0]).max() for o in outs) <= 1e-5


_VARIANT64_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import voronoi_map
m = voronoi_map(200, seed=7, target_unique=20000, sigma=0.8)
res = P.run(m, P.StoppingCriteria(1e-300, 10**9, 30), k={k}, field_dtype="float64")
np.save({out!r}, np.concatenate([res.state.mapmodel.vertex_array().ravel(),
                                 res.state.pixel_counts.astype(np.float64)]))
"""


@pytest.mark.parametrize("k", [9, 10])
@pytest.mark.parametrize("env", [{"DET_SAT3X": "0"}, {"DET_SAT3W": "0"}])
def test_float64_band_kernel_variants_agree(P, tmp_path, env, k):
    """The float64 field's sweep kernels -- k_sat3x (edge records, rows unrolled four times), k_sat3w
    (running edge sums) and the barrier-per-row k_sat3 -- give the same cartogram after 30
    iterations: vertices within 1e-10 (only the grouping of the edge sums differs), identical counts."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for i, e in enumerate([{}, env]):
        out = str(tmp_path / f"w{i}.npy")
        code = _VARIANT64_SCRIPT.format(root=root, out=out, k=k)
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **e), capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    nv = outs[0].size - 200
    dv = np.abs(outs[0][:nv] - outs[1][:nv]).max()
    assert dv <= 1e-10, dv
    assert np.array_equal(outs[0][nv:], outs[1][nv:])


def test_float64_band_height_independence(P):
    """k_sat3x / k_sat1w(TAB) at 1024^2 for band heights 1, 2 (the unroll's tail rows), 32 and 64 (two
    record chunks per warp): the same cartogram as the automatic height within 1e-10."""
    from paper_2604_13880_b200.synthetic import voronoi_map

    m = voronoi_map(120, seed=5, target_unique=12000, sigma=0.6)
    crit = P.StoppingCriteria(1e-300, 10**9, 6)
    outs = []
    for h in (0, 1, 2, 32, 64):
        be = P.BatchEngine(m, np.atleast_2d(m.statistics()), criteria=crit, k=10, bdv_multiplier=1.0,
                           field_dtype="float64")
        ctx = be._ctx()
        if h:
            ctx.set_band_height(h)
        outs.append(be.run_all(crit)[0].state.mapmodel.vertex_array())
        ctx.set_band_height(0)
    assert max(np.abs(o - outs[0]).max() for o in outs) <= 1e-10


@pytest.mark.parametrize("k", [9, 10])
@pytest.mark.parametrize("env", [{"DET_FUSE_ADVECT": "1"}, {"DET_UQ_STATE": "0"}])
def test_float64_vertex_state_variants_bit_identical(P, tmp_path, env, k):
    """The three float64 advect forms -- per-row state with k_advect_uniq64, the unique-vertex state
    with k_advect_uniq64s (the default), and the experimental band-fused advect inside k_sat3x (+ k_advect_bnd) -- evaluate the
    same expressions on the same field: bit-identical vertices and counts after 30 iterations."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for i, e in enumerate([{}, env]):
        out = str(tmp_path / f"u{i}.npy")
        code = _VARIANT64_SCRIPT.format(root=root, out=out, k=k)
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **e), capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
