"""Oracle vs the real reference, live (build container only; skipped where /root/reference is absent)."""

import numpy as np
import pytest

import fixture_maps as fm
from oracle import det_oracle as O

pytestmark = pytest.mark.live_reference


@pytest.fixture(scope="module")
def cm():
    from refshim import import_reference

    return import_reference()


@pytest.mark.parametrize("seed", [11, 12])
def test_oracle_engine_equals_reference(cm, seed):
    from refshim import to_reference_map

    m = fm.small_voronoi(seed=seed, r=30, target=700)
    crit = cm.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=6)
    ref = cm.CartogramEngine(to_reference_map(cm, m), criteria=crit, k=7, bdv_multiplier=0.7).run()
    got = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=7, bdv_multiplier=0.7).run(1e-300, 10**9, 6)
    assert np.array_equal(got.rows, ref.state.mapmodel.vertex_array())
    assert np.array_equal(got.labels, ref.state.labels.labels)


def test_oracle_channels_equal_reference(cm):
    from cartomorph import integral

    d = np.random.default_rng(3).uniform(0, 2, (40, 40))
    ref = integral.integral_images(d)
    got = O.all_channels(d)
    for a, b in zip(got[:8], ref.straight_channels() + ref.tilted_channels()):
        assert np.array_equal(a, b)


def _random_map(rng, n_regions):
    """Random (possibly self-intersecting, overlapping) rings with shuffled ids and a hole or two."""
    from paper_2604_13880_b200.geomodel import MapModel, Region

    regs = []
    ids = rng.permutation(n_regions)
    for i in range(n_regions):
        cx, cy = rng.uniform(0.15, 0.85, 2)
        v = int(rng.integers(3, 12))
        ang = np.sort(rng.uniform(0, 2 * np.pi, v)) if rng.random() < 0.7 else rng.uniform(0, 2 * np.pi, v)
        rad = rng.uniform(0.03, 0.25, v)
        ring = np.clip(np.stack([cx + rad * np.cos(ang), cy + rad * np.sin(ang)], 1), 0, 1)
        rings = [ring]
        if rng.random() < 0.2:  # a hole (reversed inner ring)
            rings.append((ring - [cx, cy]) * 0.3 + [cx, cy])
            rings[-1] = rings[-1][::-1].copy()
        regs.append(Region(f"R{ids[i]}", f"R{ids[i]}", tuple(rings), float(rng.uniform(0.5, 2))))
    return MapModel(regions=tuple(regs))


def test_oracle_raster_equals_reference_random(cm):
    """Random overlapping / self-intersecting maps, k 4..8: oracle labels == rasterize_labels."""
    from cartomorph import raster
    from refshim import to_reference_map

    rng = np.random.default_rng(2024)
    for _ in range(60):
        m = _random_map(rng, int(rng.integers(1, 9)))
        k = int(rng.integers(4, 9))
        try:
            ref = raster.rasterize_labels(to_reference_map(cm, m), k, check_collapse=False).labels
        except ValueError:  # negative bincount index: the oracle must raise as well
            with pytest.raises(ValueError):
                O.FlatMap.from_mapmodel(m).labels(k)
            continue
        assert np.array_equal(O.FlatMap.from_mapmodel(m).labels(k), ref)


def test_oracle_hamming_equals_reference_random(cm):
    from cartomorph import metrics as cmet

    from oracle import metrics_oracle as MO

    rng = np.random.default_rng(77)
    for _ in range(25):
        m = _random_map(rng, 2)
        a = [np.asarray(r) for r in m.regions[0].rings]
        b = [np.asarray(r) for r in m.regions[1].rings]
        k, resc = int(rng.integers(4, 8)), bool(rng.integers(2))
        try:
            want = cmet.hamming_distance(a, b, raster_k=k, rescale=resc)
        except Exception as exc:  # noqa: BLE001 -- the oracle raises the same kind of error
            with pytest.raises(Exception) as err:
                MO.hamming(a, b, k, resc)
            assert str(err.value) == str(exc)
            continue
        assert MO.hamming(a, b, k, resc) == want


def test_oracle_engine_equals_reference_random_criteria(cm):
    """Random criteria / bdv modes on small Voronoi maps: stop reason, iteration, vertices identical."""
    from refshim import to_reference_map

    rng = np.random.default_rng(5)
    for _ in range(6):
        m = fm.small_voronoi(seed=int(rng.integers(1 << 20)), r=int(rng.integers(3, 12)), target=300)
        m = m.with_statistics(np.exp(rng.normal(0, 1.0, len(m.regions))))
        mode = str(rng.choice(["fixed-mass", "rederive"]))
        thr, win, its = float(rng.choice([0.05, 0.2])), int(rng.choice([3, 10**9])), int(rng.integers(5, 20))
        crit = cm.StoppingCriteria(error_threshold=thr, stagnation_window=win, max_iterations=its)
        try:
            ref = cm.CartogramEngine(to_reference_map(cm, m), criteria=crit, k=6, bdv_mode=mode).run()
        except cm.RegionCollapsedError as exc:
            with pytest.raises(O.OracleCollapseError) as err:
                O.OracleEngine(O.FlatMap.from_mapmodel(m), k=6, bdv_mode=mode).run(thr, win, its)
            assert str(err.value) == str(exc)
            continue
        got = O.OracleEngine(O.FlatMap.from_mapmodel(m), k=6, bdv_mode=mode).run(thr, win, its)
        assert got.stop_reason == ref.stop_reason and got.iteration == ref.state.iteration
        assert np.array_equal(got.rows, ref.state.mapmodel.vertex_array())
