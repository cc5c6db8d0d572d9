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
