"""Pin the metrics oracle against reference-generated fixtures (no GPU).

tests/golden/make_golden.py sections 7-8 hold the reference's own full_report /
shape_distortion / detect_adjacencies / relative_position_error outputs on
map/cartogram pairs; the oracle (oracle/metrics_oracle.py) must reproduce them
bit for bit.
"""

import json
import os

import numpy as np
import pytest

import fixture_maps as fm
from oracle import metrics_oracle as MO

CASES = ["c1", "c1_k6_raw", "overlap", "vor_k8", "two"]


@pytest.fixture(scope="module")
def met(golden_dir):
    return np.load(os.path.join(golden_dir, "metrics.npz"))


def region_rings(z, prefix, xy=None):
    m = fm.unpack_map(z, prefix=prefix)
    if xy is not None:
        m = m.with_vertex_array(xy)
    return [[np.asarray(r, dtype=float) for r in reg.rings] for reg in m.regions]


@pytest.mark.parametrize("case", CASES)
def test_oracle_hamming_areas_centroids(met, case):
    rm = region_rings(met, f"{case}_m_")
    rc = region_rings(met, f"{case}_m_", met[f"{case}_c_xy"])
    k = int(met[f"{case}_k"])
    resc = bool(met[f"{case}_rescale"])
    got = np.array([MO.hamming(a, b, k, resc) for a, b in zip(rm, rc)])
    np.testing.assert_array_equal(got, met[f"{case}_hamming"])
    np.testing.assert_array_equal(np.array([MO.region_area(r) for r in rc]), met[f"{case}_areas"])
    np.testing.assert_array_equal(np.array([MO.region_centroid(r) for r in rm]), met[f"{case}_cent_m"])
    np.testing.assert_array_equal(np.array([MO.region_centroid(r) for r in rc]), met[f"{case}_cent_c"])


@pytest.mark.parametrize("case", CASES)
def test_oracle_adjacency_and_position(met, case):
    rm = region_rings(met, f"{case}_m_")
    rc = region_rings(met, f"{case}_m_", met[f"{case}_c_xy"])
    eps = 0.5 / 1024
    assert MO.adjacency(rm, eps) == set(map(tuple, met[f"{case}_adj_m"].tolist()))
    assert MO.adjacency(rc, eps) == set(map(tuple, met[f"{case}_adj_c"].tolist()))
    cm_ = [MO.region_centroid(r) for r in rm]
    cc_ = [MO.region_centroid(r) for r in rc]
    assert MO.position_error(cm_, cc_) == float(met[f"{case}_poserr"])


def test_oracle_square_disk_and_errors(met):
    a, b = [met["sqdisk_a"]], [met["sqdisk_b"]]
    assert MO.hamming(a, b, 6) == float(met["sqdisk_hamming"])
    assert MO.hamming(a, b, 6, rescale=False) == float(met["sqdisk_hamming_raw"])
    with pytest.raises(MO.OracleNumericError) as err:
        MO.hamming([a[0][::-1]], b, 6)
    assert str(err.value) == str(met["neg_area_message"])


def test_report_fixture_consistency(met):
    """The stored report aggregates are the mean/max of the stored per-region values."""
    for case in CASES:
        rep = json.loads(str(met[f"{case}_json"]))
        h = met[f"{case}_hamming"]
        assert rep["hamming_avg"] == float(h.mean())
        assert rep["hamming_max"] == float(h.max())
        assert rep["position_error"] == float(met[f"{case}_poserr"])
