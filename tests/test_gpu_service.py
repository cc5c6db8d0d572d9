"""Steering-service frame on the GPU (service.py:181-241).

compute_frame (engine + report + GeoJSON) against the reference's own composition of the same
steps (tests/golden/service_frames.npz), and per-session isolation: frames computed on two
threads at once (each thread has its own device context / stream) equal sequential ones.
"""

import json
import os
import threading
from types import SimpleNamespace

import numpy as np
import pytest

import fixture_maps as fm

pytestmark = pytest.mark.gpu


def _params(k, hk):
    return SimpleNamespace(threshold=1e-300, stagnation=10**9, max_iter=12, texture_k=int(k), hamming_k=int(hk))


@pytest.fixture(scope="module")
def sv(golden_dir):
    return np.load(os.path.join(golden_dir, "service_frames.npz"))


@pytest.mark.parametrize("t", [0, 1])
def test_compute_frame_matches_reference(sv, t):
    from paper_2604_13880_b200.service import compute_frame

    m = fm.unpack_map(sv, prefix="m_")
    mass, k, hk = sv[f"f{t}_cfg"]
    fr = compute_frame(m, m, sv[f"f{t}_stats"], float(mass), None, _params(k, hk), field_dtype="float64")
    assert fr.error is None and fr.stop_reason == str(sv[f"f{t}_stop"])
    np.testing.assert_allclose(fr.mapmodel.vertex_array(), sv[f"f{t}_xy"], atol=1e-9)
    ref = json.loads(str(sv[f"f{t}_report"]))
    rep = fr.report
    # vertices agree to ~1e-12 (device fp64 field summation order), masks/adjacency exactly
    for key in ("tau", "hamming_avg", "hamming_max"):
        assert rep[key] == ref[key], key
    for key in ("epsilon", "xi", "position_error"):
        assert rep[key] == pytest.approx(ref[key], rel=1e-9, abs=1e-12), key
    gj_ref = json.loads(str(sv[f"f{t}_geojson"]))
    assert [f["id"] for f in fr.geojson["features"]] == [f["id"] for f in gj_ref["features"]]
    for a, b in zip(fr.geojson["features"], gj_ref["features"]):
        assert a["geometry"]["type"] == b["geometry"]["type"]
        assert set(a["properties"]) == set(b["properties"])
        np.testing.assert_allclose(np.array(a["geometry"]["coordinates"], dtype=object).size,
                                   np.array(b["geometry"]["coordinates"], dtype=object).size)


def test_sessions_on_separate_threads_are_isolated(sv):
    from paper_2604_13880_b200.service import compute_frame

    m = fm.unpack_map(sv, prefix="m_")
    jobs = []
    for t in (0, 1):
        mass, k, hk = sv[f"f{t}_cfg"]
        jobs.append((sv[f"f{t}_stats"], float(mass), _params(k, hk)))
    seq = [compute_frame(m, m, s, mb, None, p) for s, mb, p in jobs]
    out, errs = [None, None], []

    def work(i):
        try:
            s, mb, p = jobs[i]
            for _ in range(3):
                out[i] = compute_frame(m, m, s, mb, None, p)
        except Exception as exc:  # noqa: BLE001 -- re-raised in the main thread
            errs.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for a, b in zip(seq, out):
        assert np.array_equal(a.mapmodel.vertex_array(), b.mapmodel.vertex_array())
        assert a.report["hamming_avg"] == b.report["hamming_avg"] and a.report["epsilon"] == b.report["epsilon"]


def test_compute_frame_error_becomes_frame_error():
    from paper_2604_13880_b200.service import compute_frame

    m = fm.sliver()
    fr = compute_frame(m, m, m.statistics(), 1.0, None,
                       SimpleNamespace(threshold=1e-6, stagnation=32, max_iter=400, texture_k=5, hamming_k=6))
    # the sliver either collapses (engine) or rasterises to nothing in the Hamming grid (report):
    # both are CartomorphErrors, which the service turns into a failed frame (service.py:237-240)
    assert fr.mapmodel is None and fr.report is None and fr.error
