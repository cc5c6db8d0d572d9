"""bench.py's bookkeeping (no GPU): the metric string, the §8(d) byte model, launch counting and the
committed ncu traffic lookup."""

import importlib.util
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_metric_is_baseline_verbatim(bench):
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert bench.METRIC == json.load(f)["metric"]


def test_algorithmic_bytes_match_survey_table(bench):
    # 55.8 MB per iteration at 1024^2 / 200k unique vertices, 601.8 MB at config 5
    assert bench.algorithmic_bytes_per_iteration(1024, 200_000) == pytest.approx(55.8e6, rel=2e-3)
    assert bench.algorithmic_bytes_per_iteration(4096, 1_000_000) == pytest.approx(601.8e6, rel=2e-3)
    ph = bench.phase_bytes(1024, 200_000, 400_000, 3000, "float32")
    assert ph["integral_images"] == 12 * 1024 * 1024 and ph["region"] == 48 * 200_000
    ph = bench.phase_bytes(1024, 200_000, 400_000, 3000, "float64")  # float64 field and state
    assert ph["integral_images"] == 20 * 1024 * 1024 and ph["region"] == 96 * 200_000


def test_traffic_lookup_reads_committed_capture(bench):
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
        per = json.load(f)["per_frame_bytes_by_phase"]
    assert bench.traffic_for("region", 16) == pytest.approx(per["region"] * 16)
    assert bench.traffic_for("no-such-phase", 16) is None


def test_timed_launch_count(bench):
    assert bench.timed_launches(64, 8, 16, 6) == 6 * 8 * 64  # 4 graph launches of 16 iterations x 8 branches
    assert bench.timed_launches(64, 8, 4, 6) == 6 * 4 * 64   # branches clamp to the batch
    assert bench.timed_launches(20, 8, 16, 7) == 7 * (8 * 16 + 4)  # 16 in the graph + 4 eager
    assert bench.timed_launches(64, 8, 296, 7, 2) == 7 * 8 * 64 + 2 * 8 * 4  # + gather / expand per branch and graph launch
    assert bench.timed_launches(20, 8, 296, 7, 2) == 7 * (8 * 16 + 4) + 2 * 8 + 2  # + one gather / expand around the eager remainder
    assert bench.kernels_per_iteration("float64") == 7  # + k_advect_uniq64
    assert bench.kernels_per_iteration("mixed") == 6
    assert bench.kernels_per_iteration("float32") == 6  # advect fused into k_region by default
