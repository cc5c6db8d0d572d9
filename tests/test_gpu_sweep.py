"""bdv multiplier sweep (cli.py:265-300) as one GPU batch, against the reference's own rows
(tests/golden/sweep.npz): stop reason, iterations, xi, epsilon, tau and Hamming values exact (float64
field), position error at 1e-9."""

import os

import numpy as np
import pytest

import fixture_maps as fm

pytestmark = pytest.mark.gpu


def test_sweep_rows_match_reference(golden_dir):
    from paper_2604_13880_b200 import IngestionError, StoppingCriteria
    from paper_2604_13880_b200.sweep import SWEEP_HEADER, sweep_bdv

    z = np.load(os.path.join(golden_dir, "sweep.npz"))
    m = fm.unpack_map(z)
    csv, results = sweep_bdv(m, [1.7, 0.5, 1.0], StoppingCriteria(0.01, 32, 15), k=6, hamming_k=6,
                             field_dtype="float64")
    lines = csv.strip().split("\n")
    assert lines[0] == SWEEP_HEADER and len(lines) == 4 and len(results) == 3
    for got, ref in zip(lines[1:], [str(r) for r in z["rows"]]):
        g, r = got.split(","), ref.split(",")
        assert g[:8] == r[:8], (got, ref)  # multiplier .. hamming_max
        assert float(g[8]) == pytest.approx(float(r[8]), rel=1e-9)  # position error
        assert g[10] == ""  # no error
    with pytest.raises(IngestionError):
        sweep_bdv(m, [0.3])
