"""Background-density multiplier sweep -- the computation of cartomorph's ``cmd_sweep_bdv``
(cli.py:265-300), batched on the GPU.

The reference runs one engine per multiplier, one after another, each followed by a quality
report.  Here all multipliers run as ONE device batch (``BatchEngine``: one cartogram per
multiplier, every kernel launch covers all of them), and their reports come from one pass of the
metric kernels (``metrics.frame_reports``).  The result is the reference's ``bdv_sweep.csv``
text, row for row.  Argument parsing and file output belong to the CLI and stay out of scope.
"""

from __future__ import annotations

import functools
import time

import numpy as np

from .engine import BatchEngine, StoppingCriteria
from .errors import CartomorphError, IngestionError
from .geomodel import ring_layout
from .metrics import frame_reports
from .shard import run_sharded

SWEEP_HEADER = "multiplier,stop_reason,iterations,xi,epsilon,tau,hamming_avg,hamming_max,position_error,wall_ms,error"


def sweep_bdv(mapmodel, multipliers, criteria: StoppingCriteria | None = None, k: int = 10, hamming_k: int = 7, *,
              device: int = 0, field_dtype: str = "float64", devices=None, distributed: bool = False):
    """``(csv_text, results)`` for the sorted multipliers (cli.py:265-300); ``results[i]`` is the
    RunResult (or the CartomorphError) of the i-th sorted multiplier.

    ``devices=[...]`` / ``distributed=True`` shard the multipliers over one process per GPU
    (shard.run_sharded); each process runs its block as one batch with its reports."""
    mults = sorted(float(m) for m in multipliers)
    if any(not (0.5 <= m <= 2.0) for m in mults):
        raise IngestionError("multipliers must lie in [0.5, 2]")
    criteria = criteria or StoppingCriteria(error_threshold=0.01, stagnation_window=32, max_iterations=512)
    rows = [SWEEP_HEADER]
    if not mults:
        return "\n".join(rows) + "\n", []
    task = functools.partial(_sweep_block, mapmodel, mults, criteria, k, hamming_k, field_dtype)
    if devices is None and not distributed:
        parts = task(0, len(mults), device)
    else:
        parts = run_sharded(len(mults), task, devices=devices, distributed=distributed)
    rows += [p[0] for p in parts]
    return "\n".join(rows) + "\n", [p[1] for p in parts]


def _sweep_block(mapmodel, all_mults, criteria, k, hamming_k, field_dtype, lo, hi, device):
    """[(csv row, result)] of multipliers [lo, hi) as one device batch on `device`."""
    mults = all_mults[lo:hi]
    rows = []
    began = time.perf_counter()
    stats = mapmodel.statistics() if hasattr(mapmodel, "statistics") else np.array([r.statistic for r in mapmodel.regions])
    try:
        be = BatchEngine(mapmodel, np.tile(np.asarray(stats, dtype=float), (len(mults), 1)), criteria=criteria, k=k,
                         bdv_multiplier=np.asarray(mults), device=device, field_dtype=field_dtype)
        results = be.run_all()
    except CartomorphError as exc:  # a start-map problem fails every multiplier alike
        wall_ms = (time.perf_counter() - began) * 1e3 / len(mults)
        return [(f"{m:.6g},failed,,,,,,,,{wall_ms:.3f},{exc}", exc) for m in mults]
    wall_ms = (time.perf_counter() - began) * 1e3 / len(mults)
    ok = [i for i, r in enumerate(results) if not isinstance(r, Exception)]
    reports = {}
    if ok:
        _, rs, rr, ids, _ = ring_layout(be.initial_map)
        xy = np.stack([results[i].state.mapmodel.vertex_array() for i in ok])
        # cli.py:155-157: the statistic share of each engine's total mass
        weights = [np.asarray(stats, dtype=float) / (be.total_statistic[i] + be.background_mass[i]) for i in ok]
        reps = frame_reports(be.initial_map, (None, rs, rr, len(ids)), xy, [stats] * len(ok), weights, hamming_k,
                             [wall_ms] * len(ok), device=device)
        reports = dict(zip(ok, reps))
    out = []
    for i, (m, res) in enumerate(zip(mults, results)):
        rep = reports.get(i)
        err = res if isinstance(res, Exception) else (rep if isinstance(rep, Exception) else None)
        if err is not None:
            if not isinstance(err, CartomorphError):
                raise err
            rows.append(f"{m:.6g},failed,,,,,,,,{wall_ms:.3f},{err}")
            out.append(err)
            continue
        st = res.state
        rows.append(f"{m:.6g},{res.stop_reason},{st.iteration},{st.xi:.9g},{st.epsilon:.9g},{rep.tau:.9g},"
                    f"{rep.hamming_avg:.9g},{rep.hamming_max:.9g},{rep.position_error:.9g},{wall_ms:.3f},")
        out.append(res)
    return list(zip(rows, out))
