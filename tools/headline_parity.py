"""Parity of the benchmarked workload against the oracle (diagnostics; the -m gpu test is
tests/test_gpu_headline.py).

python tools/headline_parity.py [frames] [iterations] [config]

Runs `frames` direct-mode frames of the bench workload (config_map(config), the bench's
random walk) for `iterations` DET iterations on the GPU in BOTH field dtypes, and the oracle
engine for the same frames in a process pool over the host cores.  Prints one JSON line per
frame plus a summary: max vertex deviation, shoelace-area relative error, pixel-count
differences, and whether the final state's raster equals the oracle raster of the same vertices.
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import det_oracle as O  # noqa: E402
from paper_2604_13880_b200.synthetic import config_map, random_walk  # noqa: E402

_M = {}
DTYPES = ("float32", "mixed", "float64")


def _oracle(args):
    b, stats, k, mult, iters = args
    t0 = time.perf_counter()
    eng = O.OracleEngine(O.FlatMap.from_mapmodel(_M["m"].with_statistics(stats)), k=k, bdv_multiplier=mult)
    r = eng.run(1e-300, 10**9, iters)
    return b, r.rows, r.counts, np.array([t[:3] for t in r.trace]), time.perf_counter() - t0


def shoelace(rows, ring_start, ring_region, R):
    out = np.zeros(R)
    for q in range(len(ring_start) - 1):
        a, e = ring_start[q], ring_start[q + 1]
        if e - a < 3:
            continue
        p = rows[a:e]
        nx = np.roll(p, -1, axis=0)
        out[ring_region[q]] += 0.5 * float(np.sum(p[:, 0] * nx[:, 1] - nx[:, 0] * p[:, 1]))
    return out


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    cfg = sys.argv[3] if len(sys.argv) > 3 else "headline"
    m, prm = config_map(cfg)
    k = prm.get("k", 10)
    mult = prm.get("bdv_multiplier", 1.0)
    walk = random_walk(m.statistics(), frames, prm.get("walk_sigma", 0.15), seed=7)
    _M["m"] = m
    procs = min(frames, len(os.sched_getaffinity(0)))
    pool = mp.get_context("fork").Pool(procs)
    jobs = pool.map_async(_oracle, [(b, walk[b], k, mult, iters) for b in range(frames)])

    import paper_2604_13880_b200 as P
    from paper_2604_13880_b200.geomodel import ring_layout

    crit = P.StoppingCriteria(1e-300, 10**9, iters)
    gpu = {}
    for fd in DTYPES:
        t0 = time.perf_counter()
        be = P.BatchEngine(m, walk, criteria=crit, k=k, bdv_multiplier=mult, field_dtype=fd)
        res = be.run_all()
        gpu[fd] = (res, time.perf_counter() - t0)
    xy0, rs, rr, ids, _ = ring_layout(gpu["float32"][0][0].state.mapmodel)
    R = len(ids)
    out = jobs.get()
    pool.close()
    summary = {"config": cfg, "frames": frames, "iterations": iters, "host_cores": procs,
               "k": k, "rows": int(xy0.shape[0])}
    worst = {}
    for b, rows_o, cnt_o, tr_o, sec in out:
        a_o = shoelace(rows_o, rs, rr, R)
        line = {"frame": b, "oracle_s": round(sec, 1)}
        for fd in DTYPES:
            res = gpu[fd][0][b]
            if isinstance(res, Exception):
                line[fd] = {"error": str(res)}
                continue
            v = res.state.mapmodel.vertex_array()
            cnt = res.state.pixel_counts
            a = shoelace(v, rs, rr, R)
            dc = np.abs(cnt.astype(np.int64) - cnt_o.astype(np.int64))
            tr = np.array([[t.iteration, t.epsilon, t.xi] for t in res.trace])
            lab = res.state.labels.labels
            lab_o = O.FlatMap.from_mapmodel(res.state.mapmodel).labels(k)
            d = {"max_vertex_dev": float(np.abs(v - rows_o).max()),
                 "area_rel_max": float((np.abs(a - a_o) / np.abs(a_o)).max()),
                 "count_absdiff_max": int(dc.max()), "count_rel_max": float((dc / cnt_o).max()),
                 "regions_count_diff": int((dc > 0).sum()),
                 "cart_err_absdiff_max": float(np.abs(res.state.per_region_error -
                                                       np.abs(cnt_o - res.weights_px) /
                                                       np.maximum(cnt_o, res.weights_px)).max()),
                 "eps_final": float(tr[-1, 1]), "eps_final_oracle": float(tr_o[-1, 1]),
                 "xi_final": float(tr[-1, 2]), "xi_final_oracle": float(tr_o[-1, 2]),
                 "trace_eps_absdiff_max": float(np.abs(tr[:, 1] - tr_o[:, 1]).max()),
                 "raster_of_own_state_exact": bool(np.array_equal(lab, lab_o))}
            line[fd] = d
            for key in ("max_vertex_dev", "area_rel_max", "count_absdiff_max", "count_rel_max",
                        "trace_eps_absdiff_max"):
                worst.setdefault(fd, {})[key] = max(worst.get(fd, {}).get(key, 0), d[key])
            worst[fd]["raster_exact_all"] = worst[fd].get("raster_exact_all", True) and d["raster_of_own_state_exact"]
        print(json.dumps(line), flush=True)
    summary["worst"] = worst
    summary["gpu_s"] = {fd: round(gpu[fd][1], 2) for fd in gpu}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
