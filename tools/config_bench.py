"""Device throughput of the DET iteration on BASELINE configs 2-5 (diagnostics, one JSON line each).

python tools/config_bench.py [c2 c3 c4 c5] -- B frames of each config's map with lognormal(0, 0.5)
statistics (random walk, sigma 0.15), bench-mode iterations timed with CUDA events, executed iterations only.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_13880_b200 as P  # noqa: E402
from paper_2604_13880_b200.synthetic import config_map, random_walk  # noqa: E402

BATCH = {"c2": 64, "c3": 16, "c4": 64, "c5": 8}
ROOF = {"c2": 189e3, "c3": 45.5e3, "c4": 189e3, "c5": 10.9e3}  # SURVEY §8(d), 100% of measured HBM


def run(name):
    t0 = time.perf_counter()
    m, prm = config_map(name)
    B = BATCH[name]
    # throughput on the config's map and texture size with lognormal(0, 0.5) statistics (as the
    # headline): the configs' own heavy-tailed statistics collapse frames within the timed window
    s0 = np.exp(np.random.default_rng(5).normal(0.0, 0.5, len(m.regions)))
    # 16-step walks (as bench.py): longer ones drift far enough for small regions to collapse
    walk = np.concatenate([random_walk(s0, min(16, B - lo), 0.15, seed=11 + lo) for lo in range(0, B, 16)])
    crit = P.StoppingCriteria(1e-300, 10**9, 1)
    be = P.BatchEngine(m, walk, criteria=crit, k=prm["k"], bdv_multiplier=prm.get("bdv_multiplier", 1.0))
    ctx = be.launch(crit)
    ctx.bench_iterations(32)
    ctx.sync()
    it0, _ = ctx.progress()
    ms = ctx.time_iterations(64)
    it1, act = ctx.progress()
    ex = int((it1 - it0).sum())
    v = ex / (ms * 1e-3)
    return {"config": name, "k": prm["k"], "regions": len(m.regions), "rows": int(be._xy.shape[0]), "frames": B,
            "it_per_s": v, "frac_of_roofline": v / ROOF[name], "active_after": int(act.sum()),
            "setup_s": time.perf_counter() - t0}


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
        print(json.dumps(run(name)))
