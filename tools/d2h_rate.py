"""Read-back rate of a batch's results (det_get_results into a pinned block): GB/s over PCIe."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import config_map, random_walk

B = int(sys.argv[1]) if len(sys.argv) > 1 else 296
m, prm = config_map("headline")
walk = np.concatenate([random_walk(m.statistics(), 8, 0.15, seed=7 + 31 * i) for i in range((B + 7) // 8)])[:B]
crit = P.StoppingCriteria(1e-300, 10**9, 16)
be = P.BatchEngine(m, walk, criteria=crit, k=10)
be.run_all()
ctx = be._ctx()
verts = ctx.pinned.empty((B, be._xy.shape[0], 2))
for rep in range(3):
    t = time.perf_counter()
    ctx.results_all(verts, 17)
    dt = time.perf_counter() - t
    print(f"results_all: {dt*1e3:.1f} ms for {verts.nbytes/1e9:.2f} GB -> {verts.nbytes/1e9/dt:.1f} GB/s")
t = time.perf_counter(); out = be.run_all(); print("run_all 16 iterations", time.perf_counter() - t, be.last_timing)
