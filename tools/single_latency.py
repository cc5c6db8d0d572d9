"""Latency of one cartogram (B=1) through CartogramEngine.run on the headline map (diagnostics)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13880_b200 as P  # noqa: E402
from paper_2604_13880_b200.synthetic import config_map  # noqa: E402

m, prm = config_map(sys.argv[1] if len(sys.argv) > 1 else "headline")
if len(sys.argv) > 2:  # band height override for the experiment
    from paper_2604_13880_b200._context import get_context
    get_context(prm["k"]).set_band_height(int(sys.argv[2]))
crit = P.StoppingCriteria(1e-300, 10**9, 200)
P.CartogramEngine(m, criteria=crit, k=prm["k"]).run()  # warm (allocation, graph capture)
out = {}
for rep in range(3):
    t0 = time.perf_counter()
    eng = P.CartogramEngine(m, criteria=crit, k=prm["k"])
    t1 = time.perf_counter()
    res = eng.run()
    t2 = time.perf_counter()
    out[rep] = {"construct_ms": (t1 - t0) * 1e3, "run_ms": (t2 - t1) * 1e3, "it_per_s": 200 / (t2 - t1)}
print(json.dumps(out))
