"""Phase timing of the end-to-end public-API call (BatchEngine.run_all) on the headline workload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import config_map, random_walk

m, prm = config_map("headline")
walk = random_walk(m.statistics(), 16, 0.15, seed=7)
crit = P.StoppingCriteria(1e-300, 10**9, 200)
t0 = time.perf_counter()
be = P.BatchEngine(m, walk, criteria=crit, k=10)
print(f"BatchEngine init  {1e3*(time.perf_counter()-t0):8.1f} ms")
if os.environ.get("NOWARM") != "1":
    be.run_all()  # warm (graph capture, allocation)
for rep in range(2):
    be._token = None
    T = {}
    t = time.perf_counter(); ctx = be._ctx(); T["load_map+set_batch (H2D)"] = time.perf_counter() - t
    t = time.perf_counter(); ctx.set_params(be._params(), be.weights_px); T["set_params"] = time.perf_counter() - t
    t = time.perf_counter(); ctx.run(crit.error_threshold, crit.stagnation_window, crit.max_iterations); T["det_run (200 it x 16)"] = time.perf_counter() - t
    t = time.perf_counter(); verts = ctx.pinned.empty((be.B, be._xy.shape[0], 2)); T["pinned block"] = time.perf_counter() - t
    t = time.perf_counter(); res = [be._collect(ctx, b, 0, 0, verts[b]) for b in range(be.B)]; T["collect (D2H + results)"] = time.perf_counter() - t
    tot = sum(T.values())
    for k, v in T.items():
        print(f"  {k:28s} {1e3*v:8.1f} ms")
    print(f"  total {1e3*tot:.1f} ms -> e2e {16*200/tot:.0f} it/s")

# finer split of collect for one frame
import time as _t
ctx = be._ctx()
pv = ctx.pinned.empty((be._xy.shape[0], 2))
for name, fn in [("result", lambda: ctx.result(0)), ("trace", lambda: ctx.trace(0, 201)), ("vertices", lambda: ctx.vertices(0)),
                 ("vertices(pinned)", lambda: ctx.vertices(0, pv)),
                 ("counts", lambda: ctx.counts(0)), ("region_error", lambda: ctx.region_error(0)),
                 ("collect(1 frame)", lambda: be._collect(ctx, 0, 0, 0, pv))]:
    t = _t.perf_counter()
    for _ in range(10):
        fn()
    print(f"  {name:20s} {1e2*(_t.perf_counter()-t):8.3f} ms")
