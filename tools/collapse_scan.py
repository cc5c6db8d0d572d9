"""Diagnostic: first-collapse iteration of headline-size maps under several statistic spreads (GPU)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import voronoi_map, random_walk

for lloyd in (0, 1):
    for sigma in (0.25, 0.5, 0.75, 1.0):
        m = voronoi_map(3000, seed=3, target_unique=200_000, sigma=sigma, lloyd=lloyd)
        walk = random_walk(m.statistics(), 8, 0.15, seed=7)
        t = time.time()
        be = P.BatchEngine(m, walk, criteria=P.StoppingCriteria(1e-300, 10**9, 2000), k=10)
        res = be.run_all()
        out = []
        for r in res:
            out.append(r.iteration if isinstance(r, P.RegionCollapsedError) else -1)
        print(f"lloyd={lloyd} sigma={sigma}: collapse iterations {out} ({time.time()-t:.1f}s)", flush=True)
