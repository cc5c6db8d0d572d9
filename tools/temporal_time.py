"""Wall time of the transition modes on BASELINE config 2 (cumulative, 12 x 100) and a direct run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_13880_b200 as P
from paper_2604_13880_b200.synthetic import config_map, random_walk

m, prm = config_map("c2")
walk = random_walk(m.statistics(), prm["steps"], prm["walk_sigma"], seed=21)
ds = P.TimeSeriesDataset(m, tuple(f"t{i}" for i in range(prm["steps"])), walk)
crit = P.StoppingCriteria(1e-300, 10**9, prm["iterations"])
for mode, fn in (("cumulative", P.run_cumulative), ("direct", P.run_direct)):
    for rep in range(2):
        t = time.perf_counter()
        seq = fn(ds, crit, k=prm["k"])
        dt = time.perf_counter() - t
        ok = sum(f.error is None for f in seq.frames)
        print(f"{mode:10s} rep{rep}: {dt*1e3:8.1f} ms for {len(seq.frames)} frames x {prm['iterations']} it "
              f"({ok} ok) -> {len(seq.frames)/dt:.1f} time steps/s, {len(seq.frames)*prm['iterations']/dt:.0f} it/s")
