"""Small engine runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).
usage: python tools/sanitize_case.py [float64|mixed|float32] [iterations]"""
import sys
import numpy as np
sys.path[:0] = ['.', 'tests']
import fixture_maps as fm
import paper_2604_13880_b200 as P

field = sys.argv[1] if len(sys.argv) > 1 else "float64"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
m = fm.config1()
crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=iters)
res = P.CartogramEngine(m, criteria=crit, k=8, bdv_multiplier=0.5, field_dtype=field).run()
print(field, "config1 k=8", [round(t.xi, 6) for t in res.trace])
# stagnation stop (best-state re-evaluation) and a collapse
res = P.CartogramEngine(m, criteria=P.StoppingCriteria(1e-300, 2, 8), k=7, field_dtype=field).run()
print(field, "stagnation-window 2:", res.stop_reason, res.state.iteration)
s = fm.sliver()
try:
    P.CartogramEngine(s, criteria=P.StoppingCriteria(1e-300, 10**9, 40), k=6, field_dtype=field).run()
    print(field, "sliver: no collapse")
except P.RegionCollapsedError as e:
    print(field, "sliver collapse:", e)
tex = P.rasterize_labels(fm.many_holes(60), 9, check_collapse=False)
print("many_holes raster", np.bincount(tex.labels[tex.labels >= 0]))
