import sys, numpy as np
sys.path[:0] = ['.', 'tests']
import fixture_maps as fm
import paper_2604_13880_b200 as P
m = fm.config1()
for field in ["float64", "float32"]:
    for T in (4, 5, 6, 6, 8):
        crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=T)
        eng = P.CartogramEngine(m, criteria=crit, k=8, bdv_multiplier=0.5, field_dtype=field)
        full = eng.run()
        print(field, T, full.stop_reason, [round(t.xi, 6) for t in full.trace], round(full.state.xi, 6), full.state.iteration, flush=True)
    # k=6 two-region (the passing test)
    for T in (3, 4, 6):
        eng = P.CartogramEngine(fm.two_region((1.0, 3.0)), P.StoppingCriteria(1e-300, 10**9, T), k=6, field_dtype=field)
        full = eng.run()
        print(field, "two", T, [round(t.xi, 6) for t in full.trace])
