import sys, time
sys.path[:0] = ['.', 'tests']
import fixture_maps as fm
import paper_2604_13880_b200 as P
m = fm.many_holes(300)
crit = P.StoppingCriteria(1e-300, 10**9, 60)
eng = P.CartogramEngine(m, criteria=crit, k=11)
eng.run()
t0 = time.perf_counter(); eng.run(); dt = time.perf_counter() - t0
print("many_holes(400) rows", eng.initial_map.vertex_array().shape[0], "it/s", round(60 / dt, 1))
