"""Per-phase eager kernel times at the headline workload (diagnostics).

python tools/phase_split.py -> JSON: ms per iteration per phase for 16 frames, with k_region
in full mode and (DET_KT_REGION_MODE=1 in a child process) advect-only mode.
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def measure():
    import numpy as np
    import paper_2604_13880_b200 as P
    from paper_2604_13880_b200.synthetic import config_map

    m, prm = config_map("headline")
    s0 = m.statistics()
    rng = np.random.default_rng(0)
    walk = np.stack([s0 * np.exp(rng.normal(0, 0.15, s0.shape)) for _ in range(16)])  # as bench.py
    crit = P.StoppingCriteria(1e-300, 10**9, 1)
    be = P.BatchEngine(m, walk, criteria=crit, k=10, bdv_multiplier=prm["bdv_multiplier"])
    ctx = be.launch(crit)
    ctx.bench_iterations(32)
    ctx.sync()
    ph = ctx.kernel_times(16)
    return dict(zip(["integral_images", "region", "row", "ctrl"], [v / 16 for v in ph]))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        print(json.dumps(measure()))
    else:
        out = {}
        for mode in ("full", "advect_only", "row_no_eval"):
            env = dict(os.environ, DET_KT_REGION_MODE="1" if mode == "advect_only" else "0",
                       DET_KT_ROW_MODE="-1" if mode == "row_no_eval" else "0")
            r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
            out[mode] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
        print(json.dumps(out))
