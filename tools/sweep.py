"""Run bench.py over a grid of options and print one summary line each (GPU box helper)."""
import itertools, json, subprocess, sys

grid = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {"groups": [1, 2, 4], "batch": [8, 16]}
base = ["python", "bench.py", "--steps", "64", "--warmup", "8", "--no-cpu", "--e2e-steps", "8"]
keys = list(grid)
for combo in itertools.product(*[grid[k] for k in keys]):
    args = base + sum([[f"--{k}", str(v)] for k, v in zip(keys, combo)], [])
    out = subprocess.run(args, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        ph = d["roofline"]["phase_ms_per_iteration"]
        print(dict(zip(keys, combo)), f"value={d['value']:.0f} it/s  step={d['ms_per_step']*1e3:.1f}us "
              f"executed={d['iterations_executed']:.0f} frac_step={d['roofline']['step']['frac']:.3f}", flush=True)
    except Exception as exc:
        print(dict(zip(keys, combo)), "FAILED", exc, out.stderr[-500:], flush=True)
