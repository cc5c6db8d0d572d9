"""Benchmark: DET iterations/s at 1024^2 texture, ~200k vertices (BASELINE.json metric).

Workload ("headline"): the 3000-region seeded Voronoi map with ~200k unique
vertices (synthetic), 1024^2 texture, run as direct-mode time
steps: every GPU holds a batch of B independent frames (statistics = a seeded
lognormal random walk over time) and one bench "step" is one DET iteration of
every frame in the batch (B = 296 by default: 37 eight-step random walks).  Inputs are device-resident before
timing; the batch working set (~45 MB per frame with the float64 field) is larger than
the 126 MB L2 for B >= 3.

    python bench.py [--gpus N --steps K --warmup W --batch B]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)
    python bench.py --impl reference ...                      (CPU reference arm)

Multi-GPU: frames are sharded across ranks (weak scaling), no collective in
the timed region; a final NCCL gather collects per-frame errors.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics as pystats
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DET iterations/s at 1024\u00b2 texture, 200k vertices; time steps/s over 8 GPUs"  # BASELINE.json verbatim
UNIT = "DET iterations/s"
K_TEX = 10
WALK_STEPS = int(os.environ.get("DET_WALK_STEPS", "8"))  # time steps per random walk of the bench batch (see build_workload)


def algorithmic_bytes_per_iteration(n: int, n_unique: int) -> float:
    """B = 28 n^2 + 32 N_u + min(100 N_u, 20 n^2) per DET iteration."""
    return 28.0 * n * n + 32.0 * n_unique + min(100.0 * n_unique, 20.0 * n * n)


def phase_bytes(n: int, n_unique: int, n_rows: int, n_regions: int, field: str = "float64") -> dict:
    """Algorithmic bytes per iteration of each phase, in the run's field dtype:
    fb = bytes per field component (8 float64, 4 float32), sb = bytes per state coordinate."""
    fb = 8 if field == "float64" else 4
    sb = 4 if field == "float32" else 8
    return {
        # integral images -> field: read labels (4 n^2), write the two-component field (2 fb n^2)
        "integral_images": (4.0 + 2 * fb) * n * n,
        # advect + crossings: per unique vertex read + write of the state (4 sb) and the four
        # two-component field texels of its bilinear tap (8 fb)
        "region": (4.0 * sb + 8.0 * fb) * n_unique,
        # paint: write labels (4 n^2)
        "row": 4.0 * n * n,
        "ctrl": 0.0,
    }


def kernels_per_iteration(field: str) -> int:
    """Band sums, carries, sweep (k_sat1x, k_sat2p, k_sat3x on the float64 path), k_region, k_row, k_ctrl, plus the
    advect as its own kernel:
    k_advect_uniq64s on the float64 path (one thread per unique vertex; DET_UNIQ_ADVECT=0 fuses it
    back into k_region), k_advect_rows on the float32 path when DET_SPLIT_ADVECT=1."""
    if field == "float64":
        split = os.environ.get("DET_UNIQ_ADVECT", "1") != "0" or os.environ.get("DET_SPLIT_ADVECT", "0") == "1"
    else:
        split = field == "float32" and os.environ.get("DET_SPLIT_ADVECT", "0") == "1"
    return 7 if split else 6


def timed_launches(steps: int, groups: int, batch: int, per_iter: int = 7, per_graph: int = 0) -> int:
    """Our kernel launches in the timed region: per_iter kernels per frame group per iteration;
    full 16-iteration chunks run as a CUDA graph with min(groups, batch) branches (plus per_graph
    kernels per branch and graph launch: the float64 path's k_uq_gather / k_uq_expand), the
    remainder eagerly over the whole batch."""
    g = min(groups, batch)
    return (per_iter * (g * 16 * (steps // 16) + steps % 16) + per_graph * g * (steps // 16)
            + (per_graph if steps % 16 else 0))  # the eager remainder gathers / expands once over the whole batch


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": float(pystats.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def build_workload(batch: int, rank: int, world: int):
    from paper_2604_13880_b200.synthetic import config_map, random_walk

    m, prm = config_map("headline")
    # weak scaling: every rank runs its own frames from the base statistics (rank 0's are the N=1
    # workload), so per-GPU work has the same distribution at every N.  The frames are time steps of
    # random walks of at most WALK_STEPS steps (a new walk from the base statistics every WALK_STEPS
    # frames): a longer walk drifts far enough (sigma 0.15 per step) for this 3000-region map's
    # smallest regions to collapse within the run (RegionCollapsedError, as in the reference), which
    # would leave frames of the batch idle
    walks = [random_walk(m.statistics(), min(WALK_STEPS, batch - lo), 0.15, seed=7 + 1009 * rank + 31 * (lo // WALK_STEPS))
             for lo in range(0, batch, WALK_STEPS)]
    return m, prm, np.concatenate(walks)


# ------------------------------------------------------------------ CPU reference arm / baseline
_CPU = {}  # the headline map, built once in the parent before the pool forks


def _cpu_map():
    if "m" not in _CPU:
        from paper_2604_13880_b200.synthetic import config_map

        _CPU["m"] = config_map("headline")[0]
    return _CPU["m"]


def _cpu_worker(args):
    """One frame of the oracle engine: set-up (densify, start raster) untimed, then `iters` timed
    iterations of OracleEngine.run; returns (iterations, seconds of the timed run)."""
    stats, iters = args
    sys.path.insert(0, ROOT)
    from oracle import det_oracle as O

    eng = O.OracleEngine(O.FlatMap.from_mapmodel(_cpu_map().with_statistics(stats)), k=K_TEX)
    bar = _CPU.get("barrier")
    if bar is not None:
        bar.wait()  # every worker starts its timed run together
    t0 = time.perf_counter()
    eng.run(error_threshold=1e-300, stagnation_window=10**9, max_iterations=iters)
    return iters, time.perf_counter() - t0


def _pool_init(bar):
    _CPU["barrier"] = bar


def cpu_measure(walk, iters: int, procs: int):
    """Oracle DET iterations/s on `procs` host cores: a process pool over independent frames, each
    worker timing only its engine's iterations (set-up excluded, all workers released together by a
    barrier); rate = sum of iterations / the slowest worker's seconds."""
    _cpu_map()
    if procs <= 1:
        it, sec = _cpu_worker((walk[0], iters))
        return it / sec, f"1 frame x {iters} iterations of the headline workload (oracle port, 1 core, set-up excluded)"
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    bar = ctx.Barrier(procs)
    jobs = [(walk[i % len(walk)], iters) for i in range(procs)]
    with ctx.Pool(procs, initializer=_pool_init, initargs=(bar,)) as pool:
        out = pool.map(_cpu_worker, jobs, chunksize=1)
    total = sum(o[0] for o in out)
    slowest = max(o[1] for o in out)
    per_core = float(np.median([o[0] / o[1] for o in out]))
    return total / slowest, (f"{procs} frames x {iters} iterations in a {procs}-process pool (oracle port); "
                             f"set-up untimed; sum(iterations)/max(worker seconds); median single-worker "
                             f"rate {per_core:.3f} it/s")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0))
    m, prm, walk = build_workload(max(args.batch, procs), 0, 1)
    iters = max(5, min(args.steps, 8))  # a bounded sample: 5-8 iterations per frame on every core
    value, sample = cpu_measure(walk, iters, procs)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "headline: 3000-region Voronoi map, ~200k unique vertices, 1024^2 texture, "
                                   "direct-mode time steps", "k": K_TEX},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": sample + "; each iteration's timing includes its raster/density/integral "
                                                "images/field/advect exactly as the reference engine"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU arm
TRAFFIC_SRC = "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch / frames per launch)"


def traffic_for(phase, batch):
    """DRAM bytes of the dominant phase per launch-iteration over `batch` frames, from a committed ncu capture."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            per = json.load(f)["per_frame_bytes_by_phase"]
        return per[phase] * batch if phase in per else None
    except (OSError, ValueError, KeyError):
        return None


def paper_units(P, m, walk, field, device):
    """One headline cartogram alone (B = 1, 200 iterations through CartogramEngine.run) and the
    config-2 cumulative chain (run_cumulative, 12 steps x 100 iterations), wall-clock around the
    public calls after a warm-up call (results read back included)."""
    import gc

    from paper_2604_13880_b200.synthetic import config_map, random_walk

    out = {}
    crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=200)
    eng = P.CartogramEngine(m.with_statistics(walk[0]), criteria=crit, k=K_TEX, device=device, field_dtype=field)
    eng.run()
    gc.collect()
    t0 = time.perf_counter()
    res = eng.run()
    dt = time.perf_counter() - t0
    out["single_cartogram"] = {"iterations": res.state.iteration, "seconds": dt,
                               "it_per_s": res.state.iteration / dt, "ms_per_iteration": 1e3 * dt / res.state.iteration,
                               "note": "one headline frame (3000 regions, 1024^2) through CartogramEngine.run, "
                                       "host map in and results out"}
    m2, prm2 = config_map("c2")
    w2 = random_walk(m2.statistics(), prm2["steps"], prm2["walk_sigma"], seed=21)
    ds = P.TimeSeriesDataset(m2, tuple(f"t{i}" for i in range(prm2["steps"])), w2)
    crit2 = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=prm2["iterations"])
    P.run_cumulative(ds, crit2, k=prm2["k"], device=device, field_dtype=field)
    gc.collect()
    t0 = time.perf_counter()
    seq = P.run_cumulative(ds, crit2, k=prm2["k"], device=device, field_dtype=field)
    dt = time.perf_counter() - t0
    ok = sum(fr.error is None for fr in seq.frames)
    out["cumulative_chain_c2"] = {"time_steps": len(seq.frames), "ok_steps": ok, "iterations_per_step": prm2["iterations"],
                                  "seconds": dt, "time_steps_per_s": len(seq.frames) / dt,
                                  "note": "BASELINE config 2: 500 regions, ~40k vertices, 1024^2, 12 warm-started "
                                          "steps x 100 iterations, per-frame quality reports included"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--batch", type=int, default=296, help="frames per GPU (DESIGN.md §5: 16-296 swept; 296 = two per SM)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--band", type=int, default=0, help="band height of the integral-image kernels (0 = auto)")
    ap.add_argument("--field", default="float64", choices=["float64", "mixed", "float32"])
    ap.add_argument("--groups", type=int, default=8, help="frame groups run as parallel graph branches")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--no-extra", action="store_true", help="skip the single-cartogram / chain measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2604_13880_b200 as P
    from paper_2604_13880_b200._lib import device_info

    m, prm, walk = build_workload(args.batch, rank, world)
    crit = P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=1)
    be = P.BatchEngine(m, walk, criteria=crit, k=K_TEX, bdv_multiplier=prm["bdv_multiplier"], device=local,
                       field_dtype=args.field)
    ctx = be._ctx()
    if args.band:
        ctx.set_band_height(args.band)
    ctx.set_groups(args.groups)
    be.launch(crit)  # state 0 -> 1 on the device; builds the CUDA graph
    n_unique = int(np.unique(be._xy.view(np.complex128).ravel()).shape[0])
    n_rows = be._xy.shape[0]
    ctx.bench_iterations(args.warmup)
    ctx.sync()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with ClockSampler(local) as clk:
        # soak ~0.5 s under the same load so the clock record covers the timed region's conditions
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.5:
            ctx.bench_iterations(16)
            ctx.sync()
        it0, _ = ctx.progress()
        barrier()
        if os.environ.get("DET_PROFILE_RANGE") == "2":  # ncu --profile-from-start off: the timed graph launches
            torch.cuda.profiler.start()
        ms = ctx.time_iterations(args.steps)
        if os.environ.get("DET_PROFILE_RANGE") == "2":
            torch.cuda.profiler.stop()
        barrier()
        it1, act = ctx.progress()
    executed = int((it1 - it0).sum())  # iterations actually executed (a collapsed frame stops counting)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    ex_t = torch.tensor([executed], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ex_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    n = 1 << K_TEX
    iters_total = float(ex_t.item())
    value = iters_total / (ms_max * 1e-3)

    # per-phase device times (eager launches, events on the same stream) -> dominant kernel
    prof_range = os.environ.get("DET_PROFILE_RANGE") == "1"  # ncu --profile-from-start off: the eager launches
    if prof_range:
        torch.cuda.profiler.start()
    ph = ctx.kernel_times(8)
    if prof_range:
        torch.cuda.profiler.stop()
    names = ["integral_images", "region", "row", "ctrl"]
    per_iter_ms = {k: v / 8 for k, v in zip(names, ph)}
    dom = max(per_iter_ms, key=per_iter_ms.get)
    pbytes = phase_bytes(n, n_unique, n_rows, len(m.regions), args.field)
    peak, peak_kind = load_peaks()
    dom_achieved = pbytes[dom] * args.batch / (per_iter_ms[dom] * 1e-3) / 1e9
    step_bytes = algorithmic_bytes_per_iteration(n, n_unique) * args.batch
    step_achieved = algorithmic_bytes_per_iteration(n, n_unique) * iters_total / world / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API: host map in, host results out ----
    e2e_steps = args.e2e_steps or prm["iterations"]  # one full time step per frame
    # settle the Python GC debt of the setup above (torch import, workload construction) and of
    # the previous repetition, so that a full collection does not land inside a timed call
    import gc

    e2e_runs = []
    res = None
    for _ in range(3):  # median of 3 timed public-API calls (host noise)
        res = None  # the previous results release their page-locked block back to the pool
        be._token = None  # every call uploads the map again
        gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = be.run_all(P.StoppingCriteria(error_threshold=1e-300, stagnation_window=10**9, max_iterations=e2e_steps))
        torch.cuda.synchronize()
        e2e_runs.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_runs))

    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    if os.environ.get("DET_E2E_DEBUG") == "1":  # per-getter host timings after the e2e call (stderr)
        cx = be._ctx()
        pv = cx.pinned.empty((n_rows, 2))
        for name, fn in [("result", lambda: cx.result(0)), ("trace", lambda: cx.trace(0, e2e_steps + 1)),
                         ("vertices(pinned)", lambda: cx.vertices(0, pv)), ("counts", lambda: cx.counts(0)),
                         ("region_error", lambda: cx.region_error(0)), ("collect", lambda: be._collect(cx, 0, 0, 0, pv))]:
            tq = time.perf_counter()
            for _ in range(10):
                fn()
            print(f"e2e-debug {name:18s} {1e2 * (time.perf_counter() - tq):8.3f} ms", file=sys.stderr)
    e2e_value = e2e_steps * args.batch * world / e2e_s
    # the map's vertex rows go up once per call (det_set_batch(xy=NULL) replicates them on the
    # device); statistics and target weights once per frame
    h2d = n_rows * 16 + len(m.regions) * 8 * 2 * args.batch
    # vertices, counts, per-region errors, trace and the result record; the label texture is
    # fetched lazily (only when a caller reads RunResult.state.labels), so it is not counted
    d2h = (n_rows * 16 + (len(m.regions) + 1) * 4 + len(m.regions) * 8 + (e2e_steps + 1) * 32 + 64) * args.batch

    # ---- the paper's own units (rank 0, after the timed regions): one cartogram's latency per
    # iteration (PAPER.md:318-327 quotes ms per iteration at 1024^2) and a cumulative chain
    # (config 2: 12 warm-started time steps x 100 iterations) in time steps per second ----
    extra = {}
    if rank == 0 and not args.no_extra:
        extra = paper_units(P, m, walk, args.field, local)

    # ---- final gather of per-frame results (the only collective) ----
    xi = torch.tensor([r.state.xi if not isinstance(r, Exception) else -1.0 for r in res], device="cuda",
                      dtype=torch.float64)
    if dist is not None:
        allxi = [torch.empty_like(xi) for _ in range(world)]
        dist.all_gather(allxi, xi)
        xi = torch.cat(allxi)

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            procs = 1
            cval, sample = cpu_measure(walk, 12, procs)
            cpu = {"value": cval, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64" if args.field == "float32" else "f64",
            "data": "synthetic",
            "config": {"workload": "headline: 3000-region Voronoi map (seed 3), %d unique vertices / %d rows, "
                                   "1024^2 texture, direct-mode time steps, %d frames per GPU, 1 step = 1 DET "
                                   "iteration of every frame" % (n_unique, n_rows, args.batch),
                       "frames_per_gpu": args.batch, "k": K_TEX, "field_storage": args.field,
                       "arithmetic": ("float32 field, vertex state and in-band sums; float64 raster crossings, "
                                      "band carries and control step" if args.field == "float32" else
                                      "float64 throughout (trajectory-identical to the reference)"),
                       "e2e_note": "median of 3 timed public-API calls (map upload, run, results back), "
                                   "gc.collect() before each; pinned result buffer reserved at BatchEngine "
                                   "construction",
                       "l2": "inputs larger than L2 (~%d MB working set per GPU vs 126 MB L2)"
                             % int(args.batch * (45 if args.field != "float32" else 35)), "iterations_per_time_step": prm["iterations"],
                       "time_steps_per_s": value / prm["iterations"]},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_achieved, "peak": peak, "unit": "GB/s",
                         "frac": dom_achieved / peak, "traffic": traffic_for(dom, args.batch),
                         "traffic_source": TRAFFIC_SRC, "peak_kind": peak_kind,
                         "phase_ms_per_iteration": per_iter_ms,
                         "step": {"algorithmic_bytes": step_bytes, "achieved": step_achieved,
                                  "frac": step_achieved / peak}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / e2e_steps,
                    "d2h_bytes_per_step": d2h / e2e_steps, "steps": e2e_steps,
                    "runs_it_per_s": [e2e_steps * args.batch * world / t for t in e2e_runs],
                    "host_split": getattr(be, "last_timing", {})},
            "gpu_launches": timed_launches(args.steps, args.groups, args.batch, kernels_per_iteration(args.field),
                                            2 if args.field == "float64" else 0),
            "iterations_executed": iters_total, "frames_active_after": int(act.sum()),
            "clocks": clk.summary(),
            "device": device_info(local),
            "final_gather": {"frames": int(xi.numel()), "xi_mean": float(xi.mean().item())},
            **extra,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
