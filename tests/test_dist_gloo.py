"""world_size-2 gloo test of the multi-process path: shard frames, compute per rank, final gather.

Runs on CPU.  Each rank runs the oracle engine (the checker) on its shard of a
tiny direct-mode job; the gathered results must equal a single-process run.
This covers the host-side logic the GPU bench uses (shard_bounds +
gather_frame_results), which is identical regardless of the compute backend.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _job(n_frames):
    import fixture_maps as fm

    m = fm.small_voronoi(seed=4, r=8, target=150, shuffle_ids=False)
    walk = np.stack([m.statistics() * (1 + 0.1 * t) ** np.arange(8) for t in range(n_frames)])
    return m, walk


def _frame(m, stats):
    from oracle import det_oracle as O

    eng = O.OracleEngine(O.FlatMap.from_mapmodel(m.with_statistics(stats)), k=5)
    r = eng.run(error_threshold=1e-300, stagnation_window=10**9, max_iterations=4)
    return r.rows, r.xi


def _worker(rank, world, port, n_frames, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    import torch.distributed as dist

    from paper_2604_13880_b200.shard import gather_frame_results, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, walk = _job(n_frames)
    lo, hi = shard_bounds(n_frames, rank, world)
    rows, xi = [], []
    for t in range(lo, hi):
        r, x = _frame(m, walk[t])
        rows.append(r)
        xi.append(x)
    out = gather_frame_results({"rows": np.stack(rows), "xi": np.array(xi)}, dist)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather():
    n_frames = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m, walk = _job(n_frames)
    for t in range(n_frames):
        r, x = _frame(m, walk[t])
        np.testing.assert_array_equal(out["rows"][t], r)
        assert out["xi"][t] == x
