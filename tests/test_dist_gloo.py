"""world_size-2 gloo tests of the multi-process path: shard frames, compute per rank, final gather.

Runs on CPU.  The product's sharding entry point (``shard.run_sharded``, used by
``run_direct`` / ``sweep_bdv`` / ``BatchEngine`` with ``distributed=True`` or ``devices=[...]``)
drives a block task; here the task runs the oracle engine (the checker) on its block of a tiny
direct-mode job, since there is no GPU.  The gathered results must equal a single-process run.
"""

import functools
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


def _block(n_frames, lo, hi, device):
    m, walk = _job(n_frames)
    return [(t, device) + _frame(m, walk[t]) for t in range(lo, hi)]


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
    # the product's entry point: every rank gets every unit's result, in unit order
    from paper_2604_13880_b200.shard import run_sharded

    objs = run_sharded(n_frames, functools.partial(_block, n_frames), distributed=True)
    out["objs"] = objs
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
    assert [o[0] for o in out["objs"]] == list(range(n_frames))
    assert [o[1] for o in out["objs"]] == [0] * n_frames  # LOCAL_RANK unset: device 0 on every rank
    for t in range(n_frames):
        r, x = _frame(m, walk[t])
        np.testing.assert_array_equal(out["rows"][t], r)
        assert out["xi"][t] == x
        np.testing.assert_array_equal(out["objs"][t][2], r)
        assert out["objs"][t][3] == x


def test_run_sharded_worker_processes():
    # devices=[...]: one spawned worker process per device id, blocks gathered in unit order
    from paper_2604_13880_b200.shard import run_sharded, shutdown_workers

    n_frames = 5
    try:
        objs = run_sharded(n_frames, functools.partial(_block_mod, n_frames), devices=[3, 7])
    finally:
        shutdown_workers()
    assert [o[0] for o in objs] == list(range(n_frames))
    assert [o[1] for o in objs] == [3, 3, 3, 7, 7]
    m, walk = _job(n_frames)
    for t in range(n_frames):
        r, x = _frame(m, walk[t])
        np.testing.assert_array_equal(objs[t][2], r)


def _block_mod(n_frames, lo, hi, device):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    return _block(n_frames, lo, hi, device)
