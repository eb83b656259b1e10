"""N>1 path on CPU: world_size 2 and 3 gloo ranks shard the config-5
workload with the engine's own partitioner (xb_shard_tasks, the C-ABI the
bench calls under torchrun and xb_extend_batch uses across devices), in both
modes: LPT on estimated cost, and locality-aware (a breadth-first sweep of the
sequence graph cut into equal-cost runs).  Every rank computes the same
assignment independently; together the shards cover every task exactly once,
balance the estimated cost, and (locality) each references about 1/N of the
pool -- what a rank's GPU then uploads.  No data-path collective exists
(units are independent); the only collectives are the bench's barrier and its
MAX / SUM reductions of time and cells."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, locality, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2304_08662_b200 as xb
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.005)
    pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x), ds.symbols, ds.offsets)
    shard_of = xb.xband.shard_tasks(pool, ds.tasks, ds.k, world, locality=locality)
    mine = np.nonzero(shard_of == rank)[0]
    cost = bench.task_cost(ds)
    ln = np.diff(ds.offsets)
    refs = np.unique(np.concatenate([ds.tasks[mine, 0], ds.tasks[mine, 1]]))
    every = [None] * world
    dist.all_gather_object(every, (shard_of.tobytes(), mine.tolist(), int(cost[mine].sum()),
                                   float(ln[refs].sum() / ln.sum())))
    t = torch.tensor([float(rank + 1), float(len(mine))], dtype=torch.float64)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((every, float(mx[0]), float(sm[1]), ds.n_tasks, int(cost.sum())))
    dist.destroy_process_group()


@pytest.mark.parametrize("locality", [False, True], ids=["lpt", "locality"])
@pytest.mark.parametrize("world", [2, 3])
def test_engine_shards_gloo(world, locality):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, locality, q)) for r in range(world)]
    for p in procs:
        p.start()
    every, tmax, total, n, cost_total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len({e[0] for e in every}) == 1                  # every rank computed the same assignment
    idx = np.concatenate([np.array(e[1], dtype=np.int64) for e in every])
    assert len(idx) == n and len(np.unique(idx)) == n       # each task exactly once
    assert total == n and tmax == world                      # SUM / MAX reductions
    costs = [e[2] for e in every]
    assert max(costs) / (cost_total / world) < 1.01          # balanced within 1%
    fracs = [e[3] for e in every]
    if locality:  # a shard references about 1/world of the pool (+ boundary reads)
        assert max(fracs) < 1.25 / world, fracs
    else:
        assert min(fracs) > 0.8, fracs
