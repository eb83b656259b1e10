"""N>1 path on CPU: world_size-2 gloo ranks each take their LPT shard of the
workload (bench.snake_shard, the same deal the bench uses under torchrun),
cover every task exactly once, balance the estimated cost, and agree on the
max-over-ranks timing reduction.  No data-path collective exists (units are
independent); the only collectives are the bench's barrier + MAX/SUM."""
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


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.002)
    cost = bench.task_cost(ds)
    mine = bench.snake_shard(cost, world, rank)
    # gather shards and costs
    sizes = [None] * world
    dist.all_gather_object(sizes, (mine.tolist(), int(cost[mine].sum())))
    t = torch.tensor([float(rank + 1), float(len(mine))], dtype=torch.float64)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put((sizes, float(mx[0]), float(sm[1]), ds.n_tasks, int(cost.sum())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_lpt_shards_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    sizes, tmax, total, n, cost_total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    idx = np.concatenate([np.array(s[0], dtype=np.int64) for s in sizes])
    assert len(idx) == n and len(np.unique(idx)) == n  # each task exactly once
    assert total == n and tmax == world               # SUM / MAX reductions
    costs = [s[1] for s in sizes]
    assert max(costs) / (cost_total / world) < 1.01    # LPT balance within 1%
