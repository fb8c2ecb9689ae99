"""N>1 path on CPU (gloo, world_size 2): bench.py shards C5 scenes by rank with no
data-path collective (scenes are independent problems); the only
collectives are the barrier and the max-over-ranks timer.  Checks that the union of
the rank shards, each solved independently, equals the single-process solve of the
same scenes bitwise, and that the shards are disjoint and cover the id range."""
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


def _worker(rank, world, port, per_rank, iters, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle

    sc = bench.make_scene(5, rank, per_rank)
    o = oracle.Oracle(sc)
    o.admm_iterate(iters)
    s = torch.from_numpy(o.s.copy())
    gathered = [torch.zeros_like(s) for _ in range(world)]
    dist.all_gather(gathered, s)
    ids = torch.tensor(list(range(rank * per_rank, (rank + 1) * per_rank)))
    all_ids = [torch.zeros_like(ids) for _ in range(world)]
    dist.all_gather(all_ids, ids)
    t = torch.tensor([10.0 * (rank + 1)])  # the bench's max-over-ranks timer
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        out.put((torch.cat(gathered).numpy(), torch.cat(all_ids).numpy(), float(t.item())))
    dist.destroy_process_group()


def test_scene_sharding_world2_gloo():
    import sys

    sys.path.insert(0, ROOT)
    import bench
    import oracle

    world, per_rank, iters = 2, 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    s_sharded, ids, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 20.0
    assert sorted(ids.tolist()) == list(range(world * per_rank))
    ref = bench.make_scene(5, 0, world * per_rank)
    o = oracle.Oracle(ref)
    o.admm_iterate(iters)
    assert np.array_equal(s_sharded, o.s)
