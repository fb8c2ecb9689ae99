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


def _worker_obs(rank, world, port, out):
    """Obstacle sharding: each rank solves the pair QPs of its obstacle block; the
    per-timestep partial sums are all-reduced (the a5 exchange of SURVEY §8(a))."""
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2406_07048_b200 as ca
    import scenes
    from parity_util import pair_geometry

    sc = scenes.make_config(2)
    j0, j1 = ca.obstacle_partition(sc, world, rank)
    part = torch.zeros(sc.horizon, dtype=torch.float64)
    M = sc.n_obs
    for p in range(sc.n_pairs):
        if not (j0 <= p % M < j1):
            continue
        b, t, A, bb, Cm, dv = pair_geometry(sc, p)
        R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, sc.s_ref[b, t])
        y, st, piv, _ = oracle.pair_solve(A, bb, Cm, dv, R, rho, 0.0, np.zeros(2))
        K, bvec, *_ = oracle.pair_lcp(A, bb, Cm, dv, R, rho, 0.0, np.zeros(2))
        u = K.T @ y + bvec
        part[t - 1] += 0.5 * float(u @ u)
    dist.all_reduce(part)
    if rank == 0:
        out.put(part.numpy())
    dist.destroy_process_group()


def test_obstacle_sharding_world2_gloo():
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import scenes
    from parity_util import pair_geometry

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_obs, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = scenes.make_config(2)
    ref = np.zeros(sc.horizon)
    for p in range(sc.n_pairs):
        b, t, A, bb, Cm, dv = pair_geometry(sc, p)
        R, rho = oracle.pose(sc.pose_model, sc.pose_idx, sc.dim, sc.s_ref[b, t])
        y, st, piv, _ = oracle.pair_solve(A, bb, Cm, dv, R, rho, 0.0, np.zeros(2))
        K, bvec, *_ = oracle.pair_lcp(A, bb, Cm, dv, R, rho, 0.0, np.zeros(2))
        u = K.T @ y + bvec
        ref[t - 1] += 0.5 * float(u @ u)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)


def _worker_grid(rank, world, port, n_scenes, eps, kmax, out):
    """Scene grid (include/ca.h ca_dist_desc, scene_shards = world): rank keeps its scene
    block; per ADMM iteration its scenes' Eq. 18 statistics go into a global table (zero
    elsewhere) that ONE all_reduce makes identical on every rank; every rank then takes
    the same per-scene stop decisions and the same global 'scenes still running' count,
    so all ranks run the same number of collectives (no rank can hang)."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import scenes
    from paper_2406_07048_b200._ca import grid_position

    full = scenes.make_c5(scene_ids=range(n_scenes))
    b0, b1 = grid_position(n_scenes, world, rank, world, 1)["scenes"]
    mine = {b: oracle.Oracle(full.subset([b])) for b in range(b0, b1)}
    active = np.ones(n_scenes, bool)
    iters = np.zeros(n_scenes, np.int64)
    loops = 0
    for k in range(kmax):
        table = torch.zeros(n_scenes, 2, dtype=torch.float64)
        for b, o in mine.items():
            if not active[b]:
                continue
            rd, _ = o.dual_sweep()
            o.primal_step()
            rp = o.multiplier_update()
            table[b, 0], table[b, 1] = float(rp[0]), float(rd[0])
        dist.all_reduce(table)  # the per-iteration exchange
        loops += 1
        for b in range(n_scenes):
            if active[b]:
                iters[b] = k + 1
                if table[b, 0] <= eps and table[b, 1] <= eps:
                    active[b] = False
        if not active.any():
            break
    s = torch.zeros(n_scenes, full.horizon + 1, full.n_state, dtype=torch.float64)
    for b, o in mine.items():
        s[b] = torch.from_numpy(o.s[0])
    dist.all_reduce(s)
    cnt = torch.tensor([loops])
    allc = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(allc, cnt)
    if rank == 0:
        out.put((s.numpy(), iters, [int(c) for c in allc]))
    dist.destroy_process_group()


def test_scene_grid_world2_gloo():
    """The library's scene-sharded protocol on two gloo ranks: the union of the shards
    equals the single-process ca_admm_solve semantics (orc_admm_solve per scene, Eq. 18)
    bitwise, and both ranks ran the same number of collective rounds."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import scenes

    world, n, eps, kmax = 2, 3, 3.0, 25
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_grid, args=(r, world, port, n, eps, kmax, q)) for r in range(world)]
    for p in procs:
        p.start()
    s, iters, loops = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert loops[0] == loops[1] == iters.max()
    ref = oracle.Oracle(scenes.make_c5(scene_ids=range(n)))
    it, cv, _, _, _ = ref.admm_solve(eps, eps, kmax)
    assert np.array_equal(it, iters)
    assert np.array_equal(s, ref.s)
