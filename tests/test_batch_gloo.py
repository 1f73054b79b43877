"""CPU, world_size 2 over gloo: the multi-GPU path's host logic (planet
partitioning + the final stats gather).  The per-planet engine here is the C
oracle standing in for the GPU (this is a test of the sharding plumbing)."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2407_02215_b200 import batch


def test_round_robin_partition():
    assert batch.planets_of_rank(8, 1, 0) == list(range(8))
    assert batch.planets_of_rank(8, 2, 1) == [1, 3, 5, 7]
    assert batch.planets_of_rank(8, 8, 5) == [5]
    assert batch.planets_of_rank(3, 4, 3) == []
    owned = [batch.planets_of_rank(8, 4, r) for r in range(4)]
    assert sorted(p for o in owned for p in o) == list(range(8))


def _planet_stats(p, frames):
    """Deterministic per-planet stats: a tiny oracle run, planet p rotated."""
    from oracle import OraclePool, OracleVerdict
    from paper_2407_02215_b200 import halfedge, lod, workloads
    mesh = halfedge.cube_sphere(workloads.EARTH_RADIUS)
    keys = lod.make_zoom_path(workloads.EARTH_RADIUS, 3 * workloads.EARTH_RADIUS, 1.0e5)
    cams = [lod.rotate_z(c, 45.0 * p) for c in lod.sample_path(keys, frames)]
    cfg = workloads.planet_config()
    op = OraclePool(mesh, 12)
    rows = []
    for cam in cams:
        s, _ = op.update(OracleVerdict.lod(mesh, lod.pack_lod_params(cfg, cam)))
        rows.append([int(x) for x in s] + [0] * 24)
    return rows


def _worker(rank, world, port, n_planets, frames, queue):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    owned = batch.planets_of_rank(n_planets, world, rank)
    local = np.array([_planet_stats(p, frames) for p in owned], dtype=np.int64).reshape(len(owned), frames, 32)
    full = batch.gather_stats(local, owned, n_planets, world)
    dist.barrier()
    if rank == 0:
        queue.put(full)
    dist.destroy_process_group()


def test_two_ranks_gather_equals_single_process():
    n_planets, frames = 5, 6
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_planets, frames, queue)) for r in range(2)]
    for p in procs:
        p.start()
    full = queue.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = np.array([_planet_stats(p, frames) for p in range(n_planets)], dtype=np.int64)
    assert full.shape == (n_planets, frames, 32)
    assert np.array_equal(full, single)
    # rotated planets really are different workloads
    assert not np.array_equal(single[0], single[1])
