"""Host-side logic of the multi-GPU path on CPU: world_size-2 gloo process groups run the
rank -> tile plan, generate their tile windows of the weak-scaling workload and exchange
them; the assembled tiles must reproduce the global arrays and agree on shared interface
nodes.  The NCCL unique id of the decomposed handle is broadcast through the same group."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_14040_b200.decomp import process_grid, tile_of, tile_windows, weak_problem


def test_process_grid_and_tiles():
    assert [process_grid(n) for n in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]
    assert tile_of(5, 4, 2) == (1, 1)
    w = tile_windows(8, 4, 2, 2, 3)
    assert w["vx"] == (slice(2, 4), slice(4, 9)) and w["b"] == (slice(2, 5), slice(4, 9))
    assert weak_problem(8, 64) == (256, 128, 4.0, 2.0, 4, 2)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth.fields import workload
        nx, ny, Lx, Ly, px, py = weak_problem(world, 32)
        win = tile_windows(nx, ny, px, py, rank)
        i0, j0 = win["b"][0].start, win["b"][1].start
        nyt, nxt = ny // py, nx // px
        tw = workload("layered", nx, ny, Lx, Ly, win_b=(i0, j0, nyt + 1, nxt + 1), win_p=(i0, j0, nyt, nxt))
        mine = {k: torch.from_numpy(tw[k]) for k in ("eta_b", "eta_p", "rho_b")}
        gathered = {}
        for k, t in mine.items():
            lst = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(lst, t)
            gathered[k] = [x.numpy() for x in lst]
        # NCCL id broadcast (plumbing of StokesDist)
        from paper_2603_14040_b200 import nccl_unique_id
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if rank == 0:
            q.put((gathered, len(obj[0])))
        else:
            q.put(len(obj[0]))
    finally:
        dist.destroy_process_group()


def test_two_rank_tiles_reassemble_the_global_workload():
    from synth.fields import workload
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered, idlen = next(r for r in res if isinstance(r, tuple))
    assert idlen == 128 and all(r == 128 for r in res if not isinstance(r, tuple))
    nx, ny, Lx, Ly, px, py = weak_problem(world, 32)
    g = workload("layered", nx, ny, Lx, Ly)
    for k, kind in (("eta_b", "b"), ("eta_p", "p"), ("rho_b", "b")):
        for r in range(world):
            rows, cols = tile_windows(nx, ny, px, py, r)[kind]
            assert np.array_equal(gathered[k][r], g[k][rows, cols]), (k, r)
    # interface column shared by the two tiles carries the same values
    assert np.array_equal(gathered["eta_b"][0][:, -1], gathered["eta_b"][1][:, 0])
