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

from paper_2603_14040_b200.decomp import process_grid, strong_problem, tile_of, tile_windows, weak_problem


def test_process_grid_and_tiles():
    assert [process_grid(n) for n in (1, 2, 4, 8)] == [(1, 1), (2, 1), (2, 2), (4, 2)]
    assert tile_of(5, 4, 2) == (1, 1)
    w = tile_windows(8, 4, 2, 2, 3)
    assert w["vx"] == (slice(2, 4), slice(4, 9)) and w["b"] == (slice(2, 5), slice(4, 9))
    assert weak_problem(8, 64) == (256, 128, 4.0, 2.0, 4, 2)
    assert strong_problem(8, 16384) == (16384, 16384, 1.0, 1.0, 4, 2)
    assert strong_problem(1, 16384) == (16384, 16384, 1.0, 1.0, 1, 1)


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


def _strong_worker(rank, world, port, q):
    """bench.py --scaling strong's host plan: the fixed global random problem, this rank's tile
    window sampled with the device generator (here on the CPU) and with numpy."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from synth.fields import random_torch, workload
        nx, ny, Lx, Ly, px, py = strong_problem(world, 64)
        win = tile_windows(nx, ny, px, py, rank)
        i0, j0 = win["b"][0].start, win["b"][1].start
        nyt, nxt = ny // py, nx // px
        wb, wp = (i0, j0, nyt + 1, nxt + 1), (i0, j0, nyt, nxt)
        tw = random_torch(nx, ny, Lx, Ly, win_b=wb, win_p=wp, device="cpu")
        nw = workload("random", nx, ny, Lx, Ly, win_b=wb, win_p=wp)
        dev = max(float(np.abs(tw[k].numpy() - nw[k]).max() / np.abs(nw[k]).max()) for k in ("eta_b", "eta_p", "rho_b"))
        gathered = {}
        for k in ("eta_b", "eta_p", "rho_b"):
            lst = [torch.zeros_like(tw[k]) for _ in range(world)]
            dist.all_gather(lst, tw[k])
            gathered[k] = [x.numpy() for x in lst]
        q.put((rank, dev, gathered if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_two_rank_strong_scaling_plan():
    from synth.fields import workload
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] <= 1e-13 for r in res), res
    gathered = next(r[2] for r in res if r[0] == 0)
    nx, ny, Lx, Ly, px, py = strong_problem(world, 64)
    g = workload("random", nx, ny, Lx, Ly)
    for k, kind in (("eta_b", "b"), ("eta_p", "p"), ("rho_b", "b")):
        for r in range(world):
            rows, cols = tile_windows(nx, ny, px, py, r)[kind]
            assert np.allclose(gathered[k][r], g[k][rows, cols], rtol=1e-13, atol=0), (k, r)
