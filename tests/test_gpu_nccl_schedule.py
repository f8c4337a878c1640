"""The multi-process NCCL transport's schedule,
checked on ONE B200 without running NCCL across GPUs.

Every rank of a px x py process grid is created in this process as a dry-run handle
(stokes_create_dist with rank r and no NCCL unique id: each NCCL call the transport would
issue is recorded, not issued), one rank after another -- no kernel ever waits on another
rank -- and makes the bench's calls (set_viscosity / set_density / set_gravity on its tile
window, a solve: the eager first iteration and the CUDA graphs of the following ones, which
record their calls when captured).  The recorded schedules must satisfy NCCL's matching rules:
  * every rank issues the same sequence of steps (a grouped point-to-point round, or a
    collective), with no collective inside a group;
  * at every collective step all ranks agree on kind, element count, datatype and reduction;
  * at every point-to-point step the sends r -> q match the receives at q from r one to one,
    in issue order, with equal counts (NCCL pairs the p2p operations between two ranks in
    issue order);
  * the peers are the tile's grid neighbours, sides or diagonals (never the rank itself).
Covers the bench's weak (BASELINE cfg 4: 4096^2 per GPU) and strong (cfg 5: 16384^2 split)
launch configurations at N = 2, 4, 8, and GCR / Anderson / viscosity stages on small tiles.
The data moved is verified elsewhere: the LOOPBACK / NCCL_SELF transports run the same
packing with device copies / real NCCL calls on one GPU (tests/test_gpu_dist.py)."""
import json
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2603_14040_b200.decomp import strong_problem, tile_windows, weak_problem  # noqa: E402
from synth.fields import random_torch, workload  # noqa: E402

from nccl_schedule_check import check_schedules  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def rank_schedule(name, NX, NY, Lx, Ly, px, py, r, device_inputs, **opts):
    from paper_2603_14040_b200 import StokesDist
    win = tile_windows(NX, NY, px, py, r)
    i0, j0 = win["b"][0].start, win["b"][1].start
    nxt, nyt = NX // px, NY // py
    wb, wp = (i0, j0, nyt + 1, nxt + 1), (i0, j0, nyt, nxt)
    if device_inputs:
        w = random_torch(NX, NY, Lx, Ly, win_b=wb, win_p=wp, device="cuda")
    else:
        w = workload(name, NX, NY, Lx, Ly, win_b=wb, win_p=wp)
        w = dict(w, **{k: torch.from_numpy(np.ascontiguousarray(w[k])).cuda() for k in ("eta_b", "eta_p", "rho_b")})
    s = StokesDist(NX, NY, Lx, Ly, w["bc"], px=px, py=py, rank=r, transport="nccl_dry", **opts)
    s.set_viscosity(w["eta_b"], w["eta_p"])
    s.set_density(w["rho_b"])
    s.set_gravity(w["gx"], w["gy"])
    del w
    r_ = s.solve(0.0)
    assert r_["iters"] >= 1
    log = s.schedule()
    s.close()
    torch.cuda.empty_cache()
    return log


def run(label, name, problem, device_inputs=False, **opts):
    NX, NY, Lx, Ly, px, py = problem
    logs = [rank_schedule(name, NX, NY, Lx, Ly, px, py, r, device_inputs, **opts) for r in range(px * py)]
    summary = check_schedules(logs, px, py)
    print(json.dumps({"config": label, "grid": [NX, NY], "px": px, "py": py, **summary}))
    return summary


@pytest.mark.parametrize("n", [2, 4, 8])
def test_weak_scaling_schedule(n):
    """bench.py --gpus n (weak, cfg 4): 4096^2 layered tile per rank, plain Uzawa-MG, overlap on."""
    s = run(f"weak cfg4 N={n}", "layered", weak_problem(n, 4096), omega_v=0.6, alpha_p=1.0, max_iter=1)
    assert s["p2p_rounds"] > 0 and s["collectives"] > 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_strong_scaling_schedule(n):
    """bench.py strong block at n GPUs (cfg 5): 16384^2 random, split px x py, device inputs."""
    run(f"strong cfg5 N={n}", "random", strong_problem(n, 16384), device_inputs=True, omega_v=0.6, alpha_p=1.0,
        max_iter=1)


@pytest.mark.parametrize("accel,extra", [(1, dict(gcr_restart=10)), (2, dict(aa_depth=5, aa_beta=1.0)),
                                         (0, dict(theta_step=0.5, theta_every=1))])
def test_accelerated_and_staged_schedules(accel, extra):
    """GCR(m), Anderson and the viscosity-rescaling stages on a 2 x 2 grid of 1024^2 tiles."""
    run(f"accel={accel} {extra}", "layered", weak_problem(4, 1024), omega_v=0.6, alpha_p=1.0, accel=accel,
        max_iter=2, **extra)
