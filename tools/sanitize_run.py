"""Small solves exercising every kernel (GCR, Anderson and viscosity stages also on decomposed
handles) (single domain Jacobi/RBGS/GCR/Anderson/RAS/Mixed
incl. the TMA streaming kernels, the one-pass RBGS (forced onto every streamed level), the
fused k_jju pass and the device-side loop graph, viscosity stages, lithostatic pressure,
decomposed virtual / loopback / NCCL_SELF with and without the overlapped split passes, the
marker-in-cell kernels) for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes, StokesDist  # noqa: E402
from synth.fields import markers, workload  # noqa: E402

os.environ["STOKES_DIST_DMIN"] = "8"
os.environ["STOKES_RBGS1"] = "2"  # the one-pass RBGS kernel on every streamed single-domain level
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(cls, n, name, **kw):
    w = workload(name, n, n)
    s = cls(n, n, w["Lx"], w["Ly"], w["bc"], **kw)
    s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    s.set_density(T(w["rho_b"]))
    s.set_gravity(w["gx"], w["gy"])
    r = s.solve(1e-6)
    print(cls.__name__, n, name, kw, r["iters"], r["status"], flush=True)


run(Stokes, 256, "layered", omega_v=0.6, alpha_p=1.0, max_iter=3)
run(Stokes, 256, "block", omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=4, max_iter=6)
run(Stokes, 64, "mms", omega_v=0.6, alpha_p=1.0, smoother=1, max_iter=3)
run(Stokes, 48, "mms", omega_v=0.6, alpha_p=1.0, accel=1, max_iter=4)
run(StokesDist, 512, "layered", px=2, py=2, transport="loopback", omega_v=0.6, alpha_p=1.0, max_iter=2)
run(StokesDist, 128, "layered", px=2, py=1, transport="virtual", omega_v=0.6, alpha_p=1.0, smoother=1, max_iter=2)
run(StokesDist, 256, "layered", px=2, py=2, transport="nccl_self", omega_v=0.6, alpha_p=1.0, max_iter=2)
os.environ["STOKES_DIST_OVERLAP"] = "1"
run(StokesDist, 512, "layered", px=2, py=1, transport="virtual", omega_v=0.6, alpha_p=1.0, max_iter=3)
os.environ.pop("STOKES_DIST_OVERLAP")
run(Stokes, 512, "layered", omega_v=0.6, alpha_p=1.0, smoother=1, max_iter=2)
run(StokesDist, 256, "block", px=2, py=2, transport="nccl_self", omega_v=0.6, alpha_p=1.0, accel=1, max_iter=4)
run(StokesDist, 256, "block", px=2, py=1, transport="loopback", omega_v=0.6, alpha_p=1.0, accel=2, aa_depth=5,
    aa_beta=0.7, max_iter=4)
run(StokesDist, 128, "block", px=2, py=1, transport="virtual", omega_v=0.6, alpha_p=1.0, theta_step=0.5,
    theta_every=2, max_iter=6)
os.environ["STOKES_HALO_2PHASE"] = "1"  # the two-round exchange of the packed transports
run(StokesDist, 256, "layered", px=2, py=2, transport="loopback", omega_v=0.6, alpha_p=1.0, max_iter=2)
os.environ.pop("STOKES_HALO_2PHASE")
os.environ.pop("STOKES_DIST_DMIN")
for r in range(4):  # every rank of a 2 x 2 NCCL grid as a schedule-recording dry run (one round, overlap on)
    from paper_2603_14040_b200.decomp import tile_windows
    win = tile_windows(2048, 2048, 2, 2, r)
    i0, j0 = win["b"][0].start, win["b"][1].start
    w = workload("layered", 2048, 2048, win_b=(i0, j0, 1025, 1025), win_p=(i0, j0, 1024, 1024))
    d = StokesDist(2048, 2048, w["Lx"], w["Ly"], w["bc"], px=2, py=2, rank=r, transport="nccl_dry", omega_v=0.6,
                   alpha_p=1.0, max_iter=2)
    d.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    d.set_density(T(w["rho_b"]))
    d.set_gravity(w["gx"], w["gy"])
    print("dry rank", r, d.solve(0.0)["iters"], len(d.schedule()), flush=True)
    d.close()
os.environ["STOKES_DIST_DMIN"] = "8"
s = Stokes(256, 256, omega_v=0.6)
w = workload("layered", 256, 256)
s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
s.set_density(T(w["rho_b"]))
s.set_gravity(0, 1)
for k in Stokes.KERNELS:
    s.time_kernel(k, 1)
run(Stokes, 256, "layered", omega_v=0.6, alpha_p=1.0, accel=2, aa_depth=5, aa_beta=0.7, max_iter=4)
run(Stokes, 256, "layered", omega_v=0.6, alpha_p=1.0, smoother=3, max_iter=2)
run(Stokes, 128, "block", omega_v=0.6, alpha_p=1.0, smoother=2, accel=1, max_iter=3)
run(Stokes, 128, "sinker", omega_v=0.3, alpha_p=0.6, theta_step=0.5, theta_every=2, max_iter=6)
s.lithostatic()
m = markers(200, 130, 1.0, 1.0, per_side=3, seed=1, order="shuffled", props="sinker")
q = Stokes(200, 130, 1.0, 1.0)
xm, ym = T(m["xm"]), T(m["ym"])
eb, ep, rb, ne = q.markers_to_grid(xm, ym, T(m["eta_m"]), T(m["rho_m"]))
vx = torch.randn(130, 201, dtype=torch.float64, device="cuda")
vy = torch.randn(131, 200, dtype=torch.float64, device="cuda")
q.grid_to_markers(xm, ym, vx, vy)
dt = q.marker_timestep(vx, vy, 0.5, 1.0)
for sch in Stokes.ADVECT:
    q.advect_markers(xm, ym, vx, vy, dt, sch)
torch.cuda.synchronize()
print("done", ne)
