"""Small solves exercising every kernel (single domain Jacobi/RBGS/GCR incl. the TMA
streaming kernels, decomposed virtual + loopback) for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes, StokesDist  # noqa: E402
from synth.fields import workload  # noqa: E402

os.environ["STOKES_DIST_DMIN"] = "8"
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
s = Stokes(256, 256, omega_v=0.6)
w = workload("layered", 256, 256)
s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
s.set_density(T(w["rho_b"]))
s.set_gravity(0, 1)
for k in Stokes.KERNELS:
    s.time_kernel(k, 1)
print("done")
