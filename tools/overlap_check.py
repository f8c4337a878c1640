"""Diagnostics of the overlapped decomposed passes: k iterations of a 2x2 decomposition
against the single domain (relative difference of the fields), repeated.
usage: STOKES_DIST_OVERLAP=0|1|2 python tools/overlap_check.py N TRANSPORT K"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2603_14040_b200 import Stokes, StokesDist  # noqa: E402
from synth.fields import workload  # noqa: E402

n, tr, k = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
w = workload("layered", n, n)
T = lambda a: torch.from_numpy(a).cuda()


def mk(cls, **kw):
    s = cls(n, n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0, max_iter=k, **kw)
    s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    s.set_density(T(w["rho_b"]))
    s.set_gravity(w["gx"], w["gy"])
    return s


a = mk(Stokes).solve(0.0)
for rep in range(2):
    b = mk(StokesDist, px=2, py=2, transport=tr).solve(0.0)
    d = max(float((b[q] - a[q]).norm() / a[q].norm()) for q in ("vx", "vy", "p"))
    print(json.dumps({"n": n, "transport": tr, "k": k, "overlap": os.environ.get("STOKES_DIST_OVERLAP", "1"),
                      "rep": rep, "E1": a["E"], "E2": b["E"], "rel": d}), flush=True)
