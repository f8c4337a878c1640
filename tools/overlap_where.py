"""Diagnostics: where do the overlapped decomposed passes differ from the single domain?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
b = mk(StokesDist, px=2, py=2, transport=tr).solve(0.0)
for q in ("vx", "vy", "p"):
    d = (b[q] - a[q]).abs().cpu().numpy()
    ref = a[q].abs().max().item()
    bad = np.argwhere(d > 1e-9 * ref)
    print(q, "n bad", len(bad), "max", d.max() / ref)
    if len(bad):
        rows = np.unique(bad[:, 0])
        cols = np.unique(bad[:, 1])
        print("  rows", rows[:20], "...", rows[-10:], len(rows))
        print("  cols", cols[:20], "...", cols[-10:], len(cols))
