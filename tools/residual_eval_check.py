"""Converged-solution residual evaluated by the GPU and by the oracle (diagnosis of the E
difference at large sizes): per size, the GPU solves `random` to rtol; both sides evaluate
r = f - L v - G p and E of that solution; prints E_gpu, E_oracle and where the residual
arrays differ (interior vs the two rows / columns next to a wall)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import random_torch, workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "random"
for n in [int(a) for a in (sys.argv[2:] or ["512", "1024", "2048", "4096"])]:
    if name == "random":
        w = random_torch(n, n, device="cuda")
        host = {k: w[k].cpu().numpy() for k in ("eta_b", "eta_p", "rho_b")}
    else:
        wn = workload(name, n, n)
        host = {k: wn[k] for k in ("eta_b", "eta_p", "rho_b")}
        w = dict(wn, **{k: torch.from_numpy(v).cuda() for k, v in host.items()})
    s = Stokes(n, n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0)
    s.set_viscosity(w["eta_b"], w["eta_p"])
    s.set_density(w["rho_b"])
    s.set_gravity(w["gx"], w["gy"])
    r = s.solve(1e-8)
    gx, gy, gp, eg = s.residual(r["vx"], r["vy"], r["p"])
    sol = {k: r[k].cpu().numpy() for k in ("vx", "vy", "p")}
    o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0)
    o.set_gravity(w["gx"], w["gy"])
    o.set_viscosity(host["eta_b"], host["eta_p"])
    o.set_density(host["rho_b"])
    ox, oy, op, eo = o.residual(sol["vx"], sol["vy"], sol["p"])
    out = {"workload": name, "n": n, "iters": r["iters"], "E_solve": r["E"], "E_gpu": eg, "E_oracle": eo}
    for k, g, e in (("rx", gx, ox), ("ry", gy, oy), ("rp", gp, op)):
        g = g.cpu().numpy()
        d = np.abs(g - e)
        out[k] = {"norm": float(np.linalg.norm(e)), "diff": float(np.linalg.norm(d)),
                  "diff_edge2": float(np.sqrt((d[:2] ** 2).sum() + (d[-2:] ** 2).sum() + (d[:, :2] ** 2).sum() + (d[:, -2:] ** 2).sum())),
                  "argmax": [int(x) for x in np.unravel_index(np.argmax(d), d.shape)], "shape": list(d.shape)}
    print(json.dumps(out), flush=True)
    s.close()
    del s, o, w, r
    torch.cuda.empty_cache()
