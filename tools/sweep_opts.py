"""Time-to-solution sweep of solver options on a workload (GPU); prints iters / ms."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import workload  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
variants = json.loads(sys.argv[3])
w = workload(name, n, n)
eb, ep, rho = (torch.from_numpy(w[k]).cuda() for k in ("eta_b", "eta_p", "rho_b"))
for v in variants:
    s = Stokes(n, n, w["Lx"], w["Ly"], w["bc"], **v)
    s.set_viscosity(eb, ep)
    s.set_density(rho)
    s.set_gravity(w["gx"], w["gy"])
    r = s.solve(1e-8)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = s.solve(1e-8)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps({"workload": name, "n": n, "opts": v, "iters": r["iters"], "status": r["status"],
                      "E": r["E"], "ms": dt * 1e3}), flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
