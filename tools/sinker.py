"""E1 run-alike on one B200: sinking inclusion,
contrast 1e8, full density, 500 x 600 cells (501 x 601 nodes), free slip, sweep growth 2.5,
coarsest by smoothing, omega_v 0.3, omega_p 0.6, 1000 Uzawa iterations; with and without the
viscosity-rescaling stages (theta += 0.25 every 25 iterations) + lithostatic initial pressure.
Prints one JSON line per run: smoother, staging, E after 100 / 250 / 1000 iterations, time."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import workload  # noqa: E402

nx, ny = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (500, 600)
w = workload("sinker", nx, ny)
dev = {k: torch.from_numpy(w[k]).cuda() for k in ("eta_b", "eta_p", "rho_b")}
for smoother in (0, 1):
    for staged in (False, True):
        out = {"workload": f"sinker {nx}x{ny} cells", "smoother": ["jacobi", "rbgs"][smoother],
               "theta_stages+lithostatic": staged}
        for n_it in (100, 250, 1000):
            opts = dict(omega_v=0.3, alpha_p=0.6, nu_growth=2.5, coarse_direct=0, smoother=smoother, max_iter=n_it)
            if staged:
                opts.update(theta_step=0.25, theta_every=25)
            s = Stokes(nx, ny, 1.0, 1.0, w["bc"], **opts)
            s.set_viscosity(dev["eta_b"], dev["eta_p"])
            s.set_density(dev["rho_b"])
            s.set_gravity(w["gx"], w["gy"])
            p0 = s.lithostatic() if staged else None
            s.solve(0.0, p=p0)  # warm-up (graph capture)
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = s.solve(0.0, p=p0)
            torch.cuda.synchronize()
            out[f"E@{n_it}"] = r["E"]
            out[f"ms@{n_it}"] = (time.perf_counter() - t) * 1e3
        out["levels"] = [s.level_shape(l) for l in range(s.num_levels)]
        print(json.dumps(out), flush=True)
