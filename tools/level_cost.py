"""Per-level cost inside the graph-replayed Uzawa iteration: time 30 iterations of layered
4096^2 with the hierarchy truncated at coarse_min (coarsest solved by 2nu smoothing sweeps,
coarse_direct=0) -- differences between truncations = real cost of the dropped levels."""
import json, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes
from synth.fields import workload
n = 4096
w = workload("layered", n, n)
eb, ep, rb = (torch.from_numpy(w[k]).cuda() for k in ("eta_b", "eta_p", "rho_b"))
out = []
for cm in (8, 16, 32, 64, 128, 256, 512, 1024):
    for direct in ((1, 0) if cm == 8 else (0,)):
        s = Stokes(n, n, 1.0, 1.0, omega_v=0.6, alpha_p=1.0, coarse_min=cm, coarse_direct=direct, max_iter=30)
        s.set_viscosity(eb, ep); s.set_density(rb); s.set_gravity(0.0, 1.0)
        s.solve(1e-30)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s.stream)
        r = s.solve(1e-30)
        b.record(s.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        out.append({"coarse_min": cm, "direct": direct, "levels": s.num_levels, "iters": r["iters"], "ms_per_iter": ms / r["iters"]})
        print(json.dumps(out[-1]), flush=True)
        del s
