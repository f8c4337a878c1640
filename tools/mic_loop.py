"""The paper's marker-in-cell simulation loop (Fig. mic-loop-diagram) on one
B200, every phase through the C ABI: (1) markers -> grid (eta_b, eta_p, rho_b), (2) Stokes solve
to E <= rtol warm-started from the previous step's velocity and pressure, (3) CFL time step,
(4) RK4 advection.  Markers are generated on the GPU (tools/mic_bench.py recipe, layered
lithosphere/mantle properties of BASELINE cfg 4 carried by the markers).  Prints one JSON line
per step with the phase times (CUDA events on the handle's stream) and the iteration count.
usage: python tools/mic_loop.py [--n 1024] [--steps 4] [--per-side 4] [--scheme rk4]
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import markers_torch  # noqa: E402


def gen_markers(nx, ny, per_side, seed, order="cell"):
    """synth.fields.markers_torch (the markers() recipe built on the GPU), optionally shuffled."""
    xm, ym, eta, rho = markers_torch(nx, ny, per_side=per_side, seed=seed, props="layered")
    if order == "shuffled":
        g = torch.Generator(device="cuda").manual_seed(seed + 1)
        p = torch.randperm(xm.numel(), generator=g, device="cuda")
        xm, ym, eta, rho = (t[p].contiguous() for t in (xm, ym, eta, rho))
    return xm, ym, eta, rho


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--per-side", type=int, default=4)
    ap.add_argument("--scheme", default="rk4")
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--cfl", type=float, default=0.5)
    args = ap.parse_args()
    n = args.n
    s = Stokes(n, n, 1.0, 1.0, omega_v=0.6, alpha_p=1.0)
    s.set_gravity(0.0, 1.0)
    xm, ym, eta, rho = gen_markers(n, n, args.per_side, 2603)
    st = s.stream
    ev = lambda: torch.cuda.Event(enable_timing=True)
    vx = vy = p = None
    for k in range(args.steps):
        e = [ev() for _ in range(5)]
        torch.cuda.synchronize()
        e[0].record(st)
        eb, ep, rb, ne = s.markers_to_grid(xm, ym, eta, rho, count_empty=False)
        e[1].record(st)
        s.set_viscosity(eb, ep)
        s.set_density(rb)
        r = s.solve(args.rtol, vx, vy, p)
        e[2].record(st)
        dt = s.marker_timestep(r["vx"], r["vy"], args.cfl, 1e9)
        e[3].record(st)
        s.advect_markers(xm, ym, r["vx"], r["vy"], dt, args.scheme, count_clamped=False)
        e[4].record(st)
        torch.cuda.synchronize()
        vx, vy, p = r["vx"], r["vy"], r["p"]
        print(json.dumps({"step": k, "n": n, "markers": xm.numel(), "iters": r["iters"], "E": r["E"], "dt": dt,
                          "ms": {"markers_to_grid": e[0].elapsed_time(e[1]), "setup+solve": e[1].elapsed_time(e[2]),
                                 "timestep": e[2].elapsed_time(e[3]), "advect": e[3].elapsed_time(e[4])}}),
              flush=True)


if __name__ == "__main__":
    main()
