"""Marker-in-cell kernels at full size on one B200.

Markers are generated ON THE GPU (torch, seeded): per_side^2 per cell on a jittered lattice in
cell order (the paper's 8-16 per cell), sinker properties; velocity = a seeded
smooth divergence-free field sampled at the velocity nodes.  Times with CUDA events on the
handle's stream (the binding's default stream) after warm-up:
  markers_to_grid (eta_b, eta_p, rho_b), grid_to_markers, advect (euler/heun/rk4), timestep.
Algorithmic bytes (8 B per double): m2g reads x, y, eta, rho once (32 B/marker) and writes
eta_b, rho_b, eta_p (24 B/cell); advect reads and writes x, y (32 B/marker) + reads vx, vy
(16 B/cell); g2m reads x, y, writes u, v (32 B/marker) + 16 B/cell.
usage: python tools/mic_bench.py [--n 4096] [--per-side 4] [--reps 5] [--order cell|shuffled]
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
    xm, ym, eta, rho = markers_torch(nx, ny, per_side=per_side, seed=seed, props="sinker")
    if order == "shuffled":
        g = torch.Generator(device="cuda").manual_seed(seed + 1)
        p = torch.randperm(xm.numel(), generator=g, device="cuda")
        xm, ym, eta, rho = (t[p].contiguous() for t in (xm, ym, eta, rho))
    return xm, ym, eta, rho


def velocity(nx, ny):
    """stream function psi = sin(pi x) sin(pi y) / pi: vx = dpsi/dy, vy = -dpsi/dx (free slip)"""
    dx, dy = 1.0 / nx, 1.0 / ny
    xv = torch.arange(nx + 1, device="cuda", dtype=torch.float64) * dx
    yv = (torch.arange(ny, device="cuda", dtype=torch.float64) + 0.5) * dy
    vx = torch.sin(math.pi * xv)[None, :] * torch.cos(math.pi * yv)[:, None]
    xw = (torch.arange(nx, device="cuda", dtype=torch.float64) + 0.5) * dx
    yw = torch.arange(ny + 1, device="cuda", dtype=torch.float64) * dy
    vy = -torch.cos(math.pi * xw)[None, :] * torch.sin(math.pi * yw)[:, None]
    return vx.contiguous(), vy.contiguous()


def timed(fn, reps, stream):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--per-side", type=int, default=4)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--order", default="cell")
    args = ap.parse_args()
    nx = ny = args.n
    peak = 6549.1
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", peak)
    except Exception:
        pass
    s = Stokes(nx, ny, 1.0, 1.0)
    xm, ym, eta, rho = gen_markers(nx, ny, args.per_side, 2603, args.order)
    vx, vy = velocity(nx, ny)
    n = xm.numel()
    cells = nx * ny
    st = s.stream  # the handle's stream: the kernels run there
    out = {"workload": f"{nx}x{ny} cells, {args.per_side ** 2} markers/cell ({n} markers), {args.order} order",
           "peak_gbs": peak, "kernels": {}}

    def rec(name, ms, nbytes):
        out["kernels"][name] = {"ms": ms, "markers_per_s": n / (ms * 1e-3), "algorithmic_GB": nbytes / 1e9,
                                "GBs": nbytes / (ms * 1e-3) / 1e9, "frac": nbytes / (ms * 1e-3) / 1e9 / peak}

    ms = timed(lambda: s.markers_to_grid(xm, ym, eta, rho, count_empty=False), args.reps, st)
    rec("markers_to_grid", ms, 32 * n + 24 * cells)
    eb, ep, rb, ne = s.markers_to_grid(xm, ym, eta, rho)
    out["n_empty"] = ne
    ms = timed(lambda: s.grid_to_markers(xm, ym, vx, vy), args.reps, st)
    rec("grid_to_markers", ms, 32 * n + 16 * cells)
    dt = s.marker_timestep(vx, vy, 0.5, 1e9)
    for scheme in ("euler", "heun", "rk4", "lpi2", "lpi3"):
        x2, y2 = xm.clone(), ym.clone()
        ms = timed(lambda: s.advect_markers(x2, y2, vx, vy, dt, scheme, count_clamped=False), args.reps, st)
        rec("advect_" + scheme, ms, 32 * n + 16 * cells)
    ms = timed(lambda: s.marker_timestep(vx, vy, 0.5, 1e9), args.reps, st)
    rec("timestep", ms, 16 * cells)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
