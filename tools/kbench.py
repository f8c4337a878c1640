"""Per-kernel CUDA-event timings (stokes_time_kernel) on a workload, + achieved GB/s."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="layered")
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
pre = json.load(open(os.path.join(ROOT, "configs", "presets.json")))[args.workload]
w = workload(args.workload, args.n, args.n)
s = Stokes(args.n, args.n, w["Lx"], w["Ly"], w["bc"], **pre["opts"])
s.set_viscosity(torch.from_numpy(w["eta_b"]).cuda(), torch.from_numpy(w["eta_p"]).cuda())
s.set_density(torch.from_numpy(w["rho_b"]).cuda())
s.set_gravity(w["gx"], w["gy"])
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
out = {}
for k in Stokes.KERNELS:
    ms, nb = s.time_kernel(k, args.reps)
    out[k] = {"ms": ms, "GB/s": nb / ms / 1e6, "frac": nb / ms / 1e6 / peak}
    print(f"{k:20s} {ms * 1e3:9.1f} us  {nb / ms / 1e6:8.1f} GB/s  {out[k]['frac'] * 100:5.1f}% of {peak}")
print(json.dumps(out))
