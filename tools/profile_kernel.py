"""Launch one hot-path kernel (stokes_time_kernel, 2 warm-ups + reps) inside a
cudaProfilerStart/Stop range on a full-size workload, for ncu --profile-from-start off."""
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
ap.add_argument("--kernels", default="jacobi,energy")
args = ap.parse_args()
pre = json.load(open(os.path.join(ROOT, "configs", "presets.json")))[args.workload]
w = workload(args.workload, args.n, args.n)
s = Stokes(args.n, args.n, w["Lx"], w["Ly"], w["bc"], **pre["opts"])
s.set_viscosity(torch.from_numpy(w["eta_b"]).cuda(), torch.from_numpy(w["eta_p"]).cuda())
s.set_density(torch.from_numpy(w["rho_b"]).cuda())
s.set_gravity(w["gx"], w["gy"])
torch.cuda.synchronize()
torch.cuda.profiler.start()
for k in args.kernels.split(","):
    s.time_kernel(k, 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
