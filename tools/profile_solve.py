"""One solve of a workload inside a cudaProfilerStart/Stop range (for ncu
--profile-from-start off): setup + one warm-up solve outside the range.  The host solve loop
is used (STOKES_DEVICE_LOOP=0): ncu's launch list does not descend into the device loop's
conditional graph nodes, so the per-iteration graphs are replayed from the host instead."""
import argparse
import json
import os
import sys

os.environ.setdefault("STOKES_DEVICE_LOOP", "0")

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes  # noqa: E402
from synth.fields import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="layered")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--max-iter", type=int, default=0)
args = ap.parse_args()
pre = json.load(open(os.path.join(ROOT, "configs", "presets.json")))[args.workload]
nx, ny = pre["n"] if not args.n else (args.n, args.n)
w = workload(args.workload, nx, ny)
opts = dict(pre["opts"])
if args.max_iter:
    opts["max_iter"] = args.max_iter
s = Stokes(nx, ny, w["Lx"], w["Ly"], w["bc"], **opts)
s.set_viscosity(torch.from_numpy(w["eta_b"]).cuda(), torch.from_numpy(w["eta_p"]).cuda())
s.set_density(torch.from_numpy(w["rho_b"]).cuda())
s.set_gravity(w["gx"], w["gy"])
r = s.solve(pre["rtol"])
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = s.solve(pre["rtol"])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(json.dumps({"workload": args.workload, "n": [nx, ny], "iters": r["iters"], "E": r["E"],
                  "levels": [s.level_shape(l) for l in range(s.num_levels)]}))
