#!/usr/bin/env python
"""Kernel-variant experiments: build the library with compile-time knobs of
csrc/ (-D defines) into build/variants/<name>.so, then time the fine-level kernels of each
variant with stokes_time_kernel (CUDA events, the bench's launch configuration).

    python tools/variants.py build NAME DEF=VAL [DEF=VAL ...]   # on the CPU box
    python tools/variants.py time [--n 4096] [--kernels residual_restrict,jacobi2] NAME ...
                                                                 # on the GPU (one subprocess per variant)
    python tools/variants.py solve [--n 4096] [--workload layered] NAME ...
                                                                 # time-to-solution (CUDA events, 3 solves)
NAME "main" is the in-tree library.  Knobs: RR_NS / RR_ROWS / RR_MINB (residual+restriction
ring depth, residual rows, CTAs per SM), J2_NSJ / J2_JT (two-sweep pass ring depth, CTA width).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "build", "variants")
sys.path.insert(0, ROOT)


def path_of(name):
    if name == "main":
        from paper_2603_14040_b200 import build
        return build.LIB
    return os.path.join(VDIR, name + ".so")


def do_build(name, defs):
    from paper_2603_14040_b200 import build
    os.makedirs(VDIR, exist_ok=True)
    build.build(out=path_of(name), defs=defs)
    json.dump({"name": name, "defs": defs}, open(os.path.join(VDIR, name + ".json"), "w"))
    print(f"built {path_of(name)} with {defs}")


CHILD = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
import torch
from paper_2603_14040_b200 import Stokes
from synth.fields import workload
pre = json.load(open(os.path.join(%(root)r, "configs", "presets.json")))["layered"]
w = workload("layered", %(n)d, %(n)d)
s = Stokes(%(n)d, %(n)d, w["Lx"], w["Ly"], w["bc"], **pre["opts"])
T = lambda a: torch.from_numpy(a).cuda()
s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
s.set_density(T(w["rho_b"]))
s.set_gravity(w["gx"], w["gy"])
out = {}
for k in %(kernels)r:
    best = None
    for _ in range(3):
        ms, nb = s.time_kernel(k, 20)
        best = ms if best is None else min(best, ms)
    out[k] = {"us": best * 1e3, "GBs": nb / best / 1e6}
print(json.dumps(out))
"""


SOLVE = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
import torch
from paper_2603_14040_b200 import Stokes
from synth.fields import workload
pre = json.load(open(os.path.join(%(root)r, "configs", "presets.json")))[%(wl)r]
w = workload(%(wl)r, %(n)d, %(n)d)
s = Stokes(%(n)d, %(n)d, w["Lx"], w["Ly"], w["bc"], **pre["opts"])
T = lambda a: torch.from_numpy(a).cuda()
s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
s.set_density(T(w["rho_b"]))
s.set_gravity(w["gx"], w["gy"])
r = s.solve(pre["rtol"])
ms = []
for _ in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = s.solve(pre["rtol"])
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print(json.dumps({"solve_ms": min(ms), "iters": r["iters"], "status": r["status"]}))
"""


def do_solve(names, n, wl):
    rows = []
    for name in names:
        env = dict(os.environ, STOKES_LIB=path_of(name))
        r = subprocess.run([sys.executable, "-c", SOLVE % {"root": ROOT, "n": n, "wl": wl}], env=env,
                           capture_output=True, text=True, timeout=1800)
        if r.returncode:
            print(name, "FAILED", r.stderr[-500:], flush=True)
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        meta = os.path.join(VDIR, name + ".json")
        defs = json.load(open(meta))["defs"] if os.path.exists(meta) else []
        row = {"variant": name, "defs": defs, "workload": wl, "n": n, **res}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows


def do_time(names, n, kernels):
    rows = []
    for name in names:
        env = dict(os.environ, STOKES_LIB=path_of(name))
        code = CHILD % {"root": ROOT, "n": n, "kernels": kernels}
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        if r.returncode:
            print(name, "FAILED", r.stderr[-500:], flush=True)
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        meta = os.path.join(VDIR, name + ".json")
        defs = json.load(open(meta))["defs"] if os.path.exists(meta) else []
        row = {"variant": name, "defs": defs, "n": n, **res}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    if sys.argv[1] == "build":
        do_build(sys.argv[2], sys.argv[3:])
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("names", nargs="+")
        ap.add_argument("--n", type=int, default=4096)
        ap.add_argument("--kernels", default="residual_restrict,jacobi2")
        ap.add_argument("--workload", default="layered")
        a = ap.parse_args()
        if a.cmd == "solve":
            do_solve(a.names, a.n, a.workload)
        else:
            do_time(a.names, a.n, a.kernels.split(","))
