#!/usr/bin/env python
"""Write tests/golden/solve_<workload>_<n>.json: the ORACLE's full solve of a headline-family
workload at a size the oracle finishes in minutes -- iteration count, the energy residual
after every iteration, and a seeded sample of the converged fields -- for the GPU parity
tests (tests/test_gpu_golden.py: counts +-1, E history, fields at equal count <= 1e-9).

Calls only oracle/ (and the shared input generators in synth/): no value here comes from
the CUDA path.   usage: python tools/make_golden_counts.py [layered:1024 random:1024 ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from synth.fields import workload  # noqa: E402

PRE = json.load(open(os.path.join(ROOT, "configs", "presets.json")))
NSAMPLE = 4096


def sample_index(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, shape[0], NSAMPLE), rng.integers(0, shape[1], NSAMPLE)


def make(name, n):
    pre = PRE[name]
    w = workload(pre["workload"], n, n)
    o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **pre["opts"])
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(w["gx"], w["gy"])
    t0 = time.perf_counter()
    r = o.solve(pre["rtol"], hist_len=20000)
    dt = time.perf_counter() - t0
    out = {"workload": name, "n": n, "opts": pre["opts"], "rtol": pre["rtol"], "status": r["status"],
           "iters": r["iters"], "E": r["E"], "hist": [float(x) for x in r["hist"]],
           "oracle_seconds": dt, "source": "tools/make_golden_counts.py (oracle/ only)", "fields": {}}
    for s, k in enumerate(("vx", "vy", "p")):
        a = r[k]
        ii, jj = sample_index(a.shape, 100 + s)
        out["fields"][k] = {"i": ii.tolist(), "j": jj.tolist(), "v": a[ii, jj].tolist(),
                            "norm": float(np.linalg.norm(a))}
    path = os.path.join(ROOT, "tests", "golden", f"solve_{name}_{n}.json")
    json.dump(out, open(path, "w"))
    print(f"{name} {n}: {r['iters']} iterations, E {r['E']:.3e}, {dt:.0f} s -> {path}", flush=True)


if __name__ == "__main__":
    jobs = sys.argv[1:] or ["layered:1024", "random:1024", "layered:2048"]
    for j in jobs:
        name, n = j.split(":")
        make(name, int(n))
