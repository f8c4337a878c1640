#!/usr/bin/env python
"""Diagnosis of GCR(m)-MG stagnation on the block workload on the CPU
ORACLE (test infrastructure; no GPU): energy-residual histories of GCR(m) with the paper's
Euclidean inner product over the unknowns (the default) and with the
energy-weighted one (the weights of the stopping test E; reading R33),
with the true-residual restart (R13) and the paper-literal recursive one.
usage: python tools/gcr_stagnation.py [--n 128] [--m 10] [--iters 400] [--out F.jsonl]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402
from synth.fields import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="block")
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--m", default="10,30")
ap.add_argument("--iters", type=int, default=400)
ap.add_argument("--out", default=None)
ap.add_argument("--inner", default="0,1")
ap.add_argument("--restart", default="1,0")
ap.add_argument("--checkpoints", default="", help="iteration counts at which ||r||_2 / ||f||_2 is evaluated")
a = ap.parse_args()
w = workload(a.workload, a.n, a.n)
rows = []
for m in [int(x) for x in a.m.split(",")]:
    for inner in [int(x) for x in a.inner.split(",")]:
        for tr in [int(x) for x in a.restart.split(",")]:
            def make(k):
                o = Oracle(a.n, a.n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=m,
                           gcr_inner=inner, gcr_true_restart=tr, max_iter=k)
                o.set_viscosity(w["eta_b"], w["eta_p"])
                o.set_density(w["rho_b"])
                o.set_gravity(w["gx"], w["gy"])
                return o
            t0 = time.perf_counter()
            o = make(a.iters)
            r = o.solve(1e-8, hist_len=a.iters)
            h = r["hist"]
            # the Euclidean norm of the true residual over the unknowns (what GCR minimises,
            # PAPER.md:1440) relative to that of f, at the checkpoints
            r2 = {}
            f0 = o.residual(o.zeros("vx"), o.zeros("vy"), o.zeros("p"))
            nf = np.sqrt(sum(float(np.sum(x * x)) for x in f0[:3]))
            for k in [int(x) for x in a.checkpoints.split(",") if x]:
                if k > r["iters"]:
                    continue
                ok = make(k)
                rk = ok.solve(0.0)
                res = ok.residual(rk["vx"], rk["vy"], rk["p"])
                r2[str(k)] = float(np.sqrt(sum(float(np.sum(x * x)) for x in res[:3])) / nf)
            row = {"workload": a.workload, "n": a.n, "m": m, "inner": ["euclidean", "energy"][inner],
                   "restart": ["recursive", "true"][tr], "iters": r["iters"], "status": r["status"], "E": r["E"],
                   "E_at": {str(k): float(h[k - 1]) for k in (10, 50, 100, 200, 400, 1000, 2000) if k <= len(h)},
                   "r2_rel_at": r2,
                   "s": time.perf_counter() - t0}
            rows.append(row)
            print(json.dumps(row), flush=True)
if a.out:
    with open(a.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
