#!/usr/bin/env python
"""Per-iteration cost of the 2D decomposition on ONE B200.

For each configuration the solve runs a fixed number of Uzawa iterations from zero twice
(k1 and k2 iterations) and reports (t(k2) - t(k1)) / (k2 - k1): the steady per-iteration
time without setup / graph capture.  CUDA events on the handle's stream.
    single   one domain of n x n cells
    dd       px x py tiles of n/px x n/py cells (the same problem, decomposed)
    weak     px x py tiles of n x n cells each (a weak-scaling problem on one GPU: divide
             the time by px * py to compare with `single`)
usage: python tools/dist_cost.py [--n 4096] [--px 2 --py 2] [--transports virtual,loopback,nccl_self]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_14040_b200 import Stokes, StokesDist  # noqa: E402
from synth.fields import workload  # noqa: E402


def per_iter(make, k1=5, k2=25):
    ts = []
    for k in (k1, k2):
        s = make(k)
        s.solve(0.0)  # graphs captured, warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s.stream)
        r = s.solve(0.0)
        e1.record(s.stream)
        torch.cuda.synchronize()
        assert r["iters"] == k
        ts.append(e0.elapsed_time(e1))
        E = r["E"]
        s.close()
    return (ts[1] - ts[0]) / (k2 - k1), E


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--px", type=int, default=2)
    ap.add_argument("--py", type=int, default=2)
    ap.add_argument("--workload", default="layered")
    ap.add_argument("--transports", default="virtual,loopback,nccl_self")
    ap.add_argument("--weak", action="store_true", help="also px x py tiles of n x n each")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    opts = dict(omega_v=0.6, alpha_p=1.0)
    rows = []

    def handle(cls, nx, ny, k, **kw):
        w = workload(a.workload, nx, ny, float(nx) / a.n, float(ny) / a.n)
        s = cls(nx, ny, w["Lx"], w["Ly"], w["bc"], max_iter=k, **opts, **kw)
        T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
        s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
        s.set_density(T(w["rho_b"]))
        s.set_gravity(w["gx"], w["gy"])
        return s

    ms, E = per_iter(lambda k: handle(Stokes, a.n, a.n, k))
    rows.append({"config": f"single {a.n}x{a.n}", "ms_per_iter": ms, "E": E})
    print(json.dumps(rows[-1]), flush=True)
    for tr in a.transports.split(","):
        ms, E = per_iter(lambda k: handle(StokesDist, a.n, a.n, k, px=a.px, py=a.py, transport=tr))
        rows.append({"config": f"dd {a.px}x{a.py} of {a.n // a.px}x{a.n // a.py} ({tr})", "ms_per_iter": ms,
                     "vs_single": ms / rows[0]["ms_per_iter"], "E": E})
        print(json.dumps(rows[-1]), flush=True)
        if a.weak:
            ms, E = per_iter(lambda k: handle(StokesDist, a.n * a.px, a.n * a.py, k, px=a.px, py=a.py, transport=tr))
            nt = a.px * a.py
            rows.append({"config": f"weak {a.px}x{a.py} tiles of {a.n}x{a.n} ({tr})", "ms_per_iter": ms,
                         "ms_per_iter_per_tile": ms / nt, "vs_single": ms / nt / rows[0]["ms_per_iter"], "E": E})
            print(json.dumps(rows[-1]), flush=True)
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
