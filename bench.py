#!/usr/bin/env python
"""Benchmark of the B200-native multigrid Stokes solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload layered] [--impl ours|reference]

metric  "Stokes MG solve time & DOF-sweeps/s to 1e-8 rel. residual; smoother % HBM peak"
value   whole-job DOF-sweeps/s: sum over levels of (velocity unknowns x smoother sweeps
        executed) of one solve to E <= 1e-8, x solves x ranks / max-over-ranks device time
step    one full solve (all of SURVEY §8(a): V-cycles, smoother, transfers, coarse solve,
        pressure update, energy residual, stopping test) from a zero initial guess on
        inputs resident in HBM; ms_per_step = solve time
workload default: BASELINE configs[3], layered lithosphere/mantle viscosity, 4096 x 4096 cells
        per GPU, plain Uzawa-MG (presets in configs/presets.json); the single-GPU config
        the metric's "% HBM peak" part is meaningful on (inputs ~1.4 GB >> 126 MB L2).
N > 1   (torchrun): weak scaling, one 4096^2 tile per GPU of a px x py global grid (2x1, 2x2,
        4x2), the exact 2D domain decomposition (stokes_create_dist: NCCL halo exchange
        over NVLink, agglomerated coarse tail); value = global DOF-sweeps / max-over-ranks time.
e2e     the same solve through the public API (Stokes.set_viscosity / set_density / solve)
        with pinned HOST inputs and outputs: H2D of eta_b, eta_p, rho_b and D2H of vx, vy, p
        inside the timed region.
roofline the dominant kernel, the fine-level two-sweep Jacobi pass (the smoother, PAPER.md:
        2396/3209, two sweeps per HBM pass): algorithmic bytes per launch (64 B/cell, DESIGN.md
        §6) / its CUDA-event time (stokes_time_kernel on the handle's stream, live in this run)
        vs the measured HBM copy peak; the other fine-level kernels listed beside it.
--impl reference: the CPU oracle (oracle/, plain C, 1 thread) on the same workload,
        each step one Uzawa iteration of the full-size problem (bounded sample).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Stokes MG solve time & DOF-sweeps/s to 1e-8 rel. residual; smoother % HBM peak"
UNIT = "DOF-sweeps/s"
WORKLOAD_DOC = {
    "mms": "cfg1 32x32 manufactured solution, eta=1, free slip",
    "block": "cfg2 sinking block [3/8,5/8]^2, eta contrast 1e3, free slip",
    "solcx": "cfg3 SolCx-like eta jump 1e6 at x=1/2, GCR(10)+MG",
    "layered": "cfg4 layered lithosphere/mantle eta (1e3/1/30), 4096x4096 cells per GPU, Uzawa-MG",
    "random": "cfg5 random log-perturbed eta in [0.1,10]",
}


def presets():
    return json.load(open(os.path.join(ROOT, "configs", "presets.json")))


def dof_sweeps_per_vcycle(level_shapes, smoother):
    """sum over non-coarsest levels of velocity unknowns x (pre + post) sweeps."""
    tot = 0
    for (nx, ny, nu) in level_shapes[:-1]:
        tot += (ny * (nx - 1) + (ny - 1) * nx) * 2 * nu
    return tot


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peak():
    try:
        m = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fine_launches(nu, fused, jju=True):
    """Fine-level launches per V-cycle (driver.cu vcycle / smooth / solve_uzawa_fused): the
    Uzawa update fused into the first pre-sweep (Uzawa mode) and, with k_jju, the last
    post-sweep fused into that pass too; sweep pairs as two-sweep passes (an even pair count
    without k_jju)."""
    pre_n = nu - (1 if fused else 0)
    post_n = nu - (1 if fused and jju else 0)
    pre, post = pre_n // 2, post_n // 2
    if not (fused and jju) and (pre + post) % 2:
        if post > 0:
            post -= 1
        else:
            pre -= 1
    out = {"jacobi2": pre + post, "jacobi": pre_n - 2 * pre + post_n - 2 * post,
           "residual_restrict": 1, "prolong": 1}
    if fused and jju:
        out["jju"] = 1
    elif fused:
        out["jacobi_uzawa"] = 1
    return out


def ncu_traffic(kernel_bytes_key, name="ncu_jacobi2_traffic.json"):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        d = json.load(open(path))
        return d.get(kernel_bytes_key)
    except Exception:
        return None


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":  # one GPU per rank, bound before the process group's first collective
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class OracleSample:
    """The oracle as it stands on this host's cores (1 thread), set up once on the full-size
    workload; one sample = one Uzawa iteration (V-cycle + pressure update + energy residual)
    from the zero initial guess, the bounded piece of a solve timed as the CPU baseline."""

    def __init__(self, name, pre):
        from oracle.oracle import Oracle
        from synth.fields import workload
        self.name, (self.nx, self.ny) = name, pre["n"]
        w = workload(name, self.nx, self.ny)
        opts = dict(pre["opts"], max_iter=1, accel=0)
        self.o = Oracle(self.nx, self.ny, w["Lx"], w["Ly"], w["bc"], **opts)
        self.o.set_viscosity(w["eta_b"], w["eta_p"])
        self.o.set_density(w["rho_b"])
        self.o.set_gravity(w["gx"], w["gy"])
        shp = [self.o.level_shape(l) for l in range(self.o.nlev)]
        self.per_vc = dof_sweeps_per_vcycle(shp, opts.get("smoother", 0))

    def step(self):
        t0 = time.perf_counter()
        r = self.o.solve(0.0)
        dt = time.perf_counter() - t0
        return r["iters"] * self.per_vc / dt, dt

    def describe(self, dt):
        return (f"1 Uzawa iteration (V-cycle + p-update + energy residual) of {self.name} {self.nx}x{self.ny}, "
                f"{dt:.2f} s on 1 thread of {os.cpu_count()} ({_cpu_model()})")


def cpu_baseline(name, pre):
    smp = OracleSample(name, pre)
    v, dt = smp.step()
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": smp.describe(dt)}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown CPU"


def run_reference(args, world, rank):
    """Reference arm: the CPU oracle (no installable reference exists: /root/reference holds
    only the paper), each step one bounded sample of the same workload."""
    if rank != 0:
        return 0
    pre = presets()[args.workload]
    smp = OracleSample(args.workload, pre)
    for _ in range(args.warmup):
        smp.step()
    vals, dts = [], []
    for _ in range(args.steps):
        v, dt = smp.step()
        vals.append(v)
        dts.append(dt)
    v = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(dts) / len(dts), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}: {WORKLOAD_DOC[args.workload]}", "grid": pre["n"],
                       "sample": "each step = 1 Uzawa iteration of the full-size problem on the CPU oracle"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": smp.describe(sum(dts) / len(dts))},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_strong(args, world, rank, local, steps, warmup):
    """BASELINE config 5: the random log-perturbed viscosity problem at its preset size
    (16384^2 cells) split over the N GPUs (strong scaling; N = 1: one domain).  Inputs are
    sampled on the device (synth.fields.random_torch, same recipe as the parity fields).
    Returns the timing block (device time, max over ranks)."""
    import torch
    from paper_2603_14040_b200 import Stokes, StokesDist
    from paper_2603_14040_b200.decomp import strong_problem, tile_windows
    from synth.fields import random_torch
    dev = torch.device("cuda", local)
    pre = presets()["random"]
    rtol, opts = pre["rtol"], dict(pre["opts"])
    NX, NY, Lx, Ly, px, py = strong_problem(world, pre["n"][0])
    if world > 1:
        win = tile_windows(NX, NY, px, py, rank)
        i0, j0 = win["b"][0].start, win["b"][1].start
        nxt, nyt = NX // px, NY // py
        w = random_torch(NX, NY, Lx, Ly, win_b=(i0, j0, nyt + 1, nxt + 1), win_p=(i0, j0, nyt, nxt), device=dev)
        s = StokesDist(NX, NY, Lx, Ly, w["bc"], px=px, py=py, rank=rank, **opts)
    else:
        w = random_torch(NX, NY, Lx, Ly, device=dev)
        s = Stokes(NX, NY, Lx, Ly, w["bc"], **opts)
    s.set_viscosity(w["eta_b"], w["eta_p"])
    s.set_density(w["rho_b"])
    s.set_gravity(w["gx"], w["gy"])
    del w
    per_vc = dof_sweeps_per_vcycle(global_levels(NX, NY, opts), opts.get("smoother", 0))
    for _ in range(warmup):
        s.solve(rtol)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    s.launch_count(reset=True)
    with Clocks(local) as clk:
        e0.record(s.stream)
        for _ in range(steps):
            r = s.solve(rtol)
            assert r["status"] == 0, f"strong-scaling solve status {r['status']}"
            iters.append(r["iters"])
        e1.record(s.stream)
        torch.cuda.synchronize()
    launches = s.launch_count()
    barrier(world)
    ms = allreduce_max(e0.elapsed_time(e1), world, dev)
    s.close()
    dofs = sum(iters) * opts.get("vcycles_per_iter", 1) * per_vc
    return {"workload": f"random: {WORKLOAD_DOC['random']}, {NX}x{NY} cells split over {world} GPU(s)",
            "grid_global": [NX, NY], "grid_per_gpu": [NX // px, NY // py], "parallelism": f"dd{px}x{py}",
            "n_gpus": world, "steps": steps, "ms_per_solve": ms / steps, "iters_per_solve": statistics.mean(iters),
            "value": dofs / (ms / 1e3), "unit": UNIT, "scaling": "strong", "gpu_launches": launches,
            "clocks": clk.summary(), "data": "synthetic (sampled on the device, synth.fields.random_torch)"}


def run_ours(args, world, rank, local):
    import torch
    from paper_2603_14040_b200 import Stokes, StokesDist
    from paper_2603_14040_b200.decomp import tile_windows, weak_problem
    from paper_2603_14040_b200.stokes import shapes
    from synth.fields import workload

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.scaling == "strong":  # the headline is BASELINE config 5 (strong scaling)
        st = run_strong(args, world, rank, local, args.steps, args.warmup)
        if rank == 0:
            line = {"metric": METRIC, "value": st["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": st["ms_per_solve"], "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": st["data"],
                    "config": {"workload": st["workload"], "grid_global": st["grid_global"],
                               "grid_per_gpu": st["grid_per_gpu"], "parallelism": st["parallelism"],
                               "iters_per_solve": st["iters_per_solve"],
                               "l2": "inputs larger than L2 (16384^2 fields, 2.1 GB each)"},
                    "gpu_launches": st["gpu_launches"], "clocks": st["clocks"]}
            print(json.dumps(line), flush=True)
        return 0
    pre = presets()[args.workload]
    rtol = pre["rtol"]
    opts = dict(pre["opts"])
    tile_n = pre["n"]
    if world > 1:
        # weak scaling (BASELINE config 4): one tile_n[0] x tile_n[1] tile per GPU, exact 2D
        # decomposition over NVLink (stokes_create_dist, NCCL transport)
        if opts.get("accel", 0):
            opts["accel"] = 0  # the decomposed path runs plain Uzawa-MG
        NX, NY, Lx, Ly, px, py = weak_problem(world, tile_n[0])
        win = tile_windows(NX, NY, px, py, rank)
        i0, j0 = win["b"][0].start, win["b"][1].start
        nxt, nyt = NX // px, NY // py
        w = workload(args.workload, NX, NY, Lx, Ly, win_b=(i0, j0, nyt + 1, nxt + 1), win_p=(i0, j0, nyt, nxt))
        s = StokesDist(NX, NY, Lx, Ly, w["bc"], px=px, py=py, rank=rank, **opts)
        gshape = [s.gnx, s.gny]
    else:
        NX, NY = tile_n
        px = py = 1
        w = workload(args.workload, NX, NY)
        s = Stokes(NX, NY, w["Lx"], w["Ly"], w["bc"], **opts)
        gshape = [NX, NY]
    nx, ny = s.nx, s.ny
    eb, ep, rho = (torch.from_numpy(w[k]).to(dev) for k in ("eta_b", "eta_p", "rho_b"))
    s.set_viscosity(eb, ep)
    s.set_density(rho)
    s.set_gravity(w["gx"], w["gy"])
    # DOF-sweeps of one V-cycle on the GLOBAL hierarchy (identical to the single-domain one)
    shp = global_levels(gshape[0], gshape[1], opts)
    if world == 1:
        assert shp == [tuple(s.level_shape(l)) for l in range(s.num_levels)], "level rule mismatch"
    per_vc = dof_sweeps_per_vcycle(shp, opts.get("smoother", 0))
    vpi = opts.get("vcycles_per_iter", 1)
    stream = s.stream

    for _ in range(args.warmup):
        r = s.solve(rtol)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    s.launch_count(reset=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = s.solve(rtol)
            iters.append(r["iters"])
            assert r["status"] == 0, f"solve status {r['status']}"
        e1.record(stream)
        torch.cuda.synchronize()
    launches = s.launch_count()
    barrier(world)
    ms = e0.elapsed_time(e1)
    ms_max = allreduce_max(ms, world, dev)
    dofs = sum(iters) * vpi * per_vc  # whole job (global problem)
    value = dofs / (ms_max / 1e3)

    # ---- e2e through the public API with pinned host buffers (this rank's arrays)
    host = {k: torch.from_numpy(w[k]).pin_memory() for k in ("eta_b", "eta_p", "rho_b")}
    sh = shapes(nx, ny)
    hz = {k: torch.zeros(sh[k], dtype=torch.float64).pin_memory() for k in ("vx", "vy", "p")}
    hout = {k: torch.empty(sh[k], dtype=torch.float64).pin_memory() for k in ("vx", "vy", "p")}
    h2d = sum(t.numel() * 8 for t in host.values()) + sum(t.numel() * 8 for t in hz.values())
    d2h = sum(t.numel() * 8 for t in hout.values())
    barrier(world)
    torch.cuda.synchronize()
    e2 = []
    e2_iters = 0
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        s.set_viscosity(host["eta_b"], host["eta_p"])
        s.set_density(host["rho_b"])
        r = s.solve(rtol, vx=hz["vx"], vy=hz["vy"], p=hz["p"], out=hout)
        torch.cuda.synchronize()
        e2.append(time.perf_counter() - t0)
        # the same computation as the device-timed solves: converged, same iteration count
        assert r["status"] == 0, f"e2e solve status {r['status']}"
        assert r["iters"] == iters[-1], f"e2e solve took {r['iters']} iterations, device solve {iters[-1]}"
        assert not r["vx"].is_cuda
        e2_iters += r["iters"]
    e2_t = allreduce_max(sum(e2), world, dev)
    e2e_value = e2_iters * vpi * per_vc / e2_t

    # ---- roofline of the dominant kernel (the fine-level two-sweep Jacobi pass), live CUDA
    # events, on a single-domain handle of this GPU's tile; the other fine-level kernels of
    # the step beside it
    kh = s if world == 1 else Stokes(nx, ny, 1.0, 1.0, w["bc"], **opts)
    if world > 1:
        kh.set_viscosity(eb, ep)
        kh.set_density(rho)
        kh.set_gravity(w["gx"], w["gy"])
    peak, peak_src = measured_peak()
    counts = fine_launches(shp[0][2], opts.get("accel", 0) == 0 and vpi == 1,
                           jju=world == 1 and os.environ.get("STOKES_JJU", "1") != "0")
    its = statistics.mean(iters)
    kernels = {}
    for name in ("jacobi2", "jju", "jacobi", "jacobi_uzawa", "residual_restrict", "prolong"):
        try:
            km, kb = kh.time_kernel(name, reps=20)
        except Exception:
            continue
        n_per = its * vpi * counts.get(name, 0)
        kernels[name] = {"launch_ms": km, "GBs": kb / (km / 1e3) / 1e9, "frac": kb / (km / 1e3) / 1e9 / peak,
                         "launches_per_solve": n_per, "share_of_step": n_per * km / (ms / args.steps)}
    dom = "jacobi2" if "jacobi2" in kernels else "jacobi"
    k_ms = kernels[dom]["launch_ms"]
    k_bytes = kernels[dom]["GBs"] * 1e9 * k_ms / 1e3
    achieved = kernels[dom]["GBs"]
    share = kernels[dom]["share_of_step"]
    tr = ncu_traffic("dram_bytes_per_launch") if dom == "jacobi2" else ncu_traffic(
        "dram_bytes_per_launch", "ncu_jacobi_traffic.json")

    # ---- informational: the same solve with the paper's Anderson acceleration AA(10, 1)
    # (PAPER.md:1502-1588), the fastest configuration measured (not the headline: its sweeps
    # per solve differ).  Single GPU only; CUDA events on its handle's stream.
    alt = None
    if world == 1 and args.workload == "layered":
        try:
            kh = None
            aa = Stokes(NX, NY, w["Lx"], w["Ly"], w["bc"], **dict(opts, accel=2, aa_depth=10, aa_beta=1.0))
            aa.set_viscosity(eb, ep)
            aa.set_density(rho)
            aa.set_gravity(w["gx"], w["gy"])
            aa.solve(rtol)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(aa.stream)
            ra = aa.solve(rtol)
            a1.record(aa.stream)
            torch.cuda.synchronize()
            alt = {"solver": "Uzawa-MG + Anderson AA(10, 1)", "ms_per_solve": a0.elapsed_time(a1),
                   "iters_per_solve": ra["iters"], "E": ra["E"], "status": ra["status"]}
            aa.close()
        except Exception as ex:  # informational only
            alt = {"error": str(ex)[:200]}

    # ---- BASELINE config 5 beside the headline: the fixed 16384^2 random problem split over
    # the same N GPUs (strong scaling; the driver's scaling run then yields both curves)
    strong = None
    if not args.no_strong:
        kh = None
        torch.cuda.empty_cache()
        try:
            strong = run_strong(args, world, rank, local, max(1, min(args.steps, 2)), 1)
        except Exception as ex:  # reported, never silently dropped
            strong = {"error": str(ex)[:300]}
    if rank != 0:
        return 0
    cb = cpu_baseline(args.workload, pre) if world == 1 and not args.no_cpu_baseline else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {WORKLOAD_DOC[args.workload]}", "grid_per_gpu": [nx, ny],
                   "grid_global": gshape, "levels": [list(x) for x in shp], "opts": opts, "rtol": rtol,
                   "iters_per_solve": statistics.mean(iters), "solve_ms": ms_max / args.steps,
                   "dof_sweeps_per_solve": dofs / args.steps,
                   "l2": "inputs larger than L2 (fine fields 16.8M cells x 8 B per GPU, hierarchy > 1 GB vs 126 MB L2)",
                   "parallelism": f"dd{px}x{py}" if world > 1 else "single GPU"},
        "roofline": {"kernel": ("fine-level two-sweep damped-Jacobi pass (k_jacobi2)" if dom == "jacobi2" else
                                "fine-level damped-Jacobi sweep (k_stream<JacobiOp>)"), "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": tr,
                     "algorithmic_bytes_per_launch": k_bytes, "launch_ms": k_ms, "peak_source": peak_src,
                     "share_of_step": share, "fine_kernels": kernels,
                     # informational: the pass performs two sweeps; one-sweep-per-pass smoothing
                     # would move these bytes twice
                     "sweep_equivalent_GBs": 2 * achieved if dom == "jacobi2" else achieved},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                "seconds_per_step": e2_t / len(e2), "iters_per_solve": e2_iters / len(e2)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if cb is not None:
        line["cpu_baseline"] = cb
    if alt is not None:
        line["accelerated"] = alt
    if strong is not None:
        line["strong_scaling"] = strong
    print(json.dumps(line), flush=True)
    return 0


def global_levels(nx, ny, opts):
    """(ncx, ncy, nu) of the global hierarchy (reading R8/R9), as the library builds it."""
    import math
    cm = opts.get("coarse_min", 8)
    nu1, g = opts.get("nu1", 5), opts.get("nu_growth", 1.0)
    out, l = [], 0
    while True:
        out.append((nx, ny, int(math.floor(nu1 * g ** l + 0.5))))
        l += 1
        if nx % 2 or ny % 2 or min(nx, ny) // 2 < cm:
            break
        nx //= 2
        ny //= 2
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="layered", choices=sorted(WORKLOAD_DOC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: BASELINE cfg 4 per GPU (default); strong: cfg 5, 16384^2 split over N")
    ap.add_argument("--no-strong", action="store_true", help="skip the cfg-5 strong-scaling block")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    world, rank, local = dist_init(args)
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank)
        return run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
