"""Pins of the oracle's solve (no GPU).

P2  manufactured closed-form solution, free slip, eta = 1: second order ("central
    differences"); the MMS is divergence free and free slip on all walls (derived)
P3  no-slip MMS (stream function sin^2 pi x sin^2 pi y, arbitrary force hook): second order
P4  fixed point == bordered dense LU with zero-mean pressure (tests/dense.py)
P9  Uzawa sign (reading R3): physical sign converges, literal PAPER.md:824 sign diverges
P10 GCR (Alg. 4) reaches the dense solution
P12 nullspace: zero-mean pressure; p0 + c gives the same velocity
P14 Uzawa iteration == brute-force spectral radius of (I + alpha eta_P D L^-1 G) on the
    zero-mean subspace (exact inner solve: one level)
P15 one Richardson step x + M^-1 (b - A x) == one Uzawa step
"""
import math

import numpy as np
import pytest

from dense import Dense
from oracle.oracle import EDIVERGED, Oracle
from synth.fields import node_coords, parity_fields, workload

PI = math.pi


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def rms(a):
    return float(np.sqrt(np.mean(a ** 2)))


def mms_errors(n):
    w = workload("mms", n, n)
    o = Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), omega_v=0.6, alpha_p=1.5)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(0.0, 1.0)
    s = o.solve(1e-11)
    assert s["status"] == 0
    y, x = node_coords("vx", n, n, 1.0, 1.0)
    ex = PI * np.sin(PI * x[None, :]) * np.cos(PI * y[:, None])
    y, x = node_coords("vy", n, n, 1.0, 1.0)
    ey = -PI * np.cos(PI * x[None, :]) * np.sin(PI * y[:, None])
    y, x = node_coords("p", n, n, 1.0, 1.0)
    ep = 2 * PI ** 2 * np.cos(PI * x[None, :]) * np.cos(PI * y[:, None])
    return rms(s["vx"] - ex), rms(s["vy"] - ey), rms(s["p"] - ep)


def test_mms_free_slip_second_order():
    errs = np.array([mms_errors(n) for n in (16, 32, 64, 128, 256)])
    orders = np.log2(errs[:-1] / errs[1:])
    assert np.all(np.abs(orders - 2.0) <= 0.2), orders


def noslip_mms(n):
    S = lambda t: np.sin(PI * t) ** 2
    S1 = lambda t: PI * np.sin(2 * PI * t)
    S2 = lambda t: 2 * PI ** 2 * np.cos(2 * PI * t)
    S3 = lambda t: -4 * PI ** 3 * np.sin(2 * PI * t)
    # v = curl psi, psi = S(x) S(y): vx = S(x) S'(y), vy = -S'(x) S(y); p = cos pi x cos pi y
    # f = L v + G p = lap v - grad p (eta = 1, div v = 0)
    y, x = node_coords("vx", n, n, 1.0, 1.0)
    x, y = x[None, :], y[:, None]
    fx = S2(x) * S1(y) + S(x) * S3(y) + PI * np.sin(PI * x) * np.cos(PI * y)
    ex = S(x) * S1(y)
    y, x = node_coords("vy", n, n, 1.0, 1.0)
    x, y = x[None, :], y[:, None]
    fy = -S3(x) * S(y) - S1(x) * S2(y) + PI * np.cos(PI * x) * np.sin(PI * y)
    ey = -S1(x) * S(y)
    y, x = node_coords("p", n, n, 1.0, 1.0)
    ep = np.cos(PI * x[None, :]) * np.cos(PI * y[:, None])
    o = Oracle(n, n, 1.0, 1.0, (1, 1, 1, 1), omega_v=0.6, alpha_p=1.5)
    o.set_viscosity(np.ones((n + 1, n + 1)), np.ones((n, n)))
    o.set_force(fx, fy)
    s = o.solve(1e-11)
    assert s["status"] == 0
    return rms(s["vx"] - ex), rms(s["vy"] - ey), rms(s["p"] - ep)


def test_mms_no_slip_second_order():
    errs = np.array([noslip_mms(n) for n in (16, 32, 64, 128)])
    orders = np.log2(errs[:-1] / errs[1:])
    # velocity is second order; pressure at least first with the mirror wall closure
    assert np.all(np.abs(orders[:, :2] - 2.0) <= 0.2), orders
    assert np.all(orders[:, 2] >= 0.9), orders


@pytest.mark.parametrize("n,bc,accel", [(4, (0, 0, 0, 0), 0), (8, (1, 1, 1, 1), 0), (16, (0, 1, 1, 0), 0),
                                        (8, (0, 0, 0, 0), 1), (16, (1, 0, 0, 1), 1),
                                        (8, (1, 0, 1, 0), 2), (16, (0, 0, 1, 1), 2)])
def test_fixed_point_is_dense_solution(n, bc, accel):
    f = parity_fields(n, n, log_contrast=1.5)
    # i.i.d. 1e3-contrast eta: lambda_max(C^-1 L) ~ 3.4, so omega_v < 0.59 (see jacobi test)
    o = Oracle(n, n, 1.0, 1.0, bc, omega_v=0.4, alpha_p=1.0, coarse_min=2, accel=accel, max_iter=5000)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.2, 1.0)
    s = o.solve(1e-12)
    assert s["status"] == 0, s["status"]
    d = Dense(n, n, 1.0, 1.0, bc, f["eta_b"], f["eta_p"])
    vx, vy, p = d.unpack(d.solve_bordered(d.force(f["rho_b"], 0.2, 1.0)))
    assert rel(s["vx"], vx) <= 1e-10
    assert rel(s["vy"], vy) <= 1e-10
    assert rel(s["p"], p) <= 1e-10


def _mms_oracle(n, **kw):
    w = workload("mms", n, n)
    o = Oracle(n, n, **kw)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(0.0, 1.0)
    return o


def test_uzawa_sign_reading():
    ok = _mms_oracle(32, omega_v=0.6, alpha_p=0.6).solve(1e-8, hist_len=200)
    assert ok["status"] == 0 and np.all(np.diff(np.log(ok["hist"][5:])) < 0.05)
    bad = _mms_oracle(32, omega_v=0.6, alpha_p=0.6, pressure_sign=-1, max_iter=200).solve(1e-8, hist_len=200)
    assert bad["status"] == EDIVERGED or bad["hist"][-1] > 10 * bad["hist"][0]


def test_nullspace_and_shift_invariance():
    o = _mms_oracle(32, omega_v=0.6, alpha_p=1.0)
    a = o.solve(1e-10)
    assert abs(a["p"].mean()) <= 1e-14 * np.abs(a["p"]).max()
    b = o.solve(1e-10, p=np.full((32, 32), 123.0))
    assert rel(b["vx"], a["vx"]) <= 1e-12 and rel(b["p"], a["p"]) <= 1e-12
    assert b["iters"] == a["iters"]


def test_demean_golden():
    """Zero-mean rule: a 1 x 3 pressure [1,2,3] -> [-1,0,1] when the
    solve is already converged (E <= rtol: 0 iterations, only the output de-mean)."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "energy_examples.json")))["demean"]
    o = Oracle(3, 2, 3.0, 2.0)
    o.set_viscosity(np.ones((3, 4)), np.ones((2, 3)))
    o.set_density(np.ones((3, 4)))
    o.set_gravity(0.0, 1.0)
    p = np.array([g["in"], g["in"]])
    s = o.solve(1e300, p=p)
    assert s["iters"] == 0
    assert np.allclose(s["p"], np.array([g["out"], g["out"]]), rtol=0, atol=1e-15)


def test_zero_force_returns_zero():
    o = Oracle(8, 8)
    o.set_viscosity(np.ones((9, 9)), np.ones((8, 8)))
    o.set_density(np.zeros((9, 9)))
    s = o.solve(1e-8, vx=np.ones((8, 9)))
    assert s["iters"] == 0 and not np.any(s["vx"])


def test_uzawa_contraction_is_spectral_radius():
    """P14: one level => the V-cycle is the exact inverse; observed E ratio -> rho(Pi M_p)."""
    n = 8
    rng = np.random.default_rng(4)
    eb = 10 ** rng.uniform(-1, 1, (n + 1, n + 1))
    ep = 10 ** rng.uniform(-1, 1, (n, n))
    rho = rng.uniform(-1, 1, (n + 1, n + 1))
    alpha = 0.8
    o = Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), alpha_p=alpha, coarse_min=8, max_iter=600)
    assert o.nlev == 1
    o.set_viscosity(eb, ep)
    o.set_density(rho)
    o.set_gravity(0.0, 1.0)
    s = o.solve(1e-300, hist_len=600)
    h = s["hist"]
    d = Dense(n, n, 1.0, 1.0, (0, 0, 0, 0), eb, ep)
    Mp = np.eye(d.np_) + alpha * np.diag(ep.ravel()) @ d.D @ np.linalg.solve(d.L, d.G)
    Pi = np.eye(d.np_) - np.full((d.np_, d.np_), 1.0 / d.np_)
    lam = np.abs(np.linalg.eigvals(Pi @ Mp)).max()
    k0, k1 = 400, 599
    observed = (h[k1] / h[k0]) ** (1.0 / (k1 - k0))
    assert observed == pytest.approx(lam, rel=1e-3)
    assert lam < 1


def test_richardson_step_equals_uzawa_step():
    """P15: x + M^-1 (b - A x) (preconditioner of GCR) == one Uzawa step (+ de-mean)."""
    n = 32
    f = parity_fields(n, n, log_contrast=1.0)
    f["vx"][:, [0, -1]] = 0.0  # wall-normal entries are not unknowns
    f["vy"][[0, -1], :] = 0.0
    kw = dict(omega_v=0.5, alpha_p=1.0)
    o = Oracle(n, n, 1.0, 1.0, (0, 1, 0, 1), max_iter=1, **kw)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.0, 1.0)
    one = o.solve(0.0, vx=f["vx"], vy=f["vy"], p=f["p"])
    assert one["iters"] == 1
    rx, ry, rp, _ = o.residual(f["vx"], f["vy"], f["p"])
    zx, zy = o.vcycle(rx, ry, np.zeros_like(rx), np.zeros_like(ry))  # V-cycle from 0 on r_v
    _, _, dz = o.apply_operator(zx, zy, np.zeros_like(rp))          # D z_v
    zp = 1.0 * f["eta_p"] * (rp - dz)
    px = f["p"] + zp
    px -= px.mean()
    assert rel(one["vx"], f["vx"] + zx) <= 1e-13
    assert rel(one["vy"], f["vy"] + zy) <= 1e-13
    assert rel(one["p"], px) <= 1e-13


def test_gcr_energy_history_converges_faster_than_uzawa():
    w = workload("solcx", 64, 64)
    res = {}
    for accel in (0, 1):
        o = Oracle(64, 64, omega_v=0.6, alpha_p=1.0, accel=accel)
        o.set_viscosity(w["eta_b"], w["eta_p"])
        o.set_density(w["rho_b"])
        o.set_gravity(0.0, 1.0)
        res[accel] = o.solve(1e-8)
        assert res[accel]["status"] == 0
    assert res[1]["iters"] < res[0]["iters"]
    assert rel(res[1]["vx"], res[0]["vx"]) < 1e-6
