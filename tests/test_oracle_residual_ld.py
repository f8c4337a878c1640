"""Pin of the oracle's extended-precision residual (oracle_residual_ld, reading R34).

It evaluates the residual r = f - L v - G p, r_p = -D v and the energy residual E
 of oracle_residual in long double.  Pinned here against an independent
numpy evaluation in np.longdouble of the STRESS form of the operator (PAPER.md:643-662:
sigma_xx on P nodes, sigma_xy on basic nodes, differences of stresses -- not the Listing's
coefficients the oracle's x row uses), with the mirror / wall boundary nodes of PAPER.md:613:
  * on O(1) residuals both equal the FP64 oracle to its rounding (a dropped term, a wrong
    sign or a transposed index would show at O(1));
  * at a converged solution (E ~ 1e-8, where the Listing form's FP64 evaluation cancels terms
    ~h^-2 larger than the residual) the long-double E agrees with numpy's to 1e-9 relative,
    closer than the FP64 oracle's E does.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from synth.fields import parity_fields, workload

LD = np.longdouble


def stress_residual_ld(nx, ny, Lx, Ly, bc, gx, gy, eta_b, eta_p, rho_b, vx, vy, p):
    """E of (vx, vy, p) in np.longdouble from the stress differences (bc = W, E, N, S; 0 free
    slip (mirror sign +1), 1 no slip (-1)); returns (rx, ry, rp, E)."""
    sW, sE, sN, sS = (1.0 if b == 0 else -1.0 for b in bc)
    dx, dy = LD(Lx) / nx, LD(Ly) / ny
    eb, ep, rb = (np.asarray(a, LD) for a in (eta_b, eta_p, rho_b))
    # padded velocities: vx rows 0..ny+1 (mirrors 0, ny+1), columns 0..nx (walls 0, nx = 0);
    # vy rows 0..ny (walls), columns 0..nx+1 (mirrors)
    X = np.zeros((ny + 2, nx + 1), LD)
    X[1:ny + 1] = np.asarray(vx, LD)
    X[:, 0] = X[:, nx] = 0
    X[0, 1:nx] = sN * X[1, 1:nx]
    X[ny + 1, 1:nx] = sS * X[ny, 1:nx]
    Y = np.zeros((ny + 1, nx + 2), LD)
    Y[:, 1:nx + 1] = np.asarray(vy, LD)
    Y[0, :] = Y[ny, :] = 0
    Y[1:ny, 0] = sW * Y[1:ny, 1]
    Y[1:ny, nx + 1] = sE * Y[1:ny, nx]
    P = np.asarray(p, LD)
    # stresses: sxx, syy on P(i, j) (cells, 0-based rows i = 0..ny-1); sxy on basic nodes (i, j)
    sxx = 2 * ep * (X[1:ny + 1, 1:] - X[1:ny + 1, :-1]) / dx                  # ny x nx
    syy = 2 * ep * (Y[1:, 1:nx + 1] - Y[:-1, 1:nx + 1]) / dy                  # ny x nx
    sxy = eb * ((X[1:, :] - X[:-1, :]) / dy + (Y[:, 1:] - Y[:, :-1]) / dx)    # (ny+1) x (nx+1)
    # x rows: vx(i, j), i = 1..ny, j = 1..nx-1 (padded); y rows: vy(i, j), i = 1..ny-1, j = 1..nx
    Lxv = (sxx[:, 1:] - sxx[:, :-1]) / dx + (sxy[1:, 1:nx] - sxy[:-1, 1:nx]) / dy
    Lyv = (syy[1:, :] - syy[:-1, :]) / dy + (sxy[1:ny, 1:] - sxy[1:ny, :-1]) / dx
    Gx = (P[:, :-1] - P[:, 1:]) / dx
    Gy = (P[:-1, :] - P[1:, :]) / dy
    fx = -LD(gx) * (rb[:-1, 1:nx] + rb[1:, 1:nx]) / 2
    fy = -LD(gy) * (rb[1:ny, :-1] + rb[1:ny, 1:]) / 2
    rx = fx - (Lxv + Gx)
    ry = fy - (Lyv + Gy)
    rp = -((X[1:ny + 1, 1:] - X[1:ny + 1, :-1]) / dx + (Y[1:, 1:nx + 1] - Y[:-1, 1:nx + 1]) / dy)
    # diag(-L) with the mirror folding (reading R5)
    ax = -(eb[:-1, 1:nx] + eb[1:, 1:nx]) / dy ** 2 - 2 * (ep[:, :-1] + ep[:, 1:]) / dx ** 2
    ax[0] += sN * eb[0, 1:nx] / dy ** 2
    ax[-1] += sS * eb[ny, 1:nx] / dy ** 2
    ay = -2 * (ep[:-1, :] + ep[1:, :]) / dy ** 2 - (eb[1:ny, :-1] + eb[1:ny, 1:]) / dx ** 2
    ay[:, 0] += sW * eb[1:ny, 0] / dx ** 2
    ay[:, -1] += sE * eb[1:ny, nx] / dx ** 2
    c = 2 / dx ** 2 + 2 / dy ** 2
    sv = (rx ** 2 / -ax).sum() + (ry ** 2 / -ay).sum()
    sp = (rp ** 2 * ep / c).sum()
    sf = (fx ** 2 / -ax).sum() + (fy ** 2 / -ay).sum()
    return rx, ry, rp, np.sqrt((sv + sp) / sf)


def setup(name, n):
    w = workload(name, n, n)
    o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(w["gx"], w["gy"])
    return o, w


def ref(w, n, v):
    return stress_residual_ld(n, n, w["Lx"], w["Ly"], w["bc"], w["gx"], w["gy"], w["eta_b"], w["eta_p"],
                              w["rho_b"], *v)


@pytest.mark.parametrize("name,n", [("layered", 48), ("random", 40), ("block", 32), ("solcx", 36)])
def test_residual_ld_equals_stress_form_on_O1_residuals(name, n):
    o, w = setup(name, n)
    f = parity_fields(n, n)
    v = (f["vx"], f["vy"], f["p"])
    e64 = o.residual(*v)
    eld = o.residual_ld(*v)
    enp = ref(w, n, v)
    # the wall columns of rx / rows of ry (not unknowns) are zero in the oracle's arrays
    cut = (lambda a: a[:, 1:n], lambda a: a[1:n, :], lambda a: a)
    for k in range(3):
        t = np.asarray(enp[k], np.float64)
        for got in (e64[k], eld[k]):
            assert np.linalg.norm(cut[k](got) - t) <= 1e-13 * np.linalg.norm(t), (name, k)
    assert abs(eld[3] - float(enp[3])) <= 1e-15 * float(enp[3])
    assert abs(e64[3] - float(enp[3])) <= 1e-13 * float(enp[3])


@pytest.mark.parametrize("name,n", [("random", 256), ("layered", 128)])
def test_residual_ld_at_a_converged_solution(name, n):
    o, w = setup(name, n)
    r = o.solve(1e-8)
    assert r["status"] == 0
    v = (r["vx"], r["vy"], r["p"])
    e_np = float(ref(w, n, v)[3])
    e_ld = o.residual_ld(*v)[3]
    e_64 = o.residual(*v)[3]
    assert e_np <= 1.01e-8
    assert abs(e_ld - e_np) <= 1e-9 * e_np, (e_ld, e_np)
    assert abs(e_ld - e_np) < abs(e_64 - e_np) or abs(e_64 - e_np) <= 1e-12 * e_np, (e_64, e_ld, e_np)
