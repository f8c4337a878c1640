"""Pins of the oracle's operator, residual and energy norm (no GPU).

P1  operator == dense assembly from the stress formulas (tests/dense.py), symmetry, G = D^T
P11 energy-norm examples, E = 0 at the exact solution
P5  hydrostatic column: force sign + pressure recursion (reading R4)
P16 wall / unused entries never influence outputs
"""
import json
import os

import numpy as np
import pytest

from dense import Dense
from oracle.oracle import Oracle
from synth.fields import parity_fields

BCS = [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0), (1, 0, 0, 1)]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("nx,ny,Lx,Ly", [(4, 4, 1.0, 1.0), (8, 8, 1.0, 1.0), (6, 10, 2.0, 1.5), (5, 3, 1.0, 0.7)])
@pytest.mark.parametrize("bc", BCS)
def test_operator_matches_dense_stress_assembly(nx, ny, Lx, Ly, bc):
    f = parity_fields(nx, ny)
    o = Oracle(nx, ny, Lx, Ly, bc, coarse_direct=0)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    ax, ay, ap = o.apply_operator(f["vx"], f["vy"], f["p"])
    d = Dense(nx, ny, Lx, Ly, bc, f["eta_b"], f["eta_p"])
    u = d.pack(f["vx"], f["vy"], f["p"])
    ex, ey, ep = d.unpack(d.A @ u)
    assert rel(ax, ex) <= 1e-13
    assert rel(ay, ey) <= 1e-13
    assert rel(ap, ep) <= 1e-13
    # walls written as zero
    assert np.all(ax[:, 0] == 0) and np.all(ax[:, -1] == 0)
    assert np.all(ay[0, :] == 0) and np.all(ay[-1, :] == 0)


@pytest.mark.parametrize("bc", BCS)
def test_dense_assembly_is_symmetric_saddle(bc):
    """L symmetric, G = D^T (derived) -- pins the dense assembly itself."""
    f = parity_fields(7, 6)
    d = Dense(7, 6, 1.3, 0.9, bc, f["eta_b"], f["eta_p"])
    assert np.allclose(d.L, d.L.T, rtol=0, atol=1e-12 * np.abs(d.L).max())
    assert np.allclose(d.G, d.D.T, rtol=0, atol=1e-14 * np.abs(d.G).max())
    # -L positive definite (L negative definite)
    assert np.linalg.eigvalsh(-0.5 * (d.L + d.L.T)).min() > 0


def test_listing_coefficients_constant_viscosity():
    """eta = 1, dx = dy = 1: centre coefficient of an interior vx row is -6
    and the 9 velocity coefficients are those of Listing vx_op_point."""
    nx = ny = 6
    d = Dense(nx, ny, 6.0, 6.0, (0, 0, 0, 0), np.ones((7, 7)), np.ones((6, 6)))
    k = d.vx_idx.index((3, 3))
    row = d.A[k]
    vxk = lambda i, j: d.vx_idx.index((i, j))
    vyk = lambda i, j: d.nvx + d.vy_idx.index((i, j))
    assert row[vxk(3, 3)] == pytest.approx(-6.0)
    assert row[vxk(3, 2)] == pytest.approx(2.0) and row[vxk(3, 4)] == pytest.approx(2.0)
    assert row[vxk(2, 3)] == pytest.approx(1.0) and row[vxk(4, 3)] == pytest.approx(1.0)
    assert row[vyk(2, 3)] == pytest.approx(1.0) and row[vyk(3, 3)] == pytest.approx(-1.0)
    assert row[vyk(2, 4)] == pytest.approx(-1.0) and row[vyk(3, 4)] == pytest.approx(1.0)
    assert np.count_nonzero(row[: d.nvx + d.nvy]) == 9


def test_transposition_symmetry():
    """x <-> y transposition of the problem maps the vx rows onto the vy rows."""
    nx, ny = 6, 4
    f = parity_fields(nx, ny)
    o = Oracle(nx, ny, 1.0, 0.8, (0, 1, 1, 0), coarse_direct=0)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    ax, ay, ap = o.apply_operator(f["vx"], f["vy"], f["p"])
    # transposed problem: swap axes, vx <-> vy, bc (W,E,N,S) -> (N,S,W,E)
    t = Oracle(ny, nx, 0.8, 1.0, (1, 0, 0, 1), coarse_direct=0)
    t.set_viscosity(f["eta_b"].T.copy(), f["eta_p"].T.copy())
    bx, by, bp = t.apply_operator(f["vy"].T.copy(), f["vx"].T.copy(), f["p"].T.copy())
    assert rel(bx, ay.T) <= 1e-13
    assert rel(by, ax.T) <= 1e-13
    assert rel(bp, ap.T) <= 1e-13


GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "energy_examples.json")))


def test_schur_surrogate_golden():
    """S~^-1 for a single unit r_p on a 1-cell-wide pressure perturbation, against the
    values of tests/golden/energy_examples.json."""
    for ex in GOLDEN["schur_surrogate"]:
        nx = ny = 6
        o = Oracle(nx, ny, 6 * ex["dx"], 6 * ex["dy"], (0, 0, 0, 0), coarse_direct=0)
        o.set_viscosity(np.ones((7, 7)), ex["eta"] * np.ones((6, 6)))
        o.set_density(np.ones((7, 7)))
        o.set_gravity(0.0, 1.0)
        vx = np.zeros((6, 7))
        vx[2, 3] = ex["dx"]  # r_p = -D v = -1 at P(2,2) and +1 at P(2,3)
        sp = o.energy_sums(vx, np.zeros((7, 6)), np.zeros((6, 6)))[1]
        assert sp == pytest.approx(2 * ex["value"], rel=1e-15)


def test_energy_norm_examples():
    """diag(-L) = 6 and S~^-1 = eta/(2/dx^2+2/dy^2) = 0.25 for eta=1, dx=dy=1."""
    nx = ny = 6
    o = Oracle(nx, ny, 6.0, 6.0, (0, 0, 0, 0), coarse_direct=0)
    o.set_viscosity(np.ones((7, 7)), np.ones((6, 6)))
    # a single unit vy force from a density pair: f_y(i,j) = -(rho(i,j-1)+rho(i,j))/2 with g_y = 1
    rho = np.zeros((7, 7))
    rho[3, 2] = -1.0
    rho[3, 3] = -1.0
    o.set_density(rho)
    o.set_gravity(0.0, 1.0)
    z = lambda k: o.zeros(k)
    s = o.energy_sums(z("vx"), z("vy"), z("p"))
    # f nonzero at vy(3,2), vy(3,3) (value 0.5) and vy(3,4) (value 1... ) -> compute from layout
    _, ry, _, _ = o.residual(z("vx"), z("vy"), z("p"))
    # interior vy rows have d = 6 (constant eta, dx = dy = 1)
    assert s[2] == pytest.approx(np.sum(ry ** 2) / GOLDEN["diag_minus_L_eta1_h1"], rel=1e-15)
    assert s[0] == pytest.approx(s[2], rel=1e-15)
    # single vx perturbation -> r_p = -Dv = -/+1 at two P nodes -> Sp = 2 * 0.25
    vx = z("vx")
    vx[2, 3] = 1.0
    s = o.energy_sums(vx, z("vy"), z("p"))
    assert s[1] == pytest.approx(0.5, rel=1e-15)
    # eta = 4 -> 1.0 per unit r_p^2 ; dx = dy = 2, eta = 1 -> 1.0
    o4 = Oracle(nx, ny, 6.0, 6.0, (0, 0, 0, 0), coarse_direct=0)
    o4.set_viscosity(np.ones((7, 7)), 4 * np.ones((6, 6)))
    o4.set_density(rho)
    assert o4.energy_sums(vx, z("vy"), z("p"))[1] == pytest.approx(2.0, rel=1e-15)
    o2 = Oracle(nx, ny, 12.0, 12.0, (0, 0, 0, 0), coarse_direct=0)
    o2.set_viscosity(np.ones((7, 7)), np.ones((6, 6)))
    o2.set_density(rho)
    vx2 = vx * 2.0  # r_p = -Dv = -/+ 2/2 = -/+1
    assert o2.energy_sums(vx2, z("vy"), z("p"))[1] == pytest.approx(2.0, rel=1e-15)


@pytest.mark.parametrize("bc", BCS)
def test_residual_zero_at_dense_solution(bc):
    nx, ny = 8, 6
    f = parity_fields(nx, ny, log_contrast=1.5)
    o = Oracle(nx, ny, 1.0, 0.75, bc, coarse_direct=0)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.3, 1.0)
    d = Dense(nx, ny, 1.0, 0.75, bc, f["eta_b"], f["eta_p"])
    u = d.solve_bordered(d.force(f["rho_b"], 0.3, 1.0))
    vx, vy, p = d.unpack(u)
    rx, ry, rp, E = o.residual(vx, vy, p)
    assert E <= 1e-12
    # E = res_v / ||f|| when r_p = 0
    vz = np.zeros_like(vx)
    rx, ry, rp, E = o.residual(vz, np.zeros_like(vy), np.zeros_like(p))
    assert E == pytest.approx(1.0, rel=1e-14)


def test_hydrostatic_column():
    """P5: laterally uniform rho(y), v = 0, p(i+1) = p(i) + g dy rho_vy(i) -> residual == 0."""
    nx, ny, Ly = 8, 10, 2.0
    dy = Ly / ny
    rng = np.random.default_rng(5)
    col = rng.uniform(1.0, 3.0, ny + 1)
    rho = np.repeat(col[:, None], nx + 1, axis=1)
    o = Oracle(nx, ny, 1.0, Ly, (0, 0, 0, 0))
    o.set_viscosity(10 ** rng.uniform(-1, 1, (ny + 1, nx + 1)), 10 ** rng.uniform(-1, 1, (ny, nx)))
    o.set_density(rho)
    g = 9.81
    o.set_gravity(0.0, g)
    p = np.zeros((ny, nx))
    for i in range(1, ny):
        p[i] = p[i - 1] + g * dy * col[i]  # vy row i sits on basic row i
    p -= p.mean()
    rx, ry, rp, E = o.residual(np.zeros((ny, nx + 1)), np.zeros((ny + 1, nx)), p)
    assert E <= 1e-14
    sol = o.solve(1e-10)
    assert sol["status"] == 0
    assert np.abs(sol["vx"]).max() <= 1e-9 * np.abs(p).max()
    assert rel(sol["p"], p) <= 1e-8


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 1, 1, 1)])
def test_wall_entries_ignored(bc):
    """P16: NaN in the wall-normal entries of the inputs changes no output."""
    nx, ny = 8, 8
    f = parity_fields(nx, ny)
    o = Oracle(nx, ny, 1.0, 1.0, bc)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.0, 1.0)
    a = o.apply_operator(f["vx"], f["vy"], f["p"])
    r = o.residual(f["vx"], f["vy"], f["p"])
    vx, vy = f["vx"].copy(), f["vy"].copy()
    vx[:, 0] = vx[:, -1] = np.nan
    vy[0, :] = vy[-1, :] = np.nan
    b = o.apply_operator(vx, vy, f["p"])
    s = o.residual(vx, vy, f["p"])
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for x, y in zip(r[:3], s[:3]):
        assert np.array_equal(x, y)
    w1 = o.vcycle(f["vx"] * 0 + 1, f["vy"] * 0 + 1, f["vx"], f["vy"])
    w2 = o.vcycle(f["vx"] * 0 + 1, f["vy"] * 0 + 1, vx, vy)
    assert np.array_equal(w1[0], w2[0]) and np.array_equal(w1[1], w2[1])
