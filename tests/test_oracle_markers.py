"""Pins of the marker-in-cell oracle (oracle/markers_oracle.c) against
what the paper and the mathematics fix -- none of them re-types the oracle's formulas:

* marker -> grid: brute force with the HAT-FUNCTION form of the bilinear
  weight, w = max(0, 1-|x-x_n|/dx) max(0, 1-|y-y_n|/dy), over every (node, marker) pair
  (no reference-node search at all); a marker on a node gives weight 1 there and 0 to its
  neighbours; constants are reproduced; empty nodes agree;
* grid -> marker: the same hat-function brute force over every node of
  padded arrays whose mirror rows/columns are built here from the BC definition
  (free slip +, no slip -); linear fields are reproduced exactly;
* advection: on a linear field the RK methods reduce to their stability
  polynomials (Euler 1+z, Heun 1+z+z^2/2, RK4 sum_{k<=4} z^k/k!, z = a dt) -- closed forms;
  on a rigid rotation the error after a full turn falls as dt^1, dt^2, dt^4;
* time step: closed form incl. the zero-velocity case.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from synth.fields import markers


def hat(d, h):
    return np.maximum(0.0, 1.0 - np.abs(d) / h)


def brute_m2g(xn, yn, xm, ym, phi, dx, dy):
    """Dense (nodes x markers) weighted average with hat weights."""
    w = hat(xn.reshape(-1, 1) - xm.reshape(1, -1), dx) * hat(yn.reshape(-1, 1) - ym.reshape(1, -1), dy)
    sw = w.sum(axis=1)
    val = np.where(sw > 0, (w * phi.reshape(1, -1)).sum(axis=1) / np.where(sw > 0, sw, 1.0), 0.0)
    return val, sw


def node_xy(kind, nx, ny, Lx, Ly):
    dx, dy = Lx / nx, Ly / ny
    if kind == "b":
        y, x = np.meshgrid(np.arange(ny + 1) * dy, np.arange(nx + 1) * dx, indexing="ij")
    else:
        y, x = np.meshgrid((np.arange(ny) + 0.5) * dy, (np.arange(nx) + 0.5) * dx, indexing="ij")
    return x.ravel(), y.ravel()


@pytest.mark.parametrize("nx,ny,Lx,Ly,nm", [(8, 6, 1.0, 1.0, 400), (5, 7, 2.0, 0.7, 60), (3, 2, 1.0, 3.0, 9)])
def test_m2g_brute_force(nx, ny, Lx, Ly, nm):
    rng = np.random.default_rng(nx * 100 + ny)
    xm = rng.random(nm) * Lx
    ym = rng.random(nm) * Ly
    xm[:3] = [0.0, Lx, Lx / nx * 2]            # walls and a node line
    ym[:3] = [Ly, 0.0, Ly / ny]
    eta = 10.0 ** rng.uniform(-3, 3, nm)
    rho = rng.normal(size=nm)
    eb, ep, rb, ne = O.markers_to_grid(nx, ny, Lx, Ly, xm, ym, eta, rho)
    dx, dy = Lx / nx, Ly / ny
    xb, yb = node_xy("b", nx, ny, Lx, Ly)
    xp, yp = node_xy("p", nx, ny, Lx, Ly)
    reb, swb = brute_m2g(xb, yb, xm, ym, eta, dx, dy)
    rrb, _ = brute_m2g(xb, yb, xm, ym, rho, dx, dy)
    rep, swp = brute_m2g(xp, yp, xm, ym, eta, dx, dy)
    np.testing.assert_allclose(eb.ravel(), reb, rtol=1e-12, atol=0)
    np.testing.assert_allclose(rb.ravel(), rrb, rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(ep.ravel(), rep, rtol=1e-12, atol=0)
    assert ne == int((swb == 0).sum() + (swp == 0).sum())


def test_m2g_marker_on_node():
    nx, ny = 6, 4
    xm, ym = np.array([2 / 6]), np.array([3 / 4])   # basic node (3, 2)
    eb, ep, rb, ne = O.markers_to_grid(nx, ny, 1.0, 1.0, xm, ym, np.array([7.0]), np.array([-2.5]))
    assert eb[3, 2] == 7.0 and rb[3, 2] == -2.5
    eb[3, 2] = 0.0
    assert not eb.any()
    # P nodes: the marker sits on the corner of four P cells -> weight 1/4 to each, value 7
    assert np.count_nonzero(ep) == 4 and np.all(ep[2:4, 1:3] == 7.0)
    assert ne == (7 * 5 - 1) + (24 - 4)


@pytest.mark.parametrize("order", ["cell", "shuffled"])
def test_m2g_constant_and_lattice(order):
    nx, ny = 16, 12
    m = markers(nx, ny, 1.0, 1.0, per_side=4, seed=3, order=order, props="block")
    c = np.full(m["xm"].shape, 3.25)
    eb, ep, rb, ne = O.markers_to_grid(nx, ny, 1.0, 1.0, m["xm"], m["ym"], c, -c)
    assert ne == 0                                  # 16 markers per cell leave no node empty
    np.testing.assert_allclose(eb, 3.25, rtol=2e-16 * 64)
    np.testing.assert_allclose(ep, 3.25, rtol=2e-16 * 64)
    np.testing.assert_allclose(rb, -3.25, rtol=2e-16 * 64)


def padded_velocity(nx, ny, bc, vx, vy):
    """Node arrays WITH mirror rows/columns built from the BC definition,
    and their positions: vx rows -1..ny, vy columns -1..nx."""
    sW, sE, sN, sS = [1.0 if b == 0 else -1.0 for b in bc]
    ux = np.zeros((ny + 2, nx + 1))
    ux[1:-1, 1:-1] = vx[:, 1:-1]                   # walls (cols 0, nx) stay 0
    ux[0, :] = sN * ux[1, :]
    ux[-1, :] = sS * ux[-2, :]
    uy = np.zeros((ny + 1, nx + 2))
    uy[1:-1, 1:-1] = vy[1:-1, :]
    uy[:, 0] = sW * uy[:, 1]
    uy[:, -1] = sE * uy[:, -2]
    dx, dy = 1.0 / nx, 1.0 / ny
    yx, xx = np.meshgrid((np.arange(-1, ny + 1) + 0.5) * dy, np.arange(nx + 1) * dx, indexing="ij")
    yy, xy = np.meshgrid(np.arange(ny + 1) * dy, (np.arange(-1, nx + 1) + 0.5) * dx, indexing="ij")
    return (ux, xx, yx), (uy, xy, yy)


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0)])
def test_g2m_brute_force(bc):
    nx, ny = 7, 5
    rng = np.random.default_rng(11)
    vx = rng.normal(size=(ny, nx + 1))
    vy = rng.normal(size=(ny + 1, nx))
    nm = 500
    xm, ym = rng.random(nm), rng.random(nm)
    xm[:4] = [0.0, 1.0, 0.0, 1.0]
    ym[:4] = [0.0, 1.0, 1.0, 0.0]
    um, vm = O.grid_to_markers(nx, ny, 1.0, 1.0, bc, xm, ym, vx, vy)
    (ux, xx, yx), (uy, xy, yy) = padded_velocity(nx, ny, bc, vx, vy)
    dx, dy = 1.0 / nx, 1.0 / ny
    wx = hat(xm.reshape(-1, 1) - xx.reshape(1, -1), dx) * hat(ym.reshape(-1, 1) - yx.reshape(1, -1), dy)
    wy = hat(xm.reshape(-1, 1) - xy.reshape(1, -1), dx) * hat(ym.reshape(-1, 1) - yy.reshape(1, -1), dy)
    np.testing.assert_allclose(wx.sum(1), 1.0, rtol=1e-14)   # every marker is covered once
    np.testing.assert_allclose(um, wx @ ux.ravel(), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(vm, wy @ uy.ravel(), rtol=1e-12, atol=1e-13)


def test_g2m_linear_exact():
    nx, ny = 10, 8
    dx, dy = 1.0 / nx, 1.0 / ny
    jx = np.arange(nx + 1) * dx
    iy = (np.arange(ny) + 0.5) * dy
    vx = 0.3 + 1.7 * jx[None, :] - 0.9 * iy[:, None]
    vy = -0.2 + 0.4 * ((np.arange(nx) + 0.5) * dx)[None, :] + 2.1 * (np.arange(ny + 1) * dy)[:, None]
    rng = np.random.default_rng(5)
    xm = dx + rng.random(300) * (1 - 2 * dx)        # away from the wall nodes and mirrors
    ym = dy + rng.random(300) * (1 - 2 * dy)
    um, vm = O.grid_to_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy)
    np.testing.assert_allclose(um, 0.3 + 1.7 * xm - 0.9 * ym, rtol=0, atol=1e-14)
    np.testing.assert_allclose(vm, -0.2 + 0.4 * xm + 2.1 * ym, rtol=0, atol=1e-14)


def test_g2m_wall_mirrors():
    """Free slip: vx constant across the half cell at the top wall; no slip: vx -> 0 at the wall."""
    nx, ny = 4, 4
    vx = np.ones((ny, nx + 1))
    vy = np.zeros((ny + 1, nx))
    xm, ym = np.array([0.5, 0.5]), np.array([0.0, 0.05])
    um, _ = O.grid_to_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy)
    np.testing.assert_allclose(um, [1.0, 1.0], rtol=1e-15)
    um, _ = O.grid_to_markers(nx, ny, 1.0, 1.0, (0, 0, 1, 0), xm, ym, vx, vy)
    np.testing.assert_allclose(um, [0.0, 0.05 / 0.125], atol=1e-15)   # linear to 0 at y = 0


def linear_field(nx, ny, a, xc, yc):
    dx, dy = 1.0 / nx, 1.0 / ny
    vx = np.repeat((a * (np.arange(nx + 1) * dx - xc))[None, :], ny, axis=0)
    vy = np.repeat((-a * (np.arange(ny + 1) * dy - yc))[:, None], nx, axis=1)
    return vx, vy


@pytest.mark.parametrize("scheme,poly", [
    ("euler", lambda z: 1 + z),
    ("heun", lambda z: 1 + z + z * z / 2),
    ("rk4", lambda z: 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24)])
def test_advect_stability_polynomial(scheme, poly):
    nx, ny, a, xc, yc = 16, 16, 0.8, 0.5, 0.5
    vx, vy = linear_field(nx, ny, a, xc, yc)
    rng = np.random.default_rng(2)
    xm = 0.3 + 0.4 * rng.random(200)
    ym = 0.3 + 0.4 * rng.random(200)
    for dt in (0.05, 0.2):
        x1, y1, nc = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy, dt, scheme)
        assert nc == 0
        np.testing.assert_allclose(x1 - xc, (xm - xc) * poly(a * dt), rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(y1 - yc, (ym - yc) * poly(-a * dt), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("scheme", ["euler", "heun", "rk4"])
def test_advect_trivial(scheme):
    nx, ny = 8, 8
    vx = np.full((ny, nx + 1), 0.7)
    vy = np.full((ny + 1, nx), -0.3)
    rng = np.random.default_rng(9)
    xm = 0.2 + 0.6 * rng.random(50)
    ym = 0.2 + 0.6 * rng.random(50)
    x0, y0, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy, 0.0, scheme)
    assert np.array_equal(x0, xm) and np.array_equal(y0, ym)          # dt = 0 -> identity
    x1, y1, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy, 0.1, scheme)
    np.testing.assert_allclose(x1, xm + 0.07, rtol=0, atol=1e-15)    # uniform velocity
    np.testing.assert_allclose(y1, ym - 0.03, rtol=0, atol=1e-15)


def test_advect_rotation_order():
    """Rigid rotation about the centre (exact in the bilinear interpolant away from the walls):
    error after one turn ~ dt^p with p = 1, 2, 4."""
    nx = ny = 32
    dx = dy = 1.0 / nx
    om = 2 * math.pi
    vx = np.repeat((-om * ((np.arange(ny) + 0.5) * dy - 0.5))[:, None], nx + 1, axis=1)
    vy = np.repeat((om * ((np.arange(nx) + 0.5) * dx - 0.5))[None, :], ny + 1, axis=0)
    xm, ym = np.array([0.75]), np.array([0.5])
    errs = {}
    for scheme in ("euler", "heun", "rk4"):
        e = []
        for nsteps in (64, 128):
            x, y = xm.copy(), ym.copy()
            for _ in range(nsteps):
                x, y, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), x, y, vx, vy, 1.0 / nsteps, scheme)
            e.append(math.hypot(x[0] - 0.75, y[0] - 0.5))
        errs[scheme] = e
    for scheme, p in (("euler", 1), ("heun", 2), ("rk4", 4)):
        ratio = errs[scheme][0] / errs[scheme][1]
        assert 0.8 * 2 ** p < ratio < 1.25 * 2 ** p, (scheme, errs[scheme])
    assert errs["rk4"][1] < errs["heun"][1] < errs["euler"][1]


def test_advect_clamp():
    nx = ny = 4
    vx = np.full((ny, nx + 1), 5.0)
    vy = np.zeros((ny + 1, nx))
    x1, y1, nc = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), np.array([0.5, 0.5]), np.array([0.5, 0.5]),
                                  vx, vy, 1.0, "euler")
    assert nc == 2 and np.all(x1 == 1.0) and np.all(y1 == 0.5)


def test_timestep_closed_form():
    nx, ny = 8, 4
    vx = np.zeros((ny, nx + 1))
    vy = np.zeros((ny + 1, nx))
    assert O.marker_timestep(nx, ny, 1.0, 1.0, vx, vy, 0.5, 3.0) == 3.0
    vx[2, 3] = -2.0
    vx[1, 0] = 100.0                                   # wall entry: ignored
    assert O.marker_timestep(nx, ny, 1.0, 1.0, vx, vy, 0.5, 3.0) == 0.5 * (1 / 8) / 2.0
    vy[2, 1] = 4.0
    assert O.marker_timestep(nx, ny, 1.0, 1.0, vx, vy, 0.5, 3.0) == min(0.5 * (1 / 8) / 2, 0.5 * (1 / 4) / 4)
    assert O.marker_timestep(nx, ny, 1.0, 1.0, vx, vy, 0.5, 1e-3) == 1e-3


# ---------------------------------------------------------------- LPI (R32)
@pytest.mark.parametrize("scheme", ["lpi2", "lpi3"])
def test_lpi_linear_field_is_heun(scheme):
    """On a linear field J is exact and H = 0: both orders give 1 + z + z^2/2 (= Heun)."""
    nx, ny, a, xc, yc = 16, 16, 0.8, 0.5, 0.5
    vx, vy = linear_field(nx, ny, a, xc, yc)
    rng = np.random.default_rng(12)
    xm = 0.3 + 0.4 * rng.random(100)
    ym = 0.3 + 0.4 * rng.random(100)
    for dt in (0.05, 0.2):
        x1, y1, nc = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy, dt, scheme)
        z = a * dt
        np.testing.assert_allclose(x1 - xc, (xm - xc) * (1 + z + z * z / 2), rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(y1 - yc, (ym - yc) * (1 - z + z * z / 2), rtol=1e-12, atol=1e-15)


def test_lpi_bilinear_field_closed_form():
    """v = (c X Y, d) with X = x - xc, Y = y - yc is reproduced exactly by the bilinear
    interpolant: J = [[cY, cX], [0, 0]], d2vx/dxdy = c, so (Eq. lpi_update)
    x' = x + dt cXY + dt^2/2 (c^2 X Y^2 + c d X) + dt^3/6 (2 c^2 d X Y),  y' = y + dt d."""
    nx = ny = 20
    c, d, xc, yc = 1.3, 0.4, 0.45, 0.55
    dx = dy = 1.0 / nx
    X = np.arange(nx + 1) * dx - xc
    Y = (np.arange(ny) + 0.5) * dy - yc
    vx = c * Y[:, None] * X[None, :]
    vy = np.full((ny + 1, nx), d)
    rng = np.random.default_rng(13)
    xm = 0.2 + 0.6 * rng.random(200)
    ym = 0.2 + 0.5 * rng.random(200)
    dt = 0.05
    Xm, Ym = xm - xc, ym - yc
    for scheme, k3 in (("lpi2", 0.0), ("lpi3", 1.0)):
        x1, y1, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xm, ym, vx, vy, dt, scheme)
        ex = xm + dt * c * Xm * Ym + dt ** 2 / 2 * (c * c * Xm * Ym ** 2 + c * d * Xm) + \
            k3 * dt ** 3 / 6 * (2 * c * c * d * Xm * Ym)
        np.testing.assert_allclose(x1, ex, rtol=0, atol=1e-14)
        np.testing.assert_allclose(y1, ym + dt * d, rtol=0, atol=1e-15)


def test_lpi_rotation_second_order():
    nx = ny = 32
    dx = dy = 1.0 / nx
    om = 2 * math.pi
    vx = np.repeat((-om * ((np.arange(ny) + 0.5) * dy - 0.5))[:, None], nx + 1, axis=1)
    vy = np.repeat((om * ((np.arange(nx) + 0.5) * dx - 0.5))[None, :], ny + 1, axis=0)
    e = []
    for nsteps in (64, 128):
        x, y = np.array([0.75]), np.array([0.5])
        for _ in range(nsteps):
            x, y, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), x, y, vx, vy, 1.0 / nsteps, "lpi2")
        e.append(math.hypot(x[0] - 0.75, y[0] - 0.5))
    assert 0.8 * 4 < e[0] / e[1] < 1.25 * 4, e
