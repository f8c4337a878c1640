"""Oracle pins for SURVEY §8(f) NEXT-1: viscosity rescaling and
the lithostatic initial pressure.

Pinned against closed forms and the discrete hydrostatic balance, not against the oracle:
  * lithostatic p of a constant / two-layer density = the analytic column integral at the
    P-node depths; g = 0 gives 0; with a laterally uniform density (v = 0, p = p_litho)
    the discrete momentum residual vanishes;
  * the rescaled viscosity is (1 - theta) eta_min + theta eta on every fine node (theta =
    0: uniform eta_min on every level; theta = 1: the caller's field, bit for bit);
  * the staged solve reaches the same fixed point as the plain one (the last stage IS the
    problem), with at least (stages - 1) x theta_every iterations.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError
from synth.fields import workload


def make(n, w, **kw):
    o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **kw)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(w["gx"], w["gy"])
    return o


def column_problem(nx, ny, rho_rows, g=1.0):
    """eta = 1, rho_B(i, j) = rho_rows[i] (laterally uniform), free slip"""
    eb, ep = np.ones((ny + 1, nx + 1)), np.ones((ny, nx))
    rho = np.repeat(np.asarray(rho_rows, float)[:, None], nx + 1, axis=1)
    o = Oracle(nx, ny, 1.0, 2.0, (0, 0, 0, 0))
    o.set_viscosity(eb, ep)
    o.set_density(rho)
    o.set_gravity(0.0, g)
    return o


def test_lithostatic_constant_density():
    nx, ny, rho, g = 6, 10, 3.3, 9.81
    o = column_problem(nx, ny, [rho] * (ny + 1), g)
    dy = 2.0 / ny
    depth = (np.arange(ny) + 0.5) * dy  # P-node depths below the top wall
    np.testing.assert_allclose(o.lithostatic(), np.repeat((rho * g * depth)[:, None], nx, axis=1), rtol=1e-14)


def test_lithostatic_two_layer_is_piecewise_linear():
    nx, ny, k = 4, 12, 5  # interface on basic row k (depth k dy)
    r1, r2, g = 1.0, 2.5, 2.0
    rows = [r1] * k + [(r1 + r2) / 2] + [r2] * (ny - k)
    o = column_problem(nx, ny, rows, g)
    dy = 2.0 / ny
    y = (np.arange(ny) + 0.5) * dy
    yk = k * dy
    exact = np.where(y <= yk, r1 * g * y, r1 * g * yk + r2 * g * (y - yk))
    np.testing.assert_allclose(o.lithostatic()[:, 0], exact, rtol=1e-13)


def test_lithostatic_zero_gravity():
    o = column_problem(5, 7, np.linspace(1, 2, 8), g=0.0)
    assert np.all(o.lithostatic() == 0.0)


def test_lithostatic_is_discrete_hydrostatic_equilibrium():
    """laterally uniform rho: (v = 0, p_litho) has zero momentum residual (P5)"""
    nx, ny = 8, 16
    rows = 1.0 + 0.5 * np.sin(np.linspace(0, 3, ny + 1))
    o = column_problem(nx, ny, rows, 1.7)
    p = o.lithostatic()
    rx, ry, rp, E = o.residual(np.zeros((ny, nx + 1)), np.zeros((ny + 1, nx)), p)
    scale = np.abs(p).max()
    assert np.abs(rx).max() <= 1e-13 * scale and np.abs(ry).max() <= 1e-13 * scale * ny
    assert E <= 1e-13  # E is a relative norm: rounding level


def test_blend_viscosity_endpoints_and_midpoint():
    n = 16
    rng = np.random.default_rng(5)
    eb = 10 ** rng.uniform(0, 2, (n + 1, n + 1))
    ep = 10 ** rng.uniform(0, 2, (n, n))
    eb[3, 4], ep[2, 2] = 1.0, 3.0  # eta_min = 1 (on a basic node), a P node of 3
    o = Oracle(n, n, 1.0, 1.0, (0, 1, 0, 1), coarse_min=4)
    o.set_viscosity(eb, ep)
    o.blend_viscosity(0.0)
    for lev in range(o.nlev):
        b, p = o.get_viscosity(lev)
        assert np.all(b == 1.0) and np.all(p == 1.0), lev
    o.blend_viscosity(0.5)
    b, p = o.get_viscosity(0)
    assert p[2, 2] == 2.0 and b[3, 4] == 1.0
    np.testing.assert_allclose(b, 0.5 + 0.5 * eb, rtol=1e-15)
    o.blend_viscosity(1.0)
    b, p = o.get_viscosity(0)
    assert np.array_equal(b, eb) and np.array_equal(p, ep)
    with pytest.raises(OracleError):
        o.blend_viscosity(1.5)


@pytest.mark.parametrize("accel", [0, 1])
def test_staged_solve_reaches_the_same_fixed_point(accel):
    n = 32
    w = workload("block", n, n)
    kw = dict(omega_v=0.6, alpha_p=1.0, accel=accel, gcr_restart=20)
    plain = make(n, w, **kw).solve(1e-11)
    staged = make(n, w, theta_step=0.25, theta_every=10, **kw).solve(1e-11)
    assert plain["status"] == 0 and staged["status"] == 0
    assert staged["iters"] >= 4 * 10
    for k in ("vx", "vy", "p"):
        d = np.linalg.norm(staged[k] - plain[k]) / np.linalg.norm(plain[k])
        assert d <= 1e-7, (k, d)


def test_staged_solve_budget_and_errors():
    n = 16
    w = workload("layered", n, n)
    r = make(n, w, omega_v=0.6, alpha_p=1.0, theta_step=0.5, theta_every=7, max_iter=10).solve(1e-12)
    assert r["iters"] == 10 and r["status"] == 1  # budget spent inside the stages
    with pytest.raises(OracleError):
        Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), theta_step=1.5)
    with pytest.raises(OracleError):
        Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), theta_every=0)
