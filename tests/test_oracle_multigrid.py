"""Pins of the oracle's multigrid pieces (no GPU).

P6  restriction = row-normalised transpose of the bilinear interpolation weights over
    same-type nodes (reading R6), built here from node positions;
    constants preserved, linears reproduced; prolongation reproduces linears
P7  one Jacobi sweep == x + w C^-1 (b - A x) with the dense matrix and its diagonal C
    (reading R5); RBGS phase-parallel == oracle serial
    (reading R11); Jacobi stability limit (derived: w < 3/4)
a7  coarse viscosity = same restriction applied to eta
a8  coarsest direct solve == dense solve of the mirror-folded L
P8  V-cycle contraction h-independent within +-20%
"""
import numpy as np
import pytest

from dense import Dense
from oracle.oracle import Oracle
from synth.fields import node_coords, parity_fields


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------------ transfers
def interp_weights(kind, nxf, nyf, Lx, Ly):
    """W[f, c] = hat_H(x_f - x_c) hat_H(y_f - y_c) over same-type nodes inside the closed domain
    (unknowns + walls; mirrors excluded), from node coordinates only."""
    nxc, nyc = nxf // 2, nyf // 2
    yf, xf = node_coords(kind, nxf, nyf, Lx, Ly)
    yc, xc = node_coords(kind, nxc, nyc, Lx, Ly)
    Hx, Hy = Lx / nxc, Ly / nyc
    hx = np.maximum(0.0, 1.0 - np.abs(xf[:, None] - xc[None, :]) / Hx)
    hy = np.maximum(0.0, 1.0 - np.abs(yf[:, None] - yc[None, :]) / Hy)
    return hy, hx  # separable factors (fine x coarse) per axis


def expected_restriction(kind, fine, nxf, nyf, Lx, Ly):
    hy, hx = interp_weights(kind, nxf, nyf, Lx, Ly)
    num = hy.T @ fine @ hx
    den = hy.sum(axis=0)[:, None] * hx.sum(axis=0)[None, :]
    return num / den


@pytest.mark.parametrize("kind", ["b", "p", "vx", "vy"])
@pytest.mark.parametrize("nx,ny", [(16, 16), (16, 32), (32, 16)])
def test_restriction_is_rownormalised_transpose(kind, nx, ny):
    rng = np.random.default_rng(7)
    o = Oracle(nx, ny, 1.0, 1.3, coarse_min=4)
    shp = Oracle.shapes(nx, ny)[kind]
    fine = rng.standard_normal(shp)
    if kind == "vx":  # walls carry value 0 but count in the weights (reading R6)
        fine[:, 0] = fine[:, -1] = 0.0
    if kind == "vy":
        fine[0, :] = fine[-1, :] = 0.0
    got = o.restrict(0, kind, fine)
    exp = expected_restriction(kind, fine, nx, ny, 1.0, 1.3)
    if kind == "vx":
        got, exp = got[:, 1:-1], exp[:, 1:-1]
    if kind == "vy":
        got, exp = got[1:-1, :], exp[1:-1, :]
    assert rel(got, exp) <= 1e-14


def test_restriction_interior_weights_full_weighting():
    """Appendix B interior stencils: P-type [1,3,3,1]/8 per axis, basic [1,2,1]/4 per axis."""
    nx = ny = 16
    o = Oracle(nx, ny, coarse_min=4)
    fine = np.zeros((ny, nx))
    fine[8, 8] = 1.0  # P node (user) -> coarse P (4,4) weight (3/8)^2, coarse (5,4)... (1/8)(3/8)
    c = o.restrict(0, "p", fine)
    assert c[4, 4] == pytest.approx((3 / 8) ** 2)
    assert c[3, 4] == pytest.approx((1 / 8) * (3 / 8))
    fb = np.zeros((ny + 1, nx + 1))
    fb[8, 8] = 1.0
    cb = o.restrict(0, "b", fb)
    assert cb[4, 4] == pytest.approx(1 / 4)
    fb[:] = 0
    fb[9, 8] = 1.0
    cb = o.restrict(0, "b", fb)
    assert cb[4, 4] == pytest.approx(1 / 8) and cb[5, 4] == pytest.approx(1 / 8)


@pytest.mark.parametrize("kind", ["b", "p"])
def test_restriction_constants_and_linears(kind):
    nx = ny = 32
    o = Oracle(nx, ny, 1.0, 1.0, coarse_min=4)
    y, x = node_coords(kind, nx, ny, 1.0, 1.0)
    c = o.restrict(0, kind, np.full((y.size, x.size), 3.25))
    assert np.allclose(c, 3.25, rtol=0, atol=1e-14)
    lin = 0.3 + 2.0 * x[None, :] - 1.5 * y[:, None]
    c = o.restrict(0, kind, lin)
    yc, xc = node_coords(kind, nx // 2, ny // 2, 1.0, 1.0)
    exp = 0.3 + 2.0 * xc[None, :] - 1.5 * yc[:, None]
    assert np.allclose(c[1:-1, 1:-1], exp[1:-1, 1:-1], rtol=0, atol=1e-13)


def test_prolongation_reproduces_linears_and_mirrors():
    nx = ny = 16
    o = Oracle(nx, ny, 1.0, 1.0, coarse_min=4)
    yc, xc = node_coords("vx", 8, 8, 1.0, 1.0)
    ex = 1.0 + 0.5 * xc[None, :] + 2.0 * yc[:, None]
    ex[:, 0] = ex[:, -1] = 0.0
    ey = np.zeros((9, 8))
    vx, vy = o.prolong(0, ex, ey, np.zeros((16, 17)), np.zeros((17, 16)))
    yf, xf = node_coords("vx", 16, 16, 1.0, 1.0)
    exp = 1.0 + 0.5 * xf[None, :] + 2.0 * yf[:, None]
    # interior rows/cols away from walls and mirrors: exact
    assert np.allclose(vx[1:-1, 2:-2], exp[1:-1, 2:-2], rtol=0, atol=1e-13)
    # free slip: fine row next to the top wall takes the coarse value (mirror = partner)
    assert vx[0, 4] == pytest.approx(ex[0, 2])
    # no slip: 1/2 of it (linear interpolation to zero at the wall) -- Appendix B
    o2 = Oracle(nx, ny, 1.0, 1.0, bc=(0, 0, 1, 0), coarse_min=4)
    vx2, _ = o2.prolong(0, ex, ey, np.zeros((16, 17)), np.zeros((17, 16)))
    assert vx2[0, 4] == pytest.approx(0.5 * ex[0, 2])


def test_coarse_viscosity_is_restricted_viscosity():
    nx = ny = 32
    f = parity_fields(nx, ny)
    o = Oracle(nx, ny, coarse_min=8)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    eb1, ep1 = o.get_viscosity(1)
    assert rel(eb1, expected_restriction("b", f["eta_b"], nx, ny, 1.0, 1.0)) <= 1e-14
    assert rel(ep1, expected_restriction("p", f["eta_p"], nx, ny, 1.0, 1.0)) <= 1e-14
    eb2, ep2 = o.get_viscosity(2)
    assert rel(ep2, expected_restriction("p", ep1, 16, 16, 1.0, 1.0)) <= 1e-14


# ------------------------------------------------------------------ smoothers
def centre_coefficients(nx, ny, Lx, Ly, bc, eta_b, eta_p):
    """a_ii = diagonal of the velocity block L with the mirror relations folded in (reading R5,
    PAPER.md:1138 Eq. jacobi_update), taken from the dense stress assembly."""
    dn = Dense(nx, ny, Lx, Ly, bc, eta_b, eta_p)
    return np.diag(dn.L).copy()


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 0, 1)])
def test_one_jacobi_sweep_dense(bc):
    nx, ny = 8, 6
    f = parity_fields(nx, ny, log_contrast=2.0)
    o = Oracle(nx, ny, 1.0, 0.8, bc, omega_v=0.6, coarse_min=2)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    d = Dense(nx, ny, 1.0, 0.8, bc, f["eta_b"], f["eta_p"])
    c = centre_coefficients(nx, ny, 1.0, 0.8, bc, f["eta_b"], f["eta_p"])
    rng = np.random.default_rng(11)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = o.smooth(0, bx, by, f["vx"], f["vy"], 1)
    x = d.pack_v(f["vx"], f["vy"])
    b = d.pack_v(bx, by)
    x1 = x + 0.6 * (b - d.L @ x) / c
    ex, ey, _ = d.unpack(np.concatenate([x1, np.zeros(d.np_)]))
    assert rel(vx, ex) <= 1e-13 and rel(vy, ey) <= 1e-13
    # zero in, zero out
    z = o.smooth(0, 0 * bx, 0 * by, 0 * f["vx"], 0 * f["vy"], 3)
    assert not np.any(z[0]) and not np.any(z[1])


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 0, 1, 0)])
def test_rbgs_phase_parallel_equals_serial(bc):
    nx, ny = 8, 8
    f = parity_fields(nx, ny, log_contrast=2.0)
    o = Oracle(nx, ny, 1.0, 1.0, bc, smoother=1, omega_v=0.9, coarse_min=2)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    d = Dense(nx, ny, 1.0, 1.0, bc, f["eta_b"], f["eta_p"])
    c = centre_coefficients(nx, ny, 1.0, 1.0, bc, f["eta_b"], f["eta_p"])
    rng = np.random.default_rng(12)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = o.smooth(0, bx, by, f["vx"], f["vy"], 2)
    x = d.pack_v(f["vx"], f["vy"])
    b = d.pack_v(bx, by)
    comp = np.array([0] * d.nvx + [1] * d.nvy)
    colour = np.array([(i + j) % 2 for (i, j) in d.vx_idx] + [(i + j) % 2 for (i, j) in d.vy_idx])
    for _ in range(2):
        for cp in (0, 1):
            for col in (0, 1):
                S = (comp == cp) & (colour == col)
                r = b - d.L @ x
                x[S] += 0.9 * r[S] / c[S]  # all of a phase at once (parallel)
    ex, ey, _ = d.unpack(np.concatenate([x, np.zeros(d.np_)]))
    assert rel(vx, ex) <= 1e-13 and rel(vy, ey) <= 1e-13


def test_jacobi_stability_limit():
    """Constant eta, dx = dy, free slip: damped Jacobi is stable for w < 2/lambda_max with
    lambda_max(C^-1 L) <= 8/3 (derived, periodic Fourier bound); the oracle's sweeps grow at
    w = 0.8 and decay at w = 0.6."""
    nx = ny = 16
    eb, ep = np.ones((17, 17)), np.ones((16, 16))
    d = Dense(nx, ny, 1.0, 1.0, (0, 0, 0, 0), eb, ep)
    c = centre_coefficients(nx, ny, 1.0, 1.0, (0, 0, 0, 0), eb, ep)
    lam = np.linalg.eigvals(d.L / c[:, None]).real  # C^-1 L = C^-1 (-L) / (-1)
    assert lam.max() < 8 / 3 + 1e-9 and lam.max() > 2.5
    rng = np.random.default_rng(13)
    vx0, vy0 = rng.standard_normal((16, 17)), rng.standard_normal((17, 16))
    z = lambda a: np.zeros_like(a)
    for w, grows in ((0.8, True), (0.6, False)):
        o = Oracle(nx, ny, omega_v=w, coarse_min=2)
        o.set_viscosity(eb, ep)
        vx, vy = o.smooth(0, z(vx0), z(vy0), vx0, vy0, 200)
        n1 = np.linalg.norm(vx) + np.linalg.norm(vy)
        n0 = np.linalg.norm(vx0) + np.linalg.norm(vy0)
        assert (n1 > n0) == grows


# ------------------------------------------------------------------ coarsest + V-cycle
@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 1, 1, 1), (1, 0, 0, 1)])
def test_coarse_direct_solve_matches_dense(bc):
    nx, ny = 16, 16
    f = parity_fields(nx, ny, log_contrast=1.0)
    o = Oracle(nx, ny, 1.0, 1.0, bc, coarse_min=8)
    assert o.nlev == 2
    o.set_viscosity(f["eta_b"], f["eta_p"])
    eb, ep = o.get_viscosity(1)
    d = Dense(8, 8, 1.0, 1.0, bc, eb, ep)
    rng = np.random.default_rng(3)
    bx, by = rng.standard_normal((8, 9)), rng.standard_normal((9, 8))
    vx, vy = o.coarse_solve(bx, by)
    x = np.linalg.solve(d.L, d.pack_v(bx, by))
    ex, ey, _ = d.unpack(np.concatenate([x, np.zeros(d.np_)]))
    assert rel(vx, ex) <= 1e-12 and rel(vy, ey) <= 1e-12


def _vcycle_factor(n, cycles=6):
    o = Oracle(n, n, 1.0, 1.0, coarse_min=8, omega_v=0.6)
    o.set_viscosity(np.ones((n + 1, n + 1)), np.ones((n, n)))
    rng = np.random.default_rng(21)
    vx, vy = rng.standard_normal((n, n + 1)), rng.standard_normal((n + 1, n))
    bx, by = np.zeros_like(vx), np.zeros_like(vy)  # error == iterate
    norms = []
    for _ in range(cycles):
        vx, vy = o.vcycle(bx, by, vx, vy)
        norms.append(np.sqrt(np.sum(vx[:, 1:-1] ** 2) + np.sum(vy[1:-1] ** 2)))
    return (norms[-1] / norms[-3]) ** 0.5


def test_vcycle_factor_h_independent():
    f = [_vcycle_factor(n) for n in (64, 128, 256)]
    assert max(f) < 0.5
    assert max(f) / min(f) <= 1.2 + 1e-12, f
