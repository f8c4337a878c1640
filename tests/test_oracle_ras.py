"""Oracle pins for SURVEY §8(f) NEXT-3: the RAS-type temporally blocked Jacobi smoother
(Alg. 3; reading R27) and the "Mixed" setting (Jacobi on the finest
level, RAS below).

The oracle's RAS sweeps are checked against an independent block-Jacobi written on the
dense matrix of tests/dense.py (assembled from the stress formulas, mirrors folded): for
every tile T, T_inner damped-Jacobi steps on  L_TT x_T = b_T - L_T,out x_out  with x_out
frozen at the start of the outer iteration.  The tile shifts come from the counter-based
generator that reading R27 specifies (splitmix64; re-implemented here from that spec, it
holds none of the method's arithmetic).  T_inner = 1 must be plain damped Jacobi.
"""
import numpy as np
import pytest

from dense import Dense
from oracle.oracle import Oracle
from synth.fields import parity_fields

M64 = (1 << 64) - 1


def splitmix64(x):
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def shift(seed, q, T):
    u = splitmix64(seed ^ ((q * 0x9E3779B97F4A7C15) & M64))
    return (u & 0xFFFFFFFF) % T, (u >> 32) % T


def dense_ras(d, b, x, omega, T, tin, nsweeps, seed):
    L = d.L
    diag = np.diag(L)
    nout = -(-nsweeps // tin)
    nout += nout % 2
    cells = [(i, j) for (i, j) in d.vx_idx] + [(i, j) for (i, j) in d.vy_idx]
    for t in range(nout):
        si, sj = shift(seed, t, T)
        tile = np.array([((i - 1 + si) // T) * 100000 + (j - 1 + sj) // T for (i, j) in cells])
        x0 = x.copy()
        xn = x0.copy()
        for tid in np.unique(tile):
            idx = np.where(tile == tid)[0]
            out = np.where(tile != tid)[0]
            rhs = b[idx] - L[np.ix_(idx, out)] @ x0[out]
            xt = x0[idx].copy()
            for _ in range(tin):
                xt = xt + omega * (rhs - L[np.ix_(idx, idx)] @ xt) / diag[idx]
            xn[idx] = xt
        x = xn
    return x


@pytest.mark.parametrize("bc", [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0)])
@pytest.mark.parametrize("T,tin,nsweeps", [(4, 2, 3), (5, 3, 6), (3, 1, 4)])
def test_ras_equals_dense_block_jacobi(bc, T, tin, nsweeps):
    nx, ny, seed, omega = 12, 10, 2603, 0.5
    f = parity_fields(nx, ny, log_contrast=1.0)
    o = Oracle(nx, ny, 1.0, 0.8, bc, smoother=2, omega_v=omega, ras_tile=T, ras_inner=tin, ras_seed=seed,
               coarse_min=2, coarse_direct=0)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    rng = np.random.default_rng(4)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    gx, gy = o.smooth(0, bx, by, vx, vy, nsweeps)
    d = Dense(nx, ny, 1.0, 0.8, bc, f["eta_b"], f["eta_p"])
    x = dense_ras(d, d.pack_v(bx, by), d.pack_v(vx, vy), omega, T, tin, nsweeps, seed)
    ex, ey, _ = d.unpack(np.concatenate([x, np.zeros(d.np_)]))
    np.testing.assert_allclose(gx[:, 1:-1], ex[:, 1:-1], rtol=0, atol=1e-12 * np.abs(ex).max())
    np.testing.assert_allclose(gy[1:-1], ey[1:-1], rtol=0, atol=1e-12 * np.abs(ey).max())


def test_ras_single_inner_is_jacobi():
    nx, ny = 16, 12
    f = parity_fields(nx, ny, log_contrast=1.0)
    rng = np.random.default_rng(6)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    out = []
    for sm in (0, 2):
        o = Oracle(nx, ny, 1.0, 1.0, (0, 1, 0, 1), smoother=sm, omega_v=0.5, ras_tile=5, ras_inner=1,
                   coarse_min=2, coarse_direct=0)
        o.set_viscosity(f["eta_b"], f["eta_p"])
        out.append(o.smooth(0, bx, by, vx, vy, 4))
    for a, b in zip(*out):
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-14 * np.abs(a).max())


@pytest.mark.parametrize("smoother", [2, 3])
def test_ras_and_mixed_solve_to_the_fixed_point(smoother):
    n = 16
    f = parity_fields(n, n, log_contrast=1.0)
    d = Dense(n, n, 1.0, 1.0, (0, 0, 0, 0), f["eta_b"], f["eta_p"])
    o = Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), smoother=smoother, omega_v=0.4, alpha_p=1.0, ras_tile=4,
               coarse_min=2, max_iter=5000)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.2, 1.0)
    s = o.solve(1e-12)
    assert s["status"] == 0
    vx, vy, p = d.unpack(d.solve_bordered(d.force(f["rho_b"], 0.2, 1.0)))
    for a, b in ((s["vx"], vx), (s["vy"], vy), (s["p"], p)):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
