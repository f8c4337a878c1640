"""Pins of the oracle's Krylov and Anderson cores (no GPU), independent of the oracle.

P10: flexible GCR(m) with modified Gram-Schmidt, Alg. 4
    * the oracle's gcr_core on <= 10 x 10 dense systems equals a numpy Alg. 4 written here,
      iterate by iterate, for both restart readings (R13 true residual / literal recursive r);
    * its normalised w_i are orthonormal to 1e-10 on a system built so that classical
      Gram-Schmidt loses orthogonality (numpy CGS > 1e-7 there): MGS, not CGS;
    * the recursive residual norm never increases (GCR minimises ||r|| over the space);
    * the Stokes instance (x = (vx, vy, p), <.,.> Euclidean over unknowns, M^-1 of the
      Uzawa splitting, energy stopping test) equals numpy Alg. 4 on tests/dense.py's
      operator with M^-1 assembled from the oracle's V-cycle (pinned by P8/P15), iterate by
      iterate across restarts; the reported E is the TRUE residual's.
Alg. 5 (reading R26) Anderson AA(m, beta)
    * aa_alpha = argmin ||R a|| s.t. 1^T a = 1, by numpy least squares on the null space of
      the constraint (a different formulation from the oracle's normal equations);
    * the oracle's AA iterates equal a numpy Alg. 5 driving the oracle's plain Uzawa map
      G(x) (one Uzawa iteration, pinned by P4/P14/P15) as a black box: beta = 0.7, m = 1..5,
      so the window order, the argmin and the mixing (1 - beta) sum a x + beta sum a G(x)
      are all checked.
"""
import numpy as np
import pytest

from dense import Dense
from oracle import oracle as O
from oracle.oracle import Oracle
from synth.fields import parity_fields


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- numpy Alg. 4 (reference)
def gcr_numpy(apply_A, precond, b, x0, m, max_iter, rtol, true_restart, energy, dot=np.dot, mgs=True):
    """Alg. 4 of PAPER.md:1416-1465: z_i = M^-1 r; w_i = A z_i; orthogonalise w_i (and z_i)
    against w_0..w_{i-1}; normalise; beta = <r, w_i>; x += beta z_i; r -= beta w_i.
    Restart every m steps (true residual if true_restart).  Exit when E(r) <= rtol and the
    true residual's E <= rtol too (otherwise restart from it).  Returns x, iters, E_true, hist, W."""
    x = x0.copy()
    r = b - apply_A(x)
    k, hist, fresh, done = 0, [], True, False
    W = []
    while k < max_iter and not done:
        if not fresh and true_restart:
            r = b - apply_A(x)
        fresh = False
        Z, W = [], []
        for i in range(m):
            if k >= max_iter:
                break
            z = precond(r)
            w = apply_A(z)
            if mgs:
                for wj, zj in zip(W, Z):
                    g = dot(w, wj)
                    w = w - g * wj
                    z = z - g * zj
            else:  # classical Gram-Schmidt (only to show the test case discriminates)
                gs = [dot(w, wj) for wj in W]
                for g, wj, zj in zip(gs, W, Z):
                    w = w - g * wj
                    z = z - g * zj
            nu = np.sqrt(dot(w, w))
            k += 1
            w, z = w / nu, z / nu
            beta = dot(r, w)
            x = x + beta * z
            r = r - beta * w
            W.append(w)
            Z.append(z)
            E = energy(r)
            hist.append(E)
            if E <= rtol:
                r = b - apply_A(x)
                fresh = True
                done = energy(r) <= rtol
                break
    return x, k, energy(b - apply_A(x)), np.array(hist), np.array(W)


def dense_case(seed, n=10):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) + 3.0 * np.eye(n)           # nonsymmetric, nonsingular
    Minv = np.linalg.inv(A + 0.5 * rng.standard_normal((n, n)))  # an inexact preconditioner
    b = rng.standard_normal(n)
    return A, Minv, b


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("m,true_restart", [(3, 1), (3, 0), (10, 1), (4, 0)])
def test_gcr_dense_iterates_equal_numpy_alg4(seed, m, true_restart):
    A, Minv, b = dense_case(seed)
    nb = np.linalg.norm(b)
    en = lambda r: np.linalg.norm(r) / nb
    for k in range(1, 13):
        o = O.gcr_dense(A, Minv, b, np.zeros_like(b), m, k, 0.0, true_restart, hist_len=k)
        x, it, E, hist, _ = gcr_numpy(lambda u: A @ u, lambda r: Minv @ r, b, np.zeros_like(b), m, k, 0.0,
                                      true_restart, en)
        assert o["iters"] == it == k
        assert rel(o["x"], x) <= 1e-12, (k, rel(o["x"], x))
        assert np.allclose(o["hist"], hist, rtol=1e-10, atol=1e-13)
        assert o["E"] == pytest.approx(E, rel=1e-10, abs=1e-13)


def test_gcr_dense_converges_to_solution_and_reports_true_residual():
    A, Minv, b = dense_case(5)
    o = O.gcr_dense(A, Minv, b, np.zeros_like(b), 4, 200, 1e-12, 1)
    assert o["status"] == 0
    assert rel(o["x"], np.linalg.solve(A, b)) <= 1e-10
    assert o["E"] == pytest.approx(np.linalg.norm(b - A @ o["x"]) / np.linalg.norm(b), rel=1e-6)
    assert o["E"] <= 1e-12


def test_gcr_dense_residual_monotone():
    for seed in range(4):
        A, Minv, b = dense_case(seed)
        for tr in (0, 1):
            o = O.gcr_dense(A, Minv, b, np.zeros_like(b), 3, 30, 0.0, tr, hist_len=30)
            h = o["hist"]
            assert np.all(h[1:] <= h[:-1] * (1 + 1e-12)), (seed, tr, h)


def test_gcr_mgs_orthogonality_where_cgs_fails():
    """M^-1 maps every residual almost onto one direction u (plus delta r): the w_i are nearly
    parallel, condition ~ 1/delta.  CGS then loses orthogonality ~ eps/delta^2, MGS ~ eps/delta."""
    n, m, delta = 10, 6, 1e-4
    rng = np.random.default_rng(8)
    A = np.eye(n) + 0.3 * rng.standard_normal((n, n))
    u = rng.standard_normal(n)
    u /= np.linalg.norm(u)
    Minv = np.outer(u, rng.standard_normal(n)) + delta * np.eye(n)
    b = rng.standard_normal(n)
    nb = np.linalg.norm(b)
    en = lambda r: np.linalg.norm(r) / nb
    ortho = lambda W: np.abs(W @ W.T - np.eye(len(W))).max()
    _, _, _, _, Wm = gcr_numpy(lambda v: A @ v, lambda r: Minv @ r, b, np.zeros(n), m, m, 0.0, 1, en, mgs=True)
    _, _, _, _, Wc = gcr_numpy(lambda v: A @ v, lambda r: Minv @ r, b, np.zeros(n), m, m, 0.0, 1, en, mgs=False)
    assert ortho(Wc) > 1e-7, ortho(Wc)  # the case discriminates
    assert ortho(Wm) <= 1e-10, ortho(Wm)
    o = O.gcr_dense(A, Minv, b, np.zeros(n), m, m, 0.0, 1)
    assert o["iters"] == m
    assert ortho(o["W"]) <= 1e-10, ortho(o["W"])
    assert np.abs(o["W"] - Wm).max() <= 1e-8


# ---------------------------------------------------------------- Stokes instance of Alg. 4
def stokes_case(n, bc, seed_contrast=1.0):
    f = parity_fields(n, n, log_contrast=seed_contrast)
    return f


@pytest.mark.parametrize("n,bc,m,true_restart", [(6, (0, 0, 0, 0), 3, 1), (8, (1, 0, 1, 0), 4, 0),
                                                  (8, (0, 1, 1, 0), 10, 1)])
def test_gcr_stokes_iterates_equal_numpy_alg4(n, bc, m, true_restart):
    f = stokes_case(n, bc)
    g = (0.2, 1.0)
    kw = dict(omega_v=0.4, alpha_p=1.0, coarse_min=2, accel=1, gcr_restart=m, gcr_true_restart=true_restart)
    d = Dense(n, n, 1.0, 1.0, bc, f["eta_b"], f["eta_p"])
    nv = d.nvx + d.nvy
    b = np.concatenate([d.force(f["rho_b"], *g)[:nv], np.zeros(d.np_)])
    o0 = Oracle(n, n, 1.0, 1.0, bc, **kw)
    o0.set_viscosity(f["eta_b"], f["eta_p"])

    def precond(r):  # z_v = V-cycle(0; r_v), z_p = alpha eta_P (r_p - D z_v), de-meaned (R3, R14)
        rx, ry, rp = d.unpack(r)
        zx, zy = o0.vcycle(rx, ry, np.zeros_like(rx), np.zeros_like(ry))
        zv = d.pack_v(zx, zy)
        zp = 1.0 * f["eta_p"].ravel() * (r[nv:] - d.D @ zv)
        return np.concatenate([zv, zp - zp.mean()])

    dv = -np.diag(d.L)
    c = 2 / d.dx ** 2 + 2 / d.dy ** 2
    Sf = np.sum(b[:nv] ** 2 / dv)
    energy = lambda r: np.sqrt((np.sum(r[:nv] ** 2 / dv) + np.sum(r[nv:] ** 2 * f["eta_p"].ravel() / c)) / Sf)
    for k in (1, 2, m, m + 1, 2 * m + 1):
        o = Oracle(n, n, 1.0, 1.0, bc, **dict(kw, max_iter=k))
        o.set_viscosity(f["eta_b"], f["eta_p"])
        o.set_density(f["rho_b"])
        o.set_gravity(*g)
        a = o.solve(0.0, hist_len=k)
        x, it, E, hist, _ = gcr_numpy(lambda u: d.A @ u, precond, b, np.zeros(d.n), m, k, 0.0, true_restart, energy)
        assert a["iters"] == it == k
        xo = d.pack(a["vx"], a["vy"], a["p"])
        x[nv:] -= x[nv:].mean()  # the solve returns the zero-mean pressure
        assert rel(xo, x) <= 1e-11, (k, rel(xo, x))
        assert np.allclose(a["hist"], hist, rtol=1e-9, atol=0)
        assert a["E"] == pytest.approx(E, rel=1e-9)  # true residual reported


def test_gcr_stokes_exit_on_true_residual():
    """Converged solves report E of the TRUE residual and it is <= rtol."""
    n = 16
    f = stokes_case(n, (0, 0, 0, 0))
    o = Oracle(n, n, 1.0, 1.0, (0, 0, 0, 0), omega_v=0.4, alpha_p=1.0, accel=1, gcr_restart=5)
    o.set_viscosity(f["eta_b"], f["eta_p"])
    o.set_density(f["rho_b"])
    o.set_gravity(0.2, 1.0)
    s = o.solve(1e-10)
    assert s["status"] == 0
    _, _, _, E = o.residual(s["vx"], s["vy"], s["p"])
    assert E <= 1e-10 and s["E"] == pytest.approx(E, rel=1e-6)


# ---------------------------------------------------------------- Alg. 5 (Anderson)
def argmin_numpy(R):
    """argmin ||R a||_2 s.t. sum a = 1: a = e_last + N g with N spanning {1^T a = 0}."""
    nn = R.shape[1]
    e = np.zeros(nn)
    e[-1] = 1.0
    N = np.zeros((nn, nn - 1))
    for q in range(nn - 1):
        N[q, q], N[nn - 1, q] = 1.0, -1.0
    g = np.linalg.lstsq(R @ N, -R @ e, rcond=None)[0]
    return e + N @ g


@pytest.mark.parametrize("nn", [1, 2, 3, 4, 6])
def test_aa_alpha_is_constrained_argmin(nn):
    rng = np.random.default_rng(nn)
    R = rng.standard_normal((40, nn)) * np.logspace(0, -2, nn)
    a = O.aa_alpha(R.T @ R)
    assert a.sum() == pytest.approx(1.0, abs=1e-14)
    # R26 regularises the normal equations by lambda = 1e-10 max diag(H) (rank-deficient
    # histories): the argmin moves by at most ~ lambda ||H^-1|| (x10 margin)
    H = R.T @ R
    bound = 10 * 1e-10 * H.diagonal().max() * np.linalg.norm(np.linalg.inv(H), 2) + 1e-12
    assert np.abs(a - argmin_numpy(R)).max() <= bound
    # optimality: no feasible perturbation lowers ||R a||
    for _ in range(20):
        d = rng.standard_normal(nn)
        d -= d.mean()
        assert np.linalg.norm(R @ (a + 1e-3 * d)) >= np.linalg.norm(R @ a) * (1 - 1e-12)


@pytest.mark.parametrize("m", [1, 2, 3, 5])
def test_anderson_iterates_equal_numpy_alg5(m):
    n, bc, beta = 8, (0, 1, 1, 0), 0.7
    f = parity_fields(n, n, log_contrast=1.0)
    kw = dict(omega_v=0.4, alpha_p=1.0, coarse_min=2)
    g = (0.2, 1.0)

    def oracle(**o):
        s = Oracle(n, n, 1.0, 1.0, bc, **dict(kw, **o))
        s.set_viscosity(f["eta_b"], f["eta_p"])
        s.set_density(f["rho_b"])
        s.set_gravity(*g)
        return s

    uz = oracle(max_iter=1)

    def G(x):  # one plain Uzawa iteration (+ de-mean) of the oracle: the black-box map
        r = uz.solve(0.0, vx=x[0], vy=x[1], p=x[2])
        assert r["iters"] == 1
        return (r["vx"], r["vy"], r["p"])

    flat = lambda x: np.concatenate([a.ravel() for a in x])
    shapes = [(n, n + 1), (n + 1, n), (n, n)]

    def unflat(v):
        out, o = [], 0
        for s in shapes:
            out.append(v[o:o + s[0] * s[1]].reshape(s))
            o += s[0] * s[1]
        return out

    # numpy Alg. 5: x^1 = G(x^0); x^{k+1} = sum a_i [(1 - beta) x^i + beta G(x^i)], window m_k = min(m, k)
    K = 8
    X, GX = [flat([np.zeros(s) for s in shapes])], []
    for k in range(K):
        GX.append(flat(G(unflat(X[k]))))
        if k == 0:
            X.append(GX[0])
            continue
        mk = min(m, k)
        idx = range(k - mk, k + 1)
        R = np.stack([GX[i] - X[i] for i in idx], axis=1)
        # the argmin with R26's regularisation (pinned against the exact argmin above); the
        # regularised and exact argmins differ by ~ lambda ||H^-1||, which the later, nearly
        # rank-deficient histories amplify beyond this test's 1e-8
        H = R.T @ R
        zz = np.linalg.solve(H + 1e-10 * H.diagonal().max() * np.eye(len(H)), np.ones(len(H)))
        a = zz / zz.sum()
        xn = sum(a[q] * ((1 - beta) * X[i] + beta * GX[i]) for q, i in enumerate(idx))
        xv = unflat(xn)
        xv[2] = xv[2] - xv[2].mean()  # zero-mean pressure after every update
        X.append(flat(xv))
    for k in (2, 3, 5, K):
        a = oracle(accel=2, aa_depth=m, aa_beta=beta, max_iter=k).solve(0.0)
        assert a["iters"] == k
        want = unflat(X[k])
        for got, exp in zip((a["vx"], a["vy"], a["p"]), want):
            assert rel(got, exp) <= 1e-8, (k, rel(got, exp))
