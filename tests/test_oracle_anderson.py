"""Oracle pins for SURVEY §8(f) NEXT-2: Anderson acceleration AA(m) with mixing beta
(Alg. 5; reading R26).

  * m = 0, beta = 1 is the plain fixed-point iteration x^{k+1} = G(x^k): cycle for cycle
    the Uzawa solve (SPEC.md "anderson beta=1, m=0 run == plain run");
  * m = 0, beta < 1 is the damped iteration (1 - beta) x + beta G(x): its error contracts
    like (1 - beta) + beta rho, so it needs more iterations, to the same fixed point;
  * AA(m >= 1) reaches the same fixed point -- the dense bordered solution
    (test_oracle_solver.test_fixed_point_is_dense_solution[accel=2]) -- in fewer
    iterations than the plain iteration (its linear-case GMRES equivalence).
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from synth.fields import workload


def run(name, n, **kw):
    w = workload(name, n, n)
    o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], omega_v=0.6, alpha_p=1.0, **kw)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    o.set_density(w["rho_b"])
    o.set_gravity(w["gx"], w["gy"])
    return o.solve(1e-10, hist_len=2000)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("name", ["block", "layered"])
def test_depth0_beta1_is_the_plain_iteration(name):
    a = run(name, 32)
    b = run(name, 32, accel=2, aa_depth=0, aa_beta=1.0)
    # identical up to the re-de-mean of an already zero-mean pressure after each update
    assert a["iters"] == b["iters"]
    np.testing.assert_allclose(b["hist"][: b["iters"]], a["hist"][: a["iters"]], rtol=0, atol=1e-12)
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-12, k


def test_depth0_damped_iteration_is_slower_to_the_same_point():
    a = run("block", 32)
    b = run("block", 32, accel=2, aa_depth=0, aa_beta=0.5)
    assert b["status"] == 0 and b["iters"] > a["iters"]
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-8, k


@pytest.mark.parametrize("m,beta", [(1, 1.0), (5, 0.7), (10, 1.0)])
def test_anderson_accelerates_to_the_same_fixed_point(m, beta):
    a = run("block", 32)
    b = run("block", 32, accel=2, aa_depth=m, aa_beta=beta)
    assert b["status"] == 0 and b["iters"] < a["iters"]
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-8, k
