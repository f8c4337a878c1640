"""GPU parity at BASELINE.json's full sizes, in bench.py's launch configuration (the same
presets, the same handle API): operator applies and the first Uzawa iterations against
the oracle element by element; converged solves via properties that hold at any size
(the oracle's own energy residual of the GPU solution <= rtol, zero-mean pressure)."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import Oracle  # noqa: E402
from synth.fields import parity_fields, workload  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRE = json.load(open(os.path.join(ROOT, "configs", "presets.json")))


def rel(a, b):
    a = a.detach().cpu().numpy() if torch.is_tensor(a) else a
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def setup(name, n=None, **extra):
    from paper_2603_14040_b200 import Stokes
    pre = PRE[name]
    nx, ny = pre["n"] if n is None else (n, n)
    w = workload(pre["workload"], nx, ny)
    opts = dict(pre["opts"], **extra)
    o = Oracle(nx, ny, w["Lx"], w["Ly"], w["bc"], **opts)
    s = Stokes(nx, ny, w["Lx"], w["Ly"], w["bc"], **opts)
    o.set_viscosity(w["eta_b"], w["eta_p"])
    s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    o.set_density(w["rho_b"])
    s.set_density(T(w["rho_b"]))
    o.set_gravity(w["gx"], w["gy"])
    s.set_gravity(w["gx"], w["gy"])
    return o, s, pre, w


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def test_layered_4096_operator_and_first_iterations():
    o, s, pre, w = setup("layered")
    n = pre["n"][0]
    f = parity_fields(n, n)
    ex = o.apply_operator(f["vx"], f["vy"], f["p"])
    got = s.apply_operator(T(f["vx"]), T(f["vy"]), T(f["p"]))
    for g_, e_ in zip(got, ex):
        assert rel(g_, e_) <= 1e-12
    # two Uzawa iterations (V-cycle + pressure update + energy) element by element
    o2, s2, _, _ = setup("layered", max_iter=2)
    a = o2.solve(0.0)
    b = s2.solve(0.0)
    assert a["iters"] == b["iters"] == 2
    assert abs(a["E"] - b["E"]) <= 1e-10 * a["E"]
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-11, k


def test_layered_4096_converged_solution_properties():
    o, s, pre, w = setup("layered")
    r = s.solve(pre["rtol"])
    assert r["status"] == 0 and r["E"] <= pre["rtol"]
    _, _, _, E = o.residual(r["vx"].cpu().numpy(), r["vy"].cpu().numpy(), r["p"].cpu().numpy())
    assert E <= 1.001 * pre["rtol"]
    p = r["p"]
    assert abs(float(p.mean())) <= 1e-12 * float(p.abs().max())


def test_block_512_full_solve_parity():
    o, s, pre, w = setup("block")
    a = o.solve(pre["rtol"])
    b = s.solve(pre["rtol"])
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["iters"] - b["iters"]) <= 1, (a["iters"], b["iters"])
    assert b["E"] <= pre["rtol"]
    # the GPU solution against the oracle's iterate at the GPU's count
    o2, _, _, _ = setup("block", max_iter=b["iters"])
    a2 = o2.solve(0.0)
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a2[k]) <= 1e-9, (k, rel(b[k], a2[k]))


def test_solcx_2048_converged_solution_properties():
    o, s, pre, w = setup("solcx")
    r = s.solve(pre["rtol"])
    assert r["status"] == 0 and r["E"] <= pre["rtol"]
    _, _, _, E = o.residual(r["vx"].cpu().numpy(), r["vy"].cpu().numpy(), r["p"].cpu().numpy())
    # GCR exits only when the TRUE residual passes too, and reports that E
    assert E <= pre["rtol"]
    assert r["E"] == pytest.approx(E, rel=1e-6)


@pytest.mark.parametrize("smoother,nsweeps", [(1, 1), (0, 2)])
def test_fine_smoothers_4096(smoother, nsweeps):
    """The fine-level smoother kernels at the bench size, element by element: one RBGS sweep
    (the one-pass four-phase kernel, whose strips are only tall enough at the large levels)
    and one two-sweep Jacobi pass, on the layered 4096^2 fields with random iterates."""
    o, s, pre, w = setup("layered", smoother=smoother)
    n = pre["n"][0]
    f = parity_fields(n, n, log_contrast=1.0)
    rng = np.random.default_rng(5)
    bx, by = rng.standard_normal((n, n + 1)), rng.standard_normal((n + 1, n))
    ex, ey = o.smooth(0, bx, by, f["vx"], f["vy"], nsweeps)
    gx, gy = s.smooth(0, T(bx), T(by), T(f["vx"]), T(f["vy"]), nsweeps)
    assert rel(gx, ex) <= 1e-12 and rel(gy, ey) <= 1e-12
