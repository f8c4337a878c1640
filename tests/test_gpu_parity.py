"""GPU parity: every hot-path step of the CUDA library (called through the C ABI via the
thin binding) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): per-operator applies <= 1e-12 relative L2; converged
vx, vy, p <= 1e-9 relative L2 at equal residual tolerance with iteration counts within
+-1.  Sizes span several 32x8 tiles with ragged tails (33 x 17, 130 x 66) and the
degenerate smallest grids; full BASELINE sizes are covered in test_gpu_fullsize.py.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import Oracle  # noqa: E402
from synth.fields import parity_fields, workload  # noqa: E402

BCS = [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0)]
SIZES = [(8, 8), (33, 17), (130, 66), (256, 256)]
TOL_OP = 1e-12
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = a.detach().cpu().numpy() if torch.is_tensor(a) else a
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_14040_b200 import Stokes
    return Stokes


def pair(S, nx, ny, bc, fields, Lx=1.0, Ly=1.0, g=(0.2, 1.0), **opts):
    o = Oracle(nx, ny, Lx, Ly, bc, **opts)
    s = S(nx, ny, Lx, Ly, bc, **opts)
    o.set_viscosity(fields["eta_b"], fields["eta_p"])
    s.set_viscosity(torch.from_numpy(fields["eta_b"]).cuda(), torch.from_numpy(fields["eta_p"]).cuda())
    o.set_density(fields["rho_b"])
    s.set_density(torch.from_numpy(fields["rho_b"]).cuda())
    o.set_gravity(*g)
    s.set_gravity(*g)
    return o, s


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("nx,ny", SIZES)
@pytest.mark.parametrize("bc", BCS)
def test_apply_operator(S, nx, ny, bc):
    f = parity_fields(nx, ny)
    o, s = pair(S, nx, ny, bc, f, 1.0, 0.7, coarse_direct=0)
    ex = o.apply_operator(f["vx"], f["vy"], f["p"])
    got = s.apply_operator(T(f["vx"]), T(f["vy"]), T(f["p"]))
    for g_, e_ in zip(got, ex):
        assert rel(g_, e_) <= TOL_OP


@pytest.mark.parametrize("nx,ny", SIZES)
@pytest.mark.parametrize("bc", BCS)
def test_residual_and_energy(S, nx, ny, bc):
    f = parity_fields(nx, ny)
    o, s = pair(S, nx, ny, bc, f, coarse_direct=0)
    rx, ry, rp, E = o.residual(f["vx"], f["vy"], f["p"])
    gx, gy, gp, gE = s.residual(T(f["vx"]), T(f["vy"]), T(f["p"]))
    assert rel(gx, rx) <= TOL_OP and rel(gy, ry) <= TOL_OP and rel(gp, rp) <= TOL_OP
    assert abs(gE - E) <= TOL_OP * E


@pytest.mark.parametrize("smoother", [0, 1])
@pytest.mark.parametrize("nx,ny", [(8, 8), (33, 17), (128, 64)])
@pytest.mark.parametrize("bc", BCS)
def test_smoother(S, smoother, nx, ny, bc):
    f = parity_fields(nx, ny, log_contrast=1.0)
    o, s = pair(S, nx, ny, bc, f, smoother=smoother, omega_v=0.5, coarse_min=4, coarse_direct=0)
    rng = np.random.default_rng(9)
    for level in range(min(o.nlev, 2)):
        lnx, lny, _ = o.level_shape(level)
        bx, by = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
        vx, vy = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
        ex, ey = o.smooth(level, bx, by, vx, vy, 3)
        gx, gy = s.smooth(level, T(bx), T(by), T(vx), T(vy), 3)
        assert rel(gx, ex) <= TOL_OP and rel(gy, ey) <= TOL_OP
        rx, ry = o.level_residual(level, bx, by, vx, vy)
        qx, qy = s.level_residual(level, T(bx), T(by), T(vx), T(vy))
        assert rel(qx[:, 1:-1], rx[:, 1:-1]) <= TOL_OP and rel(qy[1:-1], ry[1:-1]) <= TOL_OP


@pytest.mark.parametrize("nsweeps", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("nx,ny", [(8, 8), (33, 17), (64, 200), (300, 250), (1030, 13)])
@pytest.mark.parametrize("bc", BCS)
def test_tile_smoother(S, nx, ny, bc, nsweeps, monkeypatch):
    """n damped-Jacobi sweeps of a small level in one launch (k_jacobi_tile: 8 x 32 tiles with an
    (n+1)-cell frame in shared memory, the sweeps shrinking region by region): ragged tiles,
    one-row / one-column tiles, every boundary set, n = 1 .. 8, against the oracle's n sweeps."""
    monkeypatch.setenv("STOKES_TILE_CELLS", str(10 ** 9))
    f = parity_fields(nx, ny, log_contrast=1.0)
    o, s = pair(S, nx, ny, bc, f, omega_v=0.5, coarse_min=4, coarse_direct=0)
    rng = np.random.default_rng(13)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx[:, [0, -1]] = 0.0
    vy[[0, -1], :] = 0.0
    ex, ey = o.smooth(0, bx, by, vx, vy, nsweeps)
    gx, gy = s.smooth(0, T(bx), T(by), T(vx), T(vy), nsweeps)
    assert rel(gx, ex) <= TOL_OP and rel(gy, ey) <= TOL_OP


@pytest.mark.parametrize("smoother,nsweeps", [(0, 2), (0, 4), (0, 5), (1, 1), (1, 2), (1, 3)])
@pytest.mark.parametrize("nx,ny", [(128, 8), (300, 250), (1030, 13)])
@pytest.mark.parametrize("bc", BCS)
def test_streamed_smoothers(S, nx, ny, bc, smoother, nsweeps, monkeypatch):
    """Levels >= 128 x 8 run Jacobi sweep pairs as one temporally blocked pass (two sweeps
    per HBM read) and RBGS sweeps as one streamed pass (the four phases as a wavefront:
    vx red row s, vx black s-2, vy red s-4, vy black s-6 per step); ragged column tiles,
    8-row strips and every mirror ghost included.  (The small-level tile smoother is switched
    off here so that these sizes exercise the streamed passes.)"""
    monkeypatch.setenv("STOKES_TILE_CELLS", "0")
    f = parity_fields(nx, ny, log_contrast=1.0)
    o, s = pair(S, nx, ny, bc, f, smoother=smoother, omega_v=0.5, coarse_min=4, coarse_direct=0)
    rng = np.random.default_rng(11)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx, vy = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    vx[:, [0, -1]] = 0.0
    vy[[0, -1], :] = 0.0
    ex, ey = o.smooth(0, bx, by, vx, vy, nsweeps)
    gx, gy = s.smooth(0, T(bx), T(by), T(vx), T(vy), nsweeps)
    assert rel(gx, ex) <= TOL_OP and rel(gy, ey) <= TOL_OP


def test_one_pass_rbgs_forced():
    """The one-pass four-phase RBGS kernel on every streamed level (STOKES_RBGS1=2, in a
    subprocess: the mode is read once per process) on ragged grids, all BC sets, 1-3 sweeps
    and a V-cycle, against the oracle (<= 1e-12)."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from oracle.oracle import Oracle
from synth.fields import parity_fields
from paper_2603_14040_b200 import Stokes
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rel = lambda a, b: float(np.linalg.norm(a.cpu().numpy() - b) / np.linalg.norm(b))
worst = 0.0
for (nx, ny) in [(128, 40), (300, 250), (1030, 23)]:
    for bc in [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0)]:
        f = parity_fields(nx, ny, log_contrast=1.0)
        kw = dict(smoother=1, omega_v=0.5, coarse_min=4, coarse_direct=0)
        o, s = Oracle(nx, ny, 1.0, 1.0, bc, **kw), Stokes(nx, ny, 1.0, 1.0, bc, **kw)
        o.set_viscosity(f["eta_b"], f["eta_p"]); s.set_viscosity(T(f["eta_b"]), T(f["eta_p"]))
        o.set_density(f["rho_b"]); s.set_density(T(f["rho_b"]))
        o.set_gravity(0.2, 1.0); s.set_gravity(0.2, 1.0)
        rng = np.random.default_rng(13)
        bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
        vx, vy = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
        vx[:, [0, -1]] = 0.0
        vy[[0, -1], :] = 0.0
        for k in (1, 3):
            ex, ey = o.smooth(0, bx, by, vx, vy, k)
            gx, gy = s.smooth(0, T(bx), T(by), T(vx), T(vy), k)
            worst = max(worst, rel(gx, ex), rel(gy, ey))
        ex, ey = o.vcycle(bx, by, vx, vy)
        gx, gy = s.vcycle(T(bx), T(by), T(vx), T(vy))
        worst = max(worst, rel(gx, ex), rel(gy, ey))
print(worst)
""" % ROOT
    env = dict(os.environ, STOKES_RBGS1="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL_OP


def test_fused_pair_residual_restriction_forced():
    """The last pre-smoothing pair fused with the residual and its restriction (k_j2rr, off by
    default: measured slower) enabled in a subprocess (STOKES_J2RR=1): V-cycles on ragged
    grids with several column tiles and coarse-row strips against the oracle (<= 1e-12)."""
    import subprocess
    import sys
    code = r"""
import numpy as np, torch, sys
sys.path.insert(0, %r)
from oracle.oracle import Oracle
from synth.fields import parity_fields
from paper_2603_14040_b200 import Stokes
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rel = lambda a, b: float(np.linalg.norm(a.cpu().numpy() - b) / np.linalg.norm(b))
worst = 0.0
for (nx, ny, bc) in [(512, 256, (0, 1, 0, 1)), (640, 384, (1, 1, 0, 0)), (128, 128, (0, 0, 0, 0))]:
    f = parity_fields(nx, ny, log_contrast=1.0)
    kw = dict(omega_v=0.5)
    o, s = Oracle(nx, ny, 1.0, 1.0, bc, **kw), Stokes(nx, ny, 1.0, 1.0, bc, **kw)
    o.set_viscosity(f["eta_b"], f["eta_p"]); s.set_viscosity(T(f["eta_b"]), T(f["eta_p"]))
    o.set_density(f["rho_b"]); s.set_density(T(f["rho_b"]))
    o.set_gravity(0.2, 1.0); s.set_gravity(0.2, 1.0)
    rng = np.random.default_rng(12)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    ex, ey = o.vcycle(bx, by, f["vx"], f["vy"])
    gx, gy = s.vcycle(T(bx), T(by), T(f["vx"]), T(f["vy"]))
    worst = max(worst, rel(gx, ex), rel(gy, ey))
print(worst)
""" % ROOT
    env = dict(os.environ, STOKES_J2RR="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL_OP


@pytest.mark.parametrize("tile,tin,nsweeps", [(8, 2, 3), (32, 4, 5), (5, 3, 8)])
@pytest.mark.parametrize("nx,ny", [(100, 60), (256, 130)])
@pytest.mark.parametrize("bc", BCS)
def test_ras_smoother(S, nx, ny, bc, tile, tin, nsweeps):
    """RAS-type temporal blocking (Alg. 3, reading R27): shifted tiles staged in shared
    memory, T_inner sweeps with a frozen frame, single writer; same counter-based shifts."""
    f = parity_fields(nx, ny, log_contrast=1.0)
    kw = dict(smoother=2, omega_v=0.5, ras_tile=tile, ras_inner=tin, ras_seed=77, coarse_min=4, coarse_direct=0)
    o, s = pair(S, nx, ny, bc, f, **kw)
    rng = np.random.default_rng(13)
    for level in range(2):
        lnx, lny, _ = o.level_shape(level)
        bx, by = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
        vx, vy = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
        ex, ey = o.smooth(level, bx, by, vx, vy, nsweeps)
        gx, gy = s.smooth(level, T(bx), T(by), T(vx), T(vy), nsweeps)
        assert rel(gx, ex) <= TOL_OP and rel(gy, ey) <= TOL_OP, level


@pytest.mark.parametrize("name,n,opts", [
    ("layered", 128, dict(smoother=2)),
    ("layered", 128, dict(smoother=3)),
    ("block", 64, dict(smoother=3, ras_tile=16)),
    ("solcx", 128, dict(smoother=2, accel=1)),
    ("block", 128, dict(smoother=3, accel=2, aa_depth=5, aa_beta=0.7)),
])
def test_ras_solve_parity(S, name, n, opts):
    """RAS / Mixed inside Uzawa, GCR and Anderson solves: a new shift per outer iteration and
    per V-cycle (device iteration index under graph replay), same as the oracle's draws."""
    opts = dict(opts, omega_v=0.6, alpha_p=1.0)
    w = workload(name, n, n)
    args = (S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]))
    o, s = pair(*args, **dict(opts, max_iter=15))
    a, b = o.solve(0.0), s.solve(0.0)
    assert a["iters"] == b["iters"] == 15
    d15 = max(rel(b[key], a[key]) for key in ("vx", "vy", "p"))
    assert d15 <= 1e-8, d15
    o, s = pair(*args, **opts)
    a, b = o.solve(1e-8), s.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    ka, kb = a["iters"], b["iters"]
    band = 1
    if opts.get("accel", 0) == 2:
        # Anderson's count is rounding-chaotic (reading R26): the ORACLE itself moves 158 ->
        # 171 / 185 / 162 iterations on block 128^2 with the Mixed smoother under 1e-15 .. 1e-14
        # perturbations of rho.  Band = twice the oracle's own spread over four perturbations
        # of rho of the size of the GPU-oracle difference after 15 iterations (d15: the
        # rounding-order difference the count is exposed to); the unique fixed point is
        # checked below to 1e-9.
        spread = 0
        for seed in range(4):
            w2 = dict(w, rho_b=w["rho_b"] * (1.0 + max(d15, 1e-15) * np.random.default_rng(seed).standard_normal(
                w["rho_b"].shape)))
            o2 = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **opts)
            o2.set_viscosity(w2["eta_b"], w2["eta_p"])
            o2.set_density(w2["rho_b"])
            o2.set_gravity(w["gx"], w["gy"])
            spread = max(spread, abs(o2.solve(1e-8)["iters"] - ka))
        band = max(2, 2 * spread)
        a, b = o.solve(1e-11), s.solve(1e-11)
        for key in ("vx", "vy", "p"):
            assert rel(b[key], a[key]) <= 1e-9, key
    assert abs(ka - kb) <= band, (ka, kb, band)


@pytest.mark.parametrize("nx,ny", [(16, 16), (64, 32), (136, 72)])
@pytest.mark.parametrize("bc", BCS)
def test_transfers_and_coarse_viscosity(S, nx, ny, bc):
    f = parity_fields(nx, ny)
    o, s = pair(S, nx, ny, bc, f, coarse_min=4)
    assert o.nlev == s.num_levels
    rng = np.random.default_rng(10)
    for level in range(o.nlev - 1):
        lnx, lny, _ = o.level_shape(level)
        for kind, shp in (("vx", (lny, lnx + 1)), ("vy", (lny + 1, lnx)), ("p", (lny, lnx)), ("b", (lny + 1, lnx + 1))):
            a = rng.standard_normal(shp)
            if kind == "vx":
                a[:, [0, -1]] = 0
            if kind == "vy":
                a[[0, -1], :] = 0
            assert rel(s.restrict(level, kind, T(a)), o.restrict(level, kind, a)) <= TOL_OP
        cnx, cny, _ = o.level_shape(level + 1)
        ex, ey = rng.standard_normal((cny, cnx + 1)), rng.standard_normal((cny + 1, cnx))
        vx, vy = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
        px, py = o.prolong(level, ex, ey, vx, vy)
        qx, qy = s.prolong(level, T(ex), T(ey), T(vx), T(vy))
        assert rel(qx, px) <= TOL_OP and rel(qy, py) <= TOL_OP
    for level in range(o.nlev):
        eb, ep = o.get_viscosity(level)
        gb, gp = s.get_viscosity(level)
        assert rel(gb, eb) <= TOL_OP and rel(gp, ep) <= TOL_OP
    lnx, lny, _ = o.level_shape(o.nlev - 1)
    bx, by = rng.standard_normal((lny, lnx + 1)), rng.standard_normal((lny + 1, lnx))
    ex, ey = o.coarse_solve(bx, by)
    qx, qy = s.coarse_solve(T(bx), T(by))
    assert rel(qx, ex) <= 1e-11 and rel(qy, ey) <= 1e-11


@pytest.mark.parametrize("smoother", [0, 1])
@pytest.mark.parametrize("nx,ny,bc", [(64, 64, (0, 0, 0, 0)), (128, 64, (1, 0, 1, 0)), (96, 48, (1, 1, 1, 1)),
                                      (512, 256, (0, 1, 0, 1)), (640, 384, (1, 1, 0, 0))])
def test_vcycle(S, smoother, nx, ny, bc):
    """Levels >= 128 x 8 take the streamed kernels (two-sweep passes, residual fused with
    its restriction: several column tiles and strips, ragged last tile at 640)."""
    f = parity_fields(nx, ny, log_contrast=1.0)
    o, s = pair(S, nx, ny, bc, f, smoother=smoother, omega_v=0.5)
    rng = np.random.default_rng(12)
    bx, by = rng.standard_normal((ny, nx + 1)), rng.standard_normal((ny + 1, nx))
    ex, ey = o.vcycle(bx, by, f["vx"], f["vy"])
    gx, gy = s.vcycle(T(bx), T(by), T(f["vx"]), T(f["vy"]))
    assert rel(gx, ex) <= TOL_OP and rel(gy, ey) <= TOL_OP


CASES = [
    ("mms", 32, dict(omega_v=0.6, alpha_p=1.5)),
    ("mms", 64, dict(omega_v=0.6, alpha_p=1.0, smoother=1)),
    ("block", 64, dict(omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=30)),
    ("layered", 128, dict(omega_v=0.6, alpha_p=1.0)),
    ("layered", 256, dict(omega_v=0.6, alpha_p=1.0, smoother=1)),
    ("solcx", 128, dict(omega_v=0.6, alpha_p=1.0, accel=1)),
    ("random", 128, dict(omega_v=0.6, alpha_p=1.0)),
]


def rounding_spread(n, w, opts, k):
    """The ORACLE's own sensitivity to rounding at a fixed iteration count k: the same k
    iterations with rho perturbed by ~1e-15 relative (a rounding-level change of the input).
    Krylov and Anderson recurrences amplify such differences; the GPU sums in a different
    (tree) order, so its fixed-count distance to the oracle is bounded by a small multiple of
    this measured spread."""
    rng = np.random.default_rng(99)
    w2 = dict(w, rho_b=w["rho_b"] * (1.0 + 1e-15 * rng.standard_normal(w["rho_b"].shape)))
    out = []
    for ww in (w, w2):
        o = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **dict(opts, max_iter=k))
        o.set_viscosity(ww["eta_b"], ww["eta_p"])
        o.set_density(ww["rho_b"])
        o.set_gravity(w["gx"], w["gy"])
        out.append(o.solve(0.0))
    return max(rel(out[1][key], out[0][key]) for key in ("vx", "vy", "p"))


@pytest.mark.parametrize("name,n,opts", CASES)
def test_solve_parity(S, name, n, opts):
    w = workload(name, n, n)
    o, s = pair(S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), **opts)
    a = o.solve(1e-8)
    b = s.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["iters"] - b["iters"]) <= 1, (a["iters"], b["iters"])
    assert b["E"] <= 1e-8  # the true residual's E (GCR: SURVEY Q13)
    # the converged GPU solution against the oracle's iterate at the SAME count (north_star:
    # <= 1e-9).  Uzawa iterates agree to rounding; GCR's Krylov recurrences amplify the
    # reduction order, so its bar is max(1e-9, 10x the oracle's own rounding spread).
    k = b["iters"]
    o2 = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **dict(opts, max_iter=k))
    o2.set_viscosity(w["eta_b"], w["eta_p"])
    o2.set_density(w["rho_b"])
    o2.set_gravity(w["gx"], w["gy"])
    a2 = o2.solve(0.0)
    bar = max(1e-9, 10 * rounding_spread(n, w, opts, k)) if opts.get("accel", 0) else 1e-9
    for key in ("vx", "vy", "p"):
        assert rel(b[key], a2[key]) <= bar, (key, rel(b[key], a2[key]), bar)
    # converged at equal (tight) residual tolerance -> <= 1e-9 (north_star bar)
    a3 = o.solve(1e-11)
    b3 = s.solve(1e-11)
    for key in ("vx", "vy", "p"):
        assert rel(b3[key], a3[key]) <= 1e-9, key


@pytest.mark.parametrize("true_restart", [0, 1])
def test_gcr_restart_readings(S, true_restart):
    """GCR restart from the true residual (R13, default) and the literal recursive one
    (Alg. 4): GPU = oracle iterate by iterate across restarts."""
    n = 64
    w = workload("solcx", n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=5, gcr_true_restart=true_restart)
    for k in (4, 5, 6, 11, 23):
        o, s = pair(S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), **dict(opts, max_iter=k))
        a, b = o.solve(0.0), s.solve(0.0)
        assert a["iters"] == b["iters"] == k
        assert abs(a["E"] - b["E"]) <= 1e-9 * a["E"]
        for key in ("vx", "vy", "p"):
            assert rel(b[key], a[key]) <= 1e-10, (k, key)


@pytest.mark.parametrize("name,n,opts", [
    ("block", 64, dict(aa_depth=5, aa_beta=0.7)),
    ("layered", 128, dict(aa_depth=10, aa_beta=1.0)),
    ("solcx", 128, dict(aa_depth=5, aa_beta=0.7, smoother=1)),
    ("random", 128, dict(aa_depth=0, aa_beta=1.0)),
])
def test_anderson_parity(S, name, n, opts):
    """Anderson AA(m, beta) (Alg. 5, reading R26).  Its iteration count is sensitive to
    rounding through the least squares: the ORACLE itself moves from 98 to 91 iterations on
    block 64^2 (m 5, beta .7) when rho is perturbed by 1e-15 relative.  So: the first 12
    iterates agree to 1e-8, the count within twice the oracle's own spread over four such
    perturbations (at least +-1), and the converged solutions (unique fixed point) to 1e-9."""
    opts = dict(opts, omega_v=0.6, alpha_p=1.0, accel=2)
    w = workload(name, n, n)
    args = (S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]))
    o, s = pair(*args, **dict(opts, max_iter=12))
    a, b = o.solve(0.0), s.solve(0.0)
    assert a["iters"] == b["iters"] == 12
    for key in ("vx", "vy", "p"):
        assert rel(b[key], a[key]) <= 1e-8, key
    o, s = pair(*args, **opts)
    a, b = o.solve(1e-8), s.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    # count band = the oracle's own spread under a rounding-level input change (the
    # least-squares history is ill-conditioned near convergence), at least +-1
    spread = 0
    for seed in range(4):
        w2 = dict(w, rho_b=w["rho_b"] * (1.0 + 1e-15 * np.random.default_rng(seed).standard_normal(w["rho_b"].shape)))
        o2 = Oracle(n, n, w["Lx"], w["Ly"], w["bc"], **opts)
        o2.set_viscosity(w2["eta_b"], w2["eta_p"])
        o2.set_density(w2["rho_b"])
        o2.set_gravity(w["gx"], w["gy"])
        spread = max(spread, abs(o2.solve(1e-8)["iters"] - a["iters"]))
    band = max(1, 2 * spread)
    assert abs(a["iters"] - b["iters"]) <= band, (a["iters"], b["iters"], band)
    a, b = o.solve(1e-11), s.solve(1e-11)
    for key in ("vx", "vy", "p"):
        assert rel(b[key], a[key]) <= 1e-9, key
    if opts["aa_depth"] == 0:  # m = 0, beta = 1 is the plain iteration: same count as Uzawa
        o2, s2 = pair(*args, omega_v=0.6, alpha_p=1.0)
        assert s2.solve(1e-8)["iters"] == s.solve(1e-8)["iters"]


@pytest.mark.parametrize("k", [1, 2, 3, 7])
@pytest.mark.parametrize("nx,ny", [(128, 32), (160, 136), (256, 64)])
def test_fused_uzawa_fixed_iterations(S, nx, ny, k):
    """Fine grids >= 128 x 8 run the Uzawa update fused into the next V-cycle's first sweep
    (a12); a fixed number of iterations must still give the oracle's (v^k, p^k, E^k)."""
    w = workload("layered", nx, ny)
    o, s = pair(S, nx, ny, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), omega_v=0.6, alpha_p=1.0,
                max_iter=k)
    a = o.solve(0.0)
    b = s.solve(0.0)
    assert a["iters"] == b["iters"] == k
    assert abs(a["E"] - b["E"]) <= 1e-9 * a["E"]
    for key in ("vx", "vy", "p"):
        assert rel(b[key], a[key]) <= 1e-10, key


@pytest.mark.parametrize("name,n,opts", [
    ("block", 64, dict(omega_v=0.6, alpha_p=1.0)),
    ("layered", 128, dict(omega_v=0.6, alpha_p=1.0)),
    ("layered", 256, dict(omega_v=0.6, alpha_p=1.0, smoother=1)),
    ("block", 128, dict(omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=20)),
])
def test_viscosity_rescaling_parity(S, name, n, opts):
    """theta stages 0, .25, .5, .75 of 10 iterations, then theta = 1 (PAPER.md:1771 with a
    shorter stage): same iteration count, same iterate at a fixed count, same fixed point."""
    opts = dict(opts, theta_step=0.25, theta_every=10)
    w = workload(name, n, n)
    o, s = pair(S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), **opts)
    a, b = o.solve(1e-8), s.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["iters"] - b["iters"]) <= 1 and a["iters"] >= 40
    k = a["iters"]
    o2, s2 = pair(S, n, n, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), **dict(opts, max_iter=k))
    a2, b2 = o2.solve(0.0), s2.solve(0.0)
    bar = 1e-8 if opts.get("accel", 0) else 1e-9
    for key in ("vx", "vy", "p"):
        assert rel(b2[key], a2[key]) <= bar, key
    eb, ep = s.get_viscosity(0)  # theta = 1 restored the caller's field exactly
    assert torch.equal(eb.cpu(), torch.from_numpy(w["eta_b"])) and torch.equal(ep.cpu(), torch.from_numpy(w["eta_p"]))


@pytest.mark.parametrize("smoother", [0, 1])
def test_sinker_paper_configuration_parity(S, smoother):
    """The paper's robustness setting at 100 x 120 cells: contrast 1e8,
    full density, sweep growth 2.5, coarsest by smoothing, omega_v 0.3, omega_p 0.6, theta
    stages every 25 iterations, lithostatic initial pressure; 150 iterations on both sides."""
    nx, ny = 100, 120
    w = workload("sinker", nx, ny)
    opts = dict(omega_v=0.3, alpha_p=0.6, nu_growth=2.5, coarse_direct=0, smoother=smoother, theta_step=0.25,
                theta_every=25, max_iter=150)
    o, s = pair(S, nx, ny, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), **opts)
    p0 = o.lithostatic()
    assert rel(s.lithostatic(), p0) <= 1e-13
    a = o.solve(0.0, p=p0)
    b = s.solve(0.0, p=torch.from_numpy(p0).cuda())
    assert a["iters"] == b["iters"] == 150
    assert abs(a["E"] - b["E"]) <= 1e-6 * a["E"]
    for key in ("vx", "vy", "p"):
        assert rel(b[key], a[key]) <= 1e-8, key


@pytest.mark.parametrize("nx,ny", [(33, 17), (256, 200)])
def test_lithostatic_parity(S, nx, ny):
    f = parity_fields(nx, ny)
    o, s = pair(S, nx, ny, (0, 1, 0, 1), f, 1.0, 0.7, (0.2, 1.3), coarse_direct=0)
    ex = o.lithostatic()
    got = s.lithostatic()
    assert rel(got, ex) <= 1e-13
    # the paper's initial guess: solve from (0, p_litho) on both sides
    w = workload("layered", 128, 128)
    o, s = pair(S, 128, 128, w["bc"], w, w["Lx"], w["Ly"], (w["gx"], w["gy"]), omega_v=0.6, alpha_p=1.0)
    p0 = o.lithostatic()
    a = o.solve(1e-8, p=p0)
    b = s.solve(1e-8, p=torch.from_numpy(p0).cuda())
    assert a["status"] == 0 and b["status"] == 0 and abs(a["iters"] - b["iters"]) <= 1


def test_error_paths(S):
    from paper_2603_14040_b200 import StokesError
    with pytest.raises(StokesError):
        S(1, 8)
    s = S(16, 16)
    with pytest.raises(StokesError):
        s.solve(1e-8)  # before set_viscosity
    eb = torch.ones(17, 17, dtype=torch.float64, device="cuda")
    ep = torch.ones(16, 16, dtype=torch.float64, device="cuda")
    ep[3, 3] = -1.0
    with pytest.raises(StokesError):
        s.set_viscosity(eb, ep)


def test_zero_force_and_wall_entries(S):
    n = 32
    f = parity_fields(n, n)
    o, s = pair(S, n, n, (0, 0, 0, 0), f, coarse_min=4)
    s.set_density(torch.zeros(n + 1, n + 1, dtype=torch.float64, device="cuda"))
    r = s.solve(1e-8, vx=T(f["vx"]))
    assert r["iters"] == 0 and float(r["vx"].abs().max()) == 0.0
    vx = f["vx"].copy()
    vx[:, [0, -1]] = np.nan
    a = s.apply_operator(T(f["vx"]), T(f["vy"]), T(f["p"]))
    b = s.apply_operator(T(vx), T(f["vy"]), T(f["p"]))
    for x, y in zip(a, b):
        assert torch.equal(x, y)
