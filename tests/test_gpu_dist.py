"""2D domain decomposition on ONE B200: the VIRTUAL decomposition runs all
px x py tiles in one process (halo strips copied between the tiles' buffers, coarse tail
agglomerated) and must reproduce the single-domain solve -- the same iteration count and
the same fields to rounding -- since the decomposition is exact by construction."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth.fields import workload  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def small_tiles():
    old = os.environ.get("STOKES_DIST_DMIN")
    os.environ["STOKES_DIST_DMIN"] = "8"  # distribute down to 8x8 tiles (many levels)
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    yield
    if old is None:
        os.environ.pop("STOKES_DIST_DMIN")
    else:
        os.environ["STOKES_DIST_DMIN"] = old


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel(a, b):
    a, b = a.cpu().numpy(), b.cpu().numpy()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(cls, w, n, **kw):
    s = cls(n, n, w["Lx"], w["Ly"], w["bc"], **kw)
    s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    s.set_density(T(w["rho_b"]))
    s.set_gravity(w["gx"], w["gy"])
    return s


TRANSPORTS = ["virtual", "loopback", "nccl_self"]


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2), (4, 2)])
@pytest.mark.parametrize("name,smoother", [("layered", 0), ("mms", 0), ("block", 1)])
def test_virtual_decomposition_is_exact(px, py, name, smoother, transport):
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 128
    w = workload(name, n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, smoother=smoother, max_iter=400)
    one = setup(Stokes, w, n, **opts)
    dd = setup(StokesDist, w, n, px=px, py=py, transport=transport, **opts)
    a = one.solve(1e-8)
    b = dd.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["iters"] - b["iters"]) <= 1, (a["iters"], b["iters"])
    # equal iteration count -> same iterate (decomposition is exact up to sum order)
    one2 = setup(Stokes, w, n, **dict(opts, max_iter=a["iters"]))
    dd2 = setup(StokesDist, w, n, px=px, py=py, transport=transport, **dict(opts, max_iter=a["iters"]))
    a2, b2 = one2.solve(0.0), dd2.solve(0.0)
    for k in ("vx", "vy", "p"):
        assert rel(b2[k], a2[k]) <= 1e-11, (k, rel(b2[k], a2[k]))
    _, _, _, e1 = one.residual(a["vx"], a["vy"], a["p"])
    _, _, _, e2 = dd.residual(a["vx"], a["vy"], a["p"])
    # E is a squared residual norm: at a converged state each residual entry is a cancellation
    # of stencil terms ~ eta_max |v| / h^2 ~ n^2 * contrast * |f| (1e3 * 128^2 here), so the two
    # kernels' (stream vs 2D-block) rounding may differ by ~eps * 1.6e7 ~ 4e-9 in sqrt(E) units
    assert abs(np.sqrt(e1) - np.sqrt(e2)) <= 1e-8, (e1, e2)


@pytest.fixture(params=["0", "1"], ids=["serial", "overlap"])
def overlap(request, monkeypatch):
    """STOKES_DIST_OVERLAP (read when a decomposed handle is created): 1 = boundary strips
    first, their halo exchange on a comm stream while the interior is swept."""
    monkeypatch.setenv("STOKES_DIST_OVERLAP", request.param)
    return request.param


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("px,py", [(2, 2), (4, 2), (1, 3)])
def test_fused_tile_kernels_fixed_iterations(transport, px, py, overlap):
    """Tiles >= 128 cells wide run the single-domain fused kernels with width-2 halos: the
    two-sweep pass (which also updates the first halo ring), the residual fused with its
    restriction and the fused Uzawa pass (a12).  A fixed number of iterations must equal the
    single-domain iterate to rounding (the decomposition is exact)."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    nx, ny = 128 * px * 2, 96 * py * 2
    w = workload("layered", nx, ny)
    opts = dict(omega_v=0.6, alpha_p=1.0, max_iter=4)
    s1 = Stokes(nx, ny, w["Lx"], w["Ly"], w["bc"], **opts)
    for s in (s1,):
        s.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
        s.set_density(T(w["rho_b"]))
        s.set_gravity(w["gx"], w["gy"])
    dd = StokesDist(nx, ny, w["Lx"], w["Ly"], w["bc"], px=px, py=py, transport=transport, **opts)
    dd.set_viscosity(T(w["eta_b"]), T(w["eta_p"]))
    dd.set_density(T(w["rho_b"]))
    dd.set_gravity(w["gx"], w["gy"])
    a, b = s1.solve(0.0), dd.solve(0.0)
    assert a["iters"] == b["iters"] == 4
    assert abs(a["E"] - b["E"]) <= 1e-11 * a["E"]
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-12, (k, rel(b[k], a[k]))


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("name,px,py", [("layered", 2, 2), ("random", 4, 2), ("block", 2, 1)])
def test_fused_tile_solve_counts_identical(transport, name, px, py, overlap):
    """Converged solves at 512 x 512 (256 x 256 .. 128 x 256 tiles, every distributed level on
    the fused kernels down to the agglomeration): the same iteration count as one domain, the
    same fields to 1e-11 (north_star count / field bars; the decomposition changes only the
    order of the global sums)."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 512
    w = workload(name, n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, max_iter=2000)
    a = setup(Stokes, w, n, **opts).solve(1e-8)
    b = setup(StokesDist, w, n, px=px, py=py, transport=transport, **opts).solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    assert a["iters"] == b["iters"], (a["iters"], b["iters"])
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-11, (k, rel(b[k], a[k]))


def test_decomposition_errors():
    from paper_2603_14040_b200 import StokesDist, StokesError
    with pytest.raises(StokesError):
        StokesDist(130, 64, px=4, py=1)  # 130 % 4 != 0
    with pytest.raises(StokesError):
        StokesDist(64, 64, px=2, py=2, smoother=2)  # RAS: single domain only


def test_nccl_transport_single_rank():
    """The NCCL transport on a 1 x 1 process grid (world size 1): NCCL communicator, graph-
    captured ncclAllReduce / ncclAllGather of the agglomeration, tile windows -- everything
    but the peer send/recv, which needs a second GPU.  Must equal the single-domain solve."""
    import torch.distributed as dist
    from paper_2603_14040_b200 import Stokes, StokesDist
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29561", rank=0, world_size=1)
    try:
        n = 256
        w = workload("layered", n, n)
        opts = dict(omega_v=0.6, alpha_p=1.0, max_iter=400)
        one = setup(Stokes, w, n, **opts)
        dd = setup(StokesDist, w, n, px=1, py=1, rank=0, **opts)
        a, b = one.solve(1e-8), dd.solve(1e-8)
        assert a["status"] == 0 and b["status"] == 0
        assert a["iters"] == b["iters"]
        for k in ("vx", "vy", "p"):
            assert rel(b[k], a[k]) <= 1e-11, k
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("transport", TRANSPORTS)
def test_overlapped_passes_large_tiles(transport, monkeypatch):
    """2 x 2 tiles of 1024^2 (the sizes where the overlapped exchange really runs beside the
    interior kernels): 3 iterations equal the single domain to rounding."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    monkeypatch.setenv("STOKES_DIST_OVERLAP", "1")
    monkeypatch.setenv("STOKES_DIST_DMIN", "128")
    n = 2048
    w = workload("layered", n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, max_iter=3)
    a = setup(Stokes, w, n, **opts).solve(0.0)
    b = setup(StokesDist, w, n, px=2, py=2, transport=transport, **opts).solve(0.0)
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-12, (k, rel(b[k], a[k]))


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("px,py", [(2, 1), (2, 2), (4, 2)])
@pytest.mark.parametrize("name,m", [("solcx", 10), ("block", 30)])
def test_gcr_on_tiles(transport, px, py, name, m):
    """Flexible GCR(m) (Alg. 4) on the tiles: the distributed V-cycle as preconditioner, the
    fused PrecondApplyOp / MGS / update kernels per tile with the GLOBAL inner products
    (every tile's per-CTA partials reduced in one fixed order).  Against the single-domain
    GCR: the same iteration count at rtol 1e-8, the iterates at a fixed count within the
    Krylov recurrences' rounding amplification (1e-8), and the converged solutions (unique)
    to 1e-9 at rtol 1e-11."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 128
    w = workload(name, n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=m)
    for k in (3, 12):
        a = setup(Stokes, w, n, max_iter=k, **opts).solve(0.0)
        b = setup(StokesDist, w, n, px=px, py=py, transport=transport, max_iter=k, **opts).solve(0.0)
        assert a["iters"] == b["iters"] == k
        for q in ("vx", "vy", "p"):
            assert rel(b[q], a[q]) <= 1e-8, (k, q, rel(b[q], a[q]))
    one = setup(Stokes, w, n, max_iter=2000, **opts)
    dd = setup(StokesDist, w, n, px=px, py=py, transport=transport, max_iter=2000, **opts)
    a, b = one.solve(1e-8), dd.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    assert abs(a["iters"] - b["iters"]) <= 1, (a["iters"], b["iters"])
    assert b["E"] <= 1e-8
    a, b = one.solve(1e-11), dd.solve(1e-11)
    for q in ("vx", "vy", "p"):
        assert rel(b[q], a[q]) <= 1e-9, (q, rel(b[q], a[q]))


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("px,py", [(2, 1), (2, 2)])
@pytest.mark.parametrize("name,m,beta", [("layered", 5, 0.7), ("block", 10, 1.0)])
def test_anderson_on_tiles(transport, px, py, name, m, beta):
    """Anderson AA(m, beta) (Alg. 5) on the tiles: G = the decomposed plain Uzawa iteration,
    the push / solve / update kernels per tile with the global Gram row and pressure mean.
    Against the single-domain AA: the first 8 iterates within 1e-8 (the least squares amplify
    the order of the sums), both converge at rtol 1e-8, and the converged solutions (the
    unique fixed point) agree to 1e-9 at rtol 1e-11."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 128
    w = workload(name, n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, accel=2, aa_depth=m, aa_beta=beta)
    a = setup(Stokes, w, n, max_iter=8, **opts).solve(0.0)
    b = setup(StokesDist, w, n, px=px, py=py, transport=transport, max_iter=8, **opts).solve(0.0)
    assert a["iters"] == b["iters"] == 8
    for q in ("vx", "vy", "p"):
        assert rel(b[q], a[q]) <= 1e-8, (q, rel(b[q], a[q]))
    one = setup(Stokes, w, n, max_iter=3000, **opts)
    dd = setup(StokesDist, w, n, px=px, py=py, transport=transport, max_iter=3000, **opts)
    a, b = one.solve(1e-8), dd.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0 and b["E"] <= 1e-8
    assert abs(a["iters"] - b["iters"]) <= max(2, a["iters"] // 5), (a["iters"], b["iters"])
    a, b = one.solve(1e-11), dd.solve(1e-11)
    for q in ("vx", "vy", "p"):
        assert rel(b[q], a[q]) <= 1e-9, (q, rel(b[q], a[q]))


@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("px,py", [(2, 1), (2, 2)])
@pytest.mark.parametrize("accel", [0, 1])
def test_viscosity_stages_on_tiles(transport, px, py, accel):
    """Viscosity-rescaling continuation (reading R24) on the tiles: eta_min reduced over every
    tile (ncclMin on the bit patterns under NCCL), the blended fine viscosity, its coarse
    hierarchy and the tail's coarsest inverse rebuilt per stage, the stages' iterations without
    a stopping test, then theta = 1 to the tolerance.  Uzawa: the decomposition is exact (the
    same count, fields 1e-11); GCR: counts +-1, converged fields 1e-9."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 128
    w = workload("block", n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, theta_step=0.25, theta_every=6, accel=accel, gcr_restart=30)
    one = setup(Stokes, w, n, max_iter=3000, **opts)
    dd = setup(StokesDist, w, n, px=px, py=py, transport=transport, max_iter=3000, **opts)
    a, b = one.solve(1e-8), dd.solve(1e-8)
    assert a["status"] == 0 and b["status"] == 0
    if accel == 0:
        assert a["iters"] == b["iters"], (a["iters"], b["iters"])
        for q in ("vx", "vy", "p"):
            assert rel(b[q], a[q]) <= 1e-11, (q, rel(b[q], a[q]))
    else:
        assert abs(a["iters"] - b["iters"]) <= 1, (a["iters"], b["iters"])
        a, b = one.solve(1e-11), dd.solve(1e-11)
        for q in ("vx", "vy", "p"):
            assert rel(b[q], a[q]) <= 1e-9, (q, rel(b[q], a[q]))
