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


@pytest.mark.parametrize("transport", ["virtual", "loopback"])
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


def test_loopback_large_tiles_stream_path():
    """256-wide tiles take the TMA streaming kernels on the distributed levels."""
    from paper_2603_14040_b200 import Stokes, StokesDist
    n = 512
    w = workload("layered", n, n)
    opts = dict(omega_v=0.6, alpha_p=1.0, max_iter=3)
    a = setup(Stokes, w, n, **opts).solve(0.0)
    b = setup(StokesDist, w, n, px=2, py=2, transport="loopback", **opts).solve(0.0)
    for k in ("vx", "vy", "p"):
        assert rel(b[k], a[k]) <= 1e-12, k


def test_decomposition_errors():
    from paper_2603_14040_b200 import StokesDist, StokesError
    with pytest.raises(StokesError):
        StokesDist(130, 64, px=4, py=1)  # 130 % 4 != 0
    with pytest.raises(StokesError):
        StokesDist(64, 64, px=2, py=2, accel=1)  # GCR not decomposed


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
        assert abs(a["iters"] - b["iters"]) <= 1
        for k in ("vx", "vy", "p"):
            assert rel(b[k], a[k]) <= 1e-6, k
    finally:
        if own:
            dist.destroy_process_group()
