"""GPU parity of the marker-in-cell kernels (csrc/markers.cu) against
the CPU oracle (oracle/markers_oracle.c), through the C ABI.

Bar: BIT-EXACT.  Both sides take every rounding in the same order (the node sums of
marker -> grid in ascending marker index, products and sums without FMA contraction), so
every output double, the empty-node count and the clamped-marker count must be identical.
Cases: ragged grids (8x6, 33x17, 130x66), random / cell-ordered / shuffled markers, markers
on walls and node lines, a crowded cell (long bins), an empty pool, all BCs, the three
integrators with clamping; at full size 2048^2 x 16 markers (the paper's 8-16 per cell,
PAPER.md:2263) the whole marker -> grid output and an RK4 step of a 1M-marker sample.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from synth.fields import markers, parity_fields  # noqa: E402

BCS = [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 1, 0)]


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2603_14040_b200 import Stokes
    return Stokes


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


def H(t):
    return t.detach().cpu().numpy()


def random_pool(nx, ny, Lx, Ly, n, seed, crowd=0):
    rng = np.random.default_rng(seed)
    xm, ym = rng.random(n) * Lx, rng.random(n) * Ly
    if n >= 6:
        xm[:6] = [0.0, Lx, 2 * Lx / nx, Lx / nx * 0.5, -0.1, Lx * 1.2]   # walls, node line, outside (clamped)
        ym[:6] = [Ly, 0.0, Ly / ny, 0.5 * Ly / ny, 0.3 * Ly, -1.0]
    if crowd:                                  # many markers in one cell: long bins
        xm[-crowd:] = (nx // 2 + rng.random(crowd)) * Lx / nx
        ym[-crowd:] = (ny // 3 + rng.random(crowd)) * Ly / ny
    return xm, ym, 10.0 ** rng.uniform(-3, 3, n), rng.normal(size=n)


def check_m2g(S, nx, ny, Lx, Ly, xm, ym, eta, rho):
    s = S(nx, ny, Lx, Ly)
    eb, ep, rb, ne = s.markers_to_grid(T(xm), T(ym), T(eta), T(rho))
    reb, rep, rrb, rne = O.markers_to_grid(nx, ny, Lx, Ly, xm, ym, eta, rho)
    assert ne == rne
    assert np.array_equal(H(eb), reb)
    assert np.array_equal(H(ep), rep)
    assert np.array_equal(H(rb), rrb)
    return s


@pytest.mark.parametrize("nx,ny,Lx,Ly,n,crowd", [(8, 6, 1.0, 1.0, 400, 0), (33, 17, 2.0, 0.7, 3000, 500),
                                                 (130, 66, 1.0, 1.0, 20000, 2000), (5, 3, 1.0, 1.0, 7, 0)])
def test_m2g_random_bitexact(S, nx, ny, Lx, Ly, n, crowd):
    check_m2g(S, nx, ny, Lx, Ly, *random_pool(nx, ny, Lx, Ly, n, nx + ny, crowd))


@pytest.mark.parametrize("order", ["cell", "shuffled"])
@pytest.mark.parametrize("nx,ny", [(33, 17), (256, 128)])
def test_m2g_lattice_bitexact(S, nx, ny, order):
    m = markers(nx, ny, 1.0, 1.0, per_side=4, seed=nx, order=order, props="sinker")
    check_m2g(S, nx, ny, 1.0, 1.0, m["xm"], m["ym"], m["eta_m"], m["rho_m"])


def test_m2g_empty_pool(S):
    s = S(8, 8)
    z = torch.zeros(0, dtype=torch.float64, device="cuda")
    eb, ep, rb, ne = s.markers_to_grid(z, z, z, z)
    assert ne == 81 + 64 and not eb.any() and not ep.any() and not rb.any()


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("nx,ny", [(8, 6), (33, 17), (130, 66)])
def test_g2m_bitexact(S, nx, ny, bc):
    f = parity_fields(nx, ny)
    xm, ym, _, _ = random_pool(nx, ny, 1.0, 0.7, 5000, 3)
    s = S(nx, ny, 1.0, 0.7, bc)
    um, vm = s.grid_to_markers(T(xm), T(ym), T(f["vx"]), T(f["vy"]))
    ru, rv = O.grid_to_markers(nx, ny, 1.0, 0.7, bc, xm, ym, f["vx"], f["vy"])
    assert np.array_equal(H(um), ru) and np.array_equal(H(vm), rv)


@pytest.mark.parametrize("scheme", ["euler", "heun", "rk4", "lpi2", "lpi3"])
@pytest.mark.parametrize("bc", BCS)
def test_advect_bitexact(S, scheme, bc):
    nx, ny = 33, 17
    f = parity_fields(nx, ny)
    xm, ym, _, _ = random_pool(nx, ny, 1.0, 0.7, 20000, 4)
    s = S(nx, ny, 1.0, 0.7, bc)
    dt = s.marker_timestep(T(f["vx"]), T(f["vy"]), 0.5, 1.0)
    assert dt == O.marker_timestep(nx, ny, 1.0, 0.7, f["vx"], f["vy"], 0.5, 1.0)
    for step_dt in (dt, 8 * dt):                      # 8x the CFL step pushes markers out: clamping
        gx, gy = T(xm), T(ym)
        nc = s.advect_markers(gx, gy, T(f["vx"]), T(f["vy"]), step_dt, scheme)
        rx, ry, rnc = O.advect_markers(nx, ny, 1.0, 0.7, bc, xm, ym, f["vx"], f["vy"], step_dt, scheme)
        assert nc == rnc
        assert np.array_equal(H(gx), rx) and np.array_equal(H(gy), ry)


def test_timestep_zero_field(S):
    s = S(16, 8)
    z = torch.zeros(8, 17, dtype=torch.float64, device="cuda")
    w = torch.zeros(9, 16, dtype=torch.float64, device="cuda")
    assert s.marker_timestep(z, w, 0.5, 2.5) == 2.5


def test_marker_errors(S):
    s = S(8, 8)
    x = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        s.advect_markers(x, x.clone(), torch.zeros(8, 9, dtype=torch.float64, device="cuda"),
                         torch.zeros(9, 8, dtype=torch.float64, device="cuda"), 0.1, "rk5")
    with pytest.raises(Exception):
        s.marker_timestep(torch.zeros(8, 9, dtype=torch.float64, device="cuda"),
                          torch.zeros(9, 8, dtype=torch.float64, device="cuda"), -1.0, 1.0)


def test_fullsize_2048(S):
    """2048^2 cells x 16 markers (67M): the whole marker -> grid output bit-exact; one RK4
    step of a 1M-marker sample bit-exact (advection is independent per marker)."""
    nx = ny = 2048
    m = markers(nx, ny, 1.0, 1.0, per_side=4, seed=2048, order="cell", props="sinker")
    s = check_m2g(S, nx, ny, 1.0, 1.0, m["xm"], m["ym"], m["eta_m"], m["rho_m"])
    rng = np.random.default_rng(1)
    vx = rng.normal(size=(ny, nx + 1))
    vy = rng.normal(size=(ny + 1, nx))
    idx = np.sort(rng.choice(m["xm"].size, 1 << 20, replace=False))
    xs, ys = m["xm"][idx], m["ym"][idx]
    dt = s.marker_timestep(T(vx), T(vy), 0.5, 1.0)
    gx, gy = T(xs), T(ys)
    nc = s.advect_markers(gx, gy, T(vx), T(vy), dt, "rk4")
    rx, ry, rnc = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), xs, ys, vx, vy, dt, "rk4")
    assert nc == rnc and np.array_equal(H(gx), rx) and np.array_equal(H(gy), ry)


def test_mic_cycle_matches_oracle(S):
    """The paper's simulation loop (steps 1-4) twice on the block at 64^2:
    markers -> grid (bit-exact), Stokes solve (parity bar 1e-9 relative), CFL step, RK4."""
    nx = ny = 64
    m = markers(nx, ny, 1.0, 1.0, per_side=4, seed=5, order="cell", props="block")
    opts = dict(omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=30)
    s = S(nx, ny, 1.0, 1.0, **opts)
    gx, gy = T(m["xm"]), T(m["ym"])
    ox, oy = m["xm"].copy(), m["ym"].copy()
    eta, rho = m["eta_m"], m["rho_m"]
    for _ in range(2):
        eb, ep, rb, ne = s.markers_to_grid(gx, gy, T(eta), T(rho))
        reb, rep, rrb, rne = O.markers_to_grid(nx, ny, 1.0, 1.0, ox, oy, eta, rho)
        assert ne == rne == 0
        np.testing.assert_allclose(H(eb), reb, rtol=1e-9)
        s.set_viscosity(eb, ep)
        s.set_density(rb)
        s.set_gravity(0.0, 1.0)
        g = s.solve(1e-10)
        o = O.Oracle(nx, ny, 1.0, 1.0, (0, 0, 0, 0), **opts)
        o.set_viscosity(reb, rep)
        o.set_density(rrb)
        o.set_gravity(0.0, 1.0)
        r = o.solve(1e-10)
        for k in ("vx", "vy"):
            assert np.linalg.norm(H(g[k]) - r[k]) <= 1e-8 * np.linalg.norm(r[k])
        dt = s.marker_timestep(g["vx"], g["vy"], 0.5, 1e9)
        rdt = O.marker_timestep(nx, ny, 1.0, 1.0, r["vx"], r["vy"], 0.5, 1e9)
        assert abs(dt - rdt) <= 1e-8 * rdt
        s.advect_markers(gx, gy, g["vx"], g["vy"], dt, "rk4")
        ox, oy, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), ox, oy, r["vx"], r["vy"], rdt, "rk4")
        assert np.max(np.abs(H(gx) - ox)) <= 1e-9 and np.max(np.abs(H(gy) - oy)) <= 1e-9


def test_mic_block_sinks(S):
    """Three steps of the MIC loop with the dense block (Delta rho = 1,
    eta 1e3, BASELINE cfg 2 recipe) carried by markers: the block's markers move DOWN (+y,
    gravity along +y, reading R4), stay centred in x (the problem is mirror-symmetric), no
    marker leaves the box, and the CFL step keeps every displacement below half a cell."""
    nx = ny = 64
    m = markers(nx, ny, 1.0, 1.0, per_side=4, seed=9, order="cell", props="block")
    s = S(nx, ny, 1.0, 1.0, omega_v=0.6, alpha_p=1.0, accel=1, gcr_restart=30)
    s.set_gravity(0.0, 1.0)
    gx, gy = T(m["xm"]), T(m["ym"])
    eta, rho = T(m["eta_m"]), T(m["rho_m"])
    inside = torch.from_numpy(m["eta_m"] > 10).cuda()
    y0 = gy[inside].mean().item()
    x0 = gx[inside].mean().item()
    r = None
    for _ in range(3):
        eb, ep, rb, ne = s.markers_to_grid(gx, gy, eta, rho)
        assert ne == 0
        s.set_viscosity(eb, ep)
        s.set_density(rb)
        r = s.solve(1e-10, *((r["vx"], r["vy"], r["p"]) if r else ()))
        assert r["status"] == 0
        dt = s.marker_timestep(r["vx"], r["vy"], 0.5, 1e9)
        px, py = gx.clone(), gy.clone()
        assert s.advect_markers(gx, gy, r["vx"], r["vy"], dt, "rk4") == 0
        assert (gx - px).abs().max().item() <= 0.5 / nx + 1e-12
        assert (gy - py).abs().max().item() <= 0.5 / ny + 1e-12
    y1 = gy[inside].mean().item()
    x1 = gx[inside].mean().item()
    assert y1 > y0 + 1e-4, (y0, y1)
    assert abs(x1 - x0) < 0.05 * (y1 - y0), (x0, x1, y0, y1)  # jittered markers: nearly symmetric


def test_fullsize_4096_window(S):
    """The measured configuration (tools/mic_bench.py: 4096^2 cells x 16 markers = 268 M, one
    launch of each kernel): marker -> grid bit-exact on the nodes of a 48^2-cell window, from the
    oracle run on the window's markers alone (a node's value depends only on the markers of its
    four surrounding cells, added in ascending index -- a subset in the same order gives the
    same bits); RK4 bit-exact on the window's markers."""
    from synth.fields import markers_torch
    nx = ny = 4096
    xm, ym, eta, rho = markers_torch(nx, ny, per_side=4, seed=2603, props="layered")
    s = S(nx, ny, 1.0, 1.0)
    eb, ep, rb, ne = s.markers_to_grid(xm, ym, eta, rho)
    assert ne == 0
    c0, W = 2000, 48                      # window cells [c0, c0 + W)^2 (+2-cell margin for the subset)
    lo, hi = (c0 - 2) / nx, (c0 + W + 2) / nx
    sel = ((xm >= lo) & (xm <= hi) & (ym >= lo) & (ym <= hi)).nonzero().squeeze(1)   # ascending index
    sx, sy, se, sr = (H(t[sel]) for t in (xm, ym, eta, rho))
    reb, rep, rrb, _ = O.markers_to_grid(nx, ny, 1.0, 1.0, sx, sy, se, sr)
    win_b = (slice(c0, c0 + W + 1), slice(c0, c0 + W + 1))     # basic nodes with all 4 cells inside
    win_p = (slice(c0, c0 + W), slice(c0, c0 + W))             # P nodes with all 4 P-cells inside
    assert np.array_equal(H(eb)[win_b], reb[win_b]) and np.array_equal(H(rb)[win_b], rrb[win_b])
    assert np.array_equal(H(ep)[win_p], rep[win_p])
    rng = np.random.default_rng(4)
    vx = rng.normal(size=(ny, nx + 1))
    vy = rng.normal(size=(ny + 1, nx))
    gvx, gvy = T(vx), T(vy)
    dt = s.marker_timestep(gvx, gvy, 0.5, 1.0)
    s.advect_markers(xm, ym, gvx, gvy, dt, "rk4", count_clamped=False)
    ox, oy, _ = O.advect_markers(nx, ny, 1.0, 1.0, (0, 0, 0, 0), sx, sy, vx, vy, dt, "rk4")
    assert np.array_equal(H(xm[sel]), ox) and np.array_equal(H(ym[sel]), oy)
