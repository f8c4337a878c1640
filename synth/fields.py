"""Seeded synthetic input generators shared by the oracle tests, the GPU parity tests and
bench.py.  This module holds NO arithmetic of the method (no stencil, transfer, smoother
or solver step): it only samples viscosity / density / initial fields at the node
positions of the staggered grid (user layout of include/stokes.h).

User layout (no ghosts), nx x ny cells, dx = Lx/nx, dy = Ly/ny, y pointing down:
    eta_b, rho_b : (ny+1) x (nx+1)  basic node [i][j] at (j dx, i dy)
    eta_p, p     : ny x nx          P node     [i][j] at ((j+1/2) dx, (i+1/2) dy)
    vx           : ny x (nx+1)      vx node    [i][j] at (j dx, (i+1/2) dy)
    vy           : (ny+1) x nx      vy node    [i][j] at ((j+1/2) dx, i dy)

Every generator accepts an optional tile window (i0, j0) .. so that a rank of a 2D
decomposition can sample its own tile of a global field without building the whole
array; the values are identical to slicing the global field.

Workload recipes:
    mms      cfg 1  unit box, eta = 1, rho_b = -4 pi^3 cos(pi x) sin(pi y), g = (0, 1)
    block    cfg 2  unit box, eta = 1 outside / 1e3 inside [3/8, 5/8]^2 (edges inclusive),
                    drho = 1 inside, 0 outside
    solcx    cfg 3  eta = 1 for x < 1/2, 1e6 for x >= 1/2; rho_b = sin(pi y) cos(pi x)
    layered  cfg 4  per unit tile (x', y') = (x mod 1, y mod 1): eta = 1e3 (y' < 0.15),
                    1 (0.15 <= y' < 0.66), 30 (y' >= 0.66); drho = cos(2 pi x') sin(pi y')
    random   cfg 5  log10 eta = xi(x, y), xi = sum_k a_k cos(2 pi (m_k x + n_k y) + phi_k) / sum a_k,
                    k = 1..32 from numpy default_rng(2603); drho = sin(pi y) cos(pi x)
    parity   kernel-parity fields: log10 eta_b, log10 eta_p iid U(-3, 3) (default_rng(1)),
                    rho_b ~ U(-1, 1) (default_rng(2)), vx, vy, p ~ N(0, 1) (default_rng(3))
"""
import math

import numpy as np

WORKLOADS = ("mms", "block", "solcx", "layered", "random", "sinker", "parity")


def _coords(n, h, off, start=0, count=None):
    count = n if count is None else count
    return (np.arange(start, start + count, dtype=np.float64) + off) * h


def node_coords(kind, nx, ny, Lx, Ly, i0=0, j0=0, nyt=None, nxt=None):
    """1D coordinate vectors (y, x) of the nodes of `kind` ('b', 'p', 'vx', 'vy') in a window.

    Window sizes default to the full global array of that kind."""
    dx, dy = Lx / nx, Ly / ny
    full = {"b": (ny + 1, nx + 1), "p": (ny, nx), "vx": (ny, nx + 1), "vy": (ny + 1, nx)}[kind]
    ox = 0.5 if kind in ("p", "vy") else 0.0
    oy = 0.5 if kind in ("p", "vx") else 0.0
    nyt = full[0] - i0 if nyt is None else nyt
    nxt = full[1] - j0 if nxt is None else nxt
    return _coords(ny, dy, oy, i0, nyt), _coords(nx, dx, ox, j0, nxt)


def _grid(kind, nx, ny, Lx, Ly, win):
    y, x = node_coords(kind, nx, ny, Lx, Ly, *win)
    return y[:, None], x[None, :]


def _win(win):
    return tuple(win) if win is not None else (0, 0, None, None)


# ---------------------------------------------------------------- workloads
def mms_density(nx, ny, Lx=1.0, Ly=1.0, win=None):
    y, x = _grid("b", nx, ny, Lx, Ly, _win(win))
    return -4.0 * math.pi ** 3 * np.cos(math.pi * x) * np.sin(math.pi * y)


def _block_eta(y, x):
    inside = (x >= 3 / 8) & (x <= 5 / 8) & (y >= 3 / 8) & (y <= 5 / 8)
    return np.where(inside, 1e3, 1.0), np.where(inside, 1.0, 0.0)


def _sinker(y, x):
    """PAPER.md:1740-1759 nondimensionalised (length 100 km, viscosity 1e18 Pa s, density
    1000 kg/m^3, g = 10 m/s^2 -> 1): circular inclusion of radius 0.2 centred in the unit
    box, eta 1e8 / 1, FULL density 3.3 / 3.2 (no anomaly split: the lithostatic pressure
    initial guess of PAPER.md:1250 matters)."""
    inside = (x - 0.5) ** 2 + (y - 0.5) ** 2 <= 0.2 ** 2
    return np.where(inside, 1e8, 1.0), np.where(inside, 3.3, 3.2)


def _solcx_eta(y, x):
    return np.where(x >= 0.5, 1e6, 1.0) + 0.0 * y


def _layered_eta(y, x):
    yp = np.mod(y, 1.0) + 0.0 * x
    return np.where(yp < 0.15, 1e3, np.where(yp < 0.66, 1.0, 30.0))


def _layered_rho(y, x):
    return np.cos(2 * math.pi * np.mod(x, 1.0)) * np.sin(math.pi * np.mod(y, 1.0))


def random_modes(seed=2603, K=32):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, K)
    m = np.empty(K, np.int64)
    n = np.empty(K, np.int64)
    for k in range(K):
        while True:
            mk, nk = rng.integers(-16, 17, 2)
            if mk != 0 or nk != 0:
                break
        m[k], n[k] = mk, nk
    phi = rng.uniform(0.0, 2 * math.pi, K)
    return a, m, n, phi


def _random_log_eta(y, x, modes):
    a, m, n, phi = modes
    yy = y[:, 0]
    xx = x[0, :]
    acc = np.zeros((yy.size, xx.size))
    for k in range(a.size):
        # separable: cos(2pi(m x + n y) + phi) = Re(e^{i(2pi m x + phi)} e^{i 2pi n y})
        ex = np.exp(1j * (2 * math.pi * m[k] * xx + phi[k]))
        ey = np.exp(1j * (2 * math.pi * n[k] * yy))
        acc += a[k] * np.real(np.outer(ey, ex))
    return acc / a.sum()


def random_torch(nx, ny, Lx=1.0, Ly=1.0, win_b=None, win_p=None, device="cuda"):
    """The cfg-5 `random` workload (same recipe and modes as workload("random", ...)) sampled
    on the device with torch in FP64: log10 eta as the rank-2K product [cos(n y) sin(n y)]
    diag(a) [cos(m x + phi) -sin(m x + phi)]^T, for full-size (16384^2) bench inputs that
    numpy would need minutes for.  Equal to the numpy fields to rounding (not bit for bit)."""
    import torch
    a, m, n, phi = random_modes()
    at = torch.tensor(a, dtype=torch.float64, device=device)
    mt = torch.tensor(m, dtype=torch.float64, device=device)
    nt = torch.tensor(n, dtype=torch.float64, device=device)
    pt = torch.tensor(phi, dtype=torch.float64, device=device)

    def coords(kind, win):
        i0, j0, nyt, nxt = _win(win)
        y, x = node_coords(kind, nx, ny, Lx, Ly, i0, j0, nyt, nxt)
        return (torch.tensor(y, dtype=torch.float64, device=device),
                torch.tensor(x, dtype=torch.float64, device=device))

    def log_eta(y, x):
        ty = 2 * math.pi * torch.outer(y, nt)
        tx = 2 * math.pi * torch.outer(x, mt) + pt
        Y = torch.cat([torch.cos(ty), torch.sin(ty)], 1) * torch.cat([at, at])
        X = torch.cat([torch.cos(tx), -torch.sin(tx)], 1)
        return (Y @ X.T) / float(a.sum())

    yb, xb = coords("b", win_b)
    yp, xp = coords("p", win_p)
    eb = torch.pow(10.0, log_eta(yb, xb))
    ep = torch.pow(10.0, log_eta(yp, xp))
    rho = torch.outer(torch.sin(math.pi * yb), torch.cos(math.pi * xb))
    return {"eta_b": eb.contiguous(), "eta_p": ep.contiguous(), "rho_b": rho.contiguous(), "gx": 0.0, "gy": 1.0,
            "Lx": Lx, "Ly": Ly, "bc": (0, 0, 0, 0)}


def workload(name, nx, ny, Lx=None, Ly=None, win_b=None, win_p=None):
    """Return dict(eta_b, eta_p, rho_b, gx, gy, Lx, Ly, bc) of a workload (global or tile windows)."""
    if name == "layered":
        Lx = Lx if Lx is not None else 1.0
        Ly = Ly if Ly is not None else 1.0
    Lx = 1.0 if Lx is None else Lx
    Ly = 1.0 if Ly is None else Ly
    yb, xb = _grid("b", nx, ny, Lx, Ly, _win(win_b))
    yp, xp = _grid("p", nx, ny, Lx, Ly, _win(win_p))
    if name == "mms":
        eb = np.ones((yb.shape[0], xb.shape[1]))
        ep = np.ones((yp.shape[0], xp.shape[1]))
        rho = mms_density(nx, ny, Lx, Ly, win_b)
    elif name == "block":
        eb, rho = _block_eta(yb, xb)
        ep, _ = _block_eta(yp, xp)
    elif name == "solcx":
        eb = _solcx_eta(yb, xb)
        ep = _solcx_eta(yp, xp)
        rho = np.sin(math.pi * yb) * np.cos(math.pi * xb)
    elif name == "layered":
        eb = _layered_eta(yb, xb)
        ep = _layered_eta(yp, xp)
        rho = _layered_rho(yb, xb)
    elif name == "random":
        modes = random_modes()
        eb = 10.0 ** _random_log_eta(yb, xb, modes)
        ep = 10.0 ** _random_log_eta(yp, xp, modes)
        rho = np.sin(math.pi * yb) * np.cos(math.pi * xb)
    elif name == "sinker":
        eb, rho = _sinker(yb, xb)
        ep, _ = _sinker(yp, xp)
    elif name == "parity":
        f = parity_fields(nx, ny)
        eb, ep, rho = f["eta_b"], f["eta_p"], f["rho_b"]
    else:
        raise ValueError(f"unknown workload {name!r}; choose from {WORKLOADS}")
    return {"eta_b": np.ascontiguousarray(eb, np.float64), "eta_p": np.ascontiguousarray(ep, np.float64),
            "rho_b": np.ascontiguousarray(rho, np.float64), "gx": 0.0, "gy": 1.0, "Lx": Lx, "Ly": Ly,
            "bc": (0, 0, 0, 0)}


def parity_fields(nx, ny, log_contrast=3.0, seed_eta=1, seed_rho=2, seed_v=3):
    """Kernel-parity fields: iid log-uniform viscosity (contrast 10^(2*log_contrast)), uniform
    density, normal velocity / pressure."""
    r1 = np.random.default_rng(seed_eta)
    eta_b = 10.0 ** r1.uniform(-log_contrast, log_contrast, (ny + 1, nx + 1))
    eta_p = 10.0 ** r1.uniform(-log_contrast, log_contrast, (ny, nx))
    r2 = np.random.default_rng(seed_rho)
    rho_b = r2.uniform(-1.0, 1.0, (ny + 1, nx + 1))
    r3 = np.random.default_rng(seed_v)
    vx = r3.standard_normal((ny, nx + 1))
    vy = r3.standard_normal((ny + 1, nx))
    p = r3.standard_normal((ny, nx))
    return {"eta_b": eta_b, "eta_p": eta_p, "rho_b": rho_b, "vx": vx, "vy": vy, "p": p}


def random_velocity(nx, ny, seed=3):
    r = np.random.default_rng(seed)
    return r.standard_normal((ny, nx + 1)), r.standard_normal((ny + 1, nx)), r.standard_normal((ny, nx))


# ---------------------------------------------------------------- markers (NEXT-4)
MARKER_PROPS = {"sinker": _sinker, "block": _block_eta,
                "layered": lambda y, x: (_layered_eta(y, x), _layered_rho(y, x))}


def markers(nx, ny, Lx=1.0, Ly=1.0, per_side=4, jitter=1.0, seed=7, order="cell", props="sinker"):
    """Seeded marker cloud (recipe DESIGN.md §9d): a per_side x per_side lattice in every cell
    (the paper's 8-16 markers per cell: per_side 4 -> 16), each marker moved by
    a uniform jitter of +-jitter/2 lattice spacings (default_rng(seed)), clipped to the closed
    box; properties (eta_m, rho_m) sampled from a workload's continuous definition at the
    marker positions.  order: "cell" (cell-major, as seeded) or "shuffled" (a seeded random
    permutation, the worst case for locality)."""
    rng = np.random.default_rng(seed)
    dx, dy = Lx / nx, Ly / ny
    s = (np.arange(per_side) + 0.5) / per_side
    # cell-major: cell (i, j), then the lattice row a, column b inside it
    ci, cj, a, b = np.meshgrid(np.arange(ny), np.arange(nx), np.arange(per_side), np.arange(per_side),
                               indexing="ij")
    xm = (cj + s[b]) * dx
    ym = (ci + s[a]) * dy
    n = xm.size
    xm = xm.reshape(n) + (rng.random(n) - 0.5) * jitter * dx / per_side
    ym = ym.reshape(n) + (rng.random(n) - 0.5) * jitter * dy / per_side
    xm = np.clip(xm, 0.0, Lx)
    ym = np.clip(ym, 0.0, Ly)
    if order == "shuffled":
        perm = rng.permutation(n)
        xm, ym = xm[perm], ym[perm]
    eta_m, rho_m = MARKER_PROPS[props](ym, xm)
    return {"xm": np.ascontiguousarray(xm), "ym": np.ascontiguousarray(ym),
            "eta_m": np.ascontiguousarray(eta_m, np.float64), "rho_m": np.ascontiguousarray(rho_m, np.float64)}


def markers_torch(nx, ny, per_side=4, seed=2603, props="layered", device="cuda"):
    """The markers() lattice recipe generated ON THE GPU with a seeded torch generator (for
    full-size runs whose marker arrays are too large to build in numpy): cell-major order,
    per_side^2 per cell, uniform jitter of +-1/2 lattice spacing, unit box; properties from the
    same continuous definitions.  Returns torch float64 tensors (xm, ym, eta_m, rho_m)."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    dx, dy = 1.0 / nx, 1.0 / ny
    s = (torch.arange(per_side, device=device, dtype=torch.float64) + 0.5) / per_side
    ci = torch.arange(ny, device=device, dtype=torch.float64).view(ny, 1, 1, 1)
    cj = torch.arange(nx, device=device, dtype=torch.float64).view(1, nx, 1, 1)
    xm = ((cj + s.view(1, 1, 1, per_side)) * dx).expand(ny, nx, per_side, per_side).reshape(-1)
    ym = ((ci + s.view(1, 1, per_side, 1)) * dy).expand(ny, nx, per_side, per_side).reshape(-1)
    n = xm.numel()
    xm = (xm + (torch.rand(n, generator=g, device=device, dtype=torch.float64) - 0.5) * dx / per_side).clamp_(0, 1)
    ym = (ym + (torch.rand(n, generator=g, device=device, dtype=torch.float64) - 0.5) * dy / per_side).clamp_(0, 1)
    one = torch.ones_like(xm)
    if props == "layered":  # the _layered_eta / _layered_rho definitions, evaluated with torch
        yp, xp = torch.remainder(ym, 1.0), torch.remainder(xm, 1.0)
        eta = torch.where(yp < 0.15, 1e3 * one, torch.where(yp < 0.66, one, 30.0 * one))
        rho = torch.cos(2 * math.pi * xp) * torch.sin(math.pi * yp)
    elif props == "block":
        inside = (xm >= 3 / 8) & (xm <= 5 / 8) & (ym >= 3 / 8) & (ym <= 5 / 8)
        eta, rho = torch.where(inside, 1e3 * one, one), torch.where(inside, one, 0.0 * one)
    elif props == "sinker":
        inside = (xm - 0.5) ** 2 + (ym - 0.5) ** 2 <= 0.2 ** 2
        eta, rho = torch.where(inside, 1e8 * one, one), torch.where(inside, 3.3 * one, 3.2 * one)
    else:
        raise ValueError(props)
    return xm.contiguous(), ym.contiguous(), eta.contiguous(), rho.contiguous()
