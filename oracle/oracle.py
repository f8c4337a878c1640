"""ctypes wrapper of the CPU oracle (oracle/stokes_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.

Arrays use the user layout of the C-ABI (no ghosts), FP64 C-contiguous numpy:
    vx: ny x (nx+1)   vy: (ny+1) x nx   p, eta_p: ny x nx   eta_b, rho_b: (ny+1) x (nx+1)
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stokes_oracle.c")
_SRC_MARKERS = os.path.join(_HERE, "markers_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, NOT_CONVERGED, EINVAL, ENOMEM, EDIVERGED, ESTATE = 0, 1, -1, -2, -5, -6


def build(force=False):
    """Compile the oracle (plain C, -O2 -ffp-contract=off, single thread)."""
    srcs = [_SRC, _SRC_MARKERS]
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in srcs):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, *srcs, "-lm"])
    return _LIB


class Opts(ctypes.Structure):
    _fields_ = [
        ("smoother", ctypes.c_int),
        ("omega_v", ctypes.c_double),
        ("alpha_p", ctypes.c_double),
        ("nu1", ctypes.c_int),
        ("nu_growth", ctypes.c_double),
        ("coarse_min", ctypes.c_int),
        ("coarse_direct", ctypes.c_int),
        ("vcycles_per_iter", ctypes.c_int),
        ("accel", ctypes.c_int),
        ("gcr_restart", ctypes.c_int),
        ("max_iter", ctypes.c_int),
        ("pressure_sign", ctypes.c_int),
        ("theta_step", ctypes.c_double),
        ("theta_every", ctypes.c_int),
        ("aa_depth", ctypes.c_int),
        ("aa_beta", ctypes.c_double),
        ("ras_tile", ctypes.c_int),
        ("ras_inner", ctypes.c_int),
        ("ras_seed", ctypes.c_uint64),
        ("gcr_true_restart", ctypes.c_int),
        ("gcr_inner", ctypes.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        D = ctypes.POINTER(ctypes.c_double)
        I = ctypes.POINTER(ctypes.c_int)
        L = _lib
        L.oracle_opts_default.argtypes = [ctypes.POINTER(Opts)]
        L.oracle_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, I,
                                    ctypes.POINTER(Opts), ctypes.POINTER(P)]
        L.oracle_destroy.argtypes = [P]
        L.oracle_num_levels.argtypes = [P]
        L.oracle_level_shape.argtypes = [P, ctypes.c_int, I, I, I]
        L.oracle_set_viscosity.argtypes = [P, D, D]
        L.oracle_set_density.argtypes = [P, D]
        L.oracle_set_gravity.argtypes = [P, ctypes.c_double, ctypes.c_double]
        L.oracle_set_force.argtypes = [P, D, D]
        L.oracle_get_viscosity.argtypes = [P, ctypes.c_int, D, D]
        L.oracle_apply_operator.argtypes = [P, D, D, D, D, D, D]
        L.oracle_residual.argtypes = [P, D, D, D, D, D, D, D]
        L.oracle_residual_ld.argtypes = [P, D, D, D, D, D, D, D]
        L.oracle_energy_sums.argtypes = [P, D, D, D, D]
        L.oracle_vcycle.argtypes = [P, D, D, D, D]
        L.oracle_smooth.argtypes = [P, ctypes.c_int, D, D, D, D, ctypes.c_int]
        L.oracle_level_residual.argtypes = [P, ctypes.c_int, D, D, D, D, D, D]
        L.oracle_restrict.argtypes = [P, ctypes.c_int, ctypes.c_int, D, D]
        L.oracle_prolong.argtypes = [P, ctypes.c_int, D, D, D, D]
        L.oracle_coarse_solve.argtypes = [P, D, D, D, D]
        L.oracle_solve_hist.argtypes = [P, ctypes.c_double, D, D, D, I, D, D, ctypes.c_int]
        L.oracle_blend_viscosity.argtypes = [P, ctypes.c_double]
        L.oracle_lithostatic.argtypes = [P, D]
        L.oracle_strerror.restype = ctypes.c_char_p
        LL = ctypes.c_longlong
        PL = ctypes.POINTER(ctypes.c_longlong)
        i, d = ctypes.c_int, ctypes.c_double
        L.oracle_markers_to_grid.argtypes = [i, i, d, d, LL, D, D, D, D, D, D, D, PL]
        L.oracle_grid_to_markers.argtypes = [i, i, d, d, I, LL, D, D, D, D, D, D]
        L.oracle_advect_markers.argtypes = [i, i, d, d, I, LL, D, D, D, D, d, i, PL]
        L.oracle_marker_timestep.argtypes = [i, i, d, d, D, D, d, d, D]
        L.oracle_gcr_dense.argtypes = [i, D, D, D, D, i, i, i, d, I, D, D, i, D]
        L.oracle_aa_alpha.argtypes = [i, D, D]
    return _lib


def default_opts(**kw):
    o = Opts()
    lib().oracle_opts_default(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous float64"
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: {lib().oracle_strerror(code).decode()} ({code})")
        self.code = code


def _check(code, what):
    if code < 0:
        raise OracleError(code, what)
    return code


class Oracle:
    """Same calls as the C-ABI (stokes_*), on host numpy arrays."""

    TYPES = {"vx": 0, "vy": 1, "p": 2, "b": 3}

    def __init__(self, nx, ny, Lx=1.0, Ly=1.0, bc=(0, 0, 0, 0), **opts):
        self.nx, self.ny, self.Lx, self.Ly = nx, ny, Lx, Ly
        self.opts = default_opts(**opts)
        self._h = ctypes.c_void_p()
        bcs = (ctypes.c_int * 4)(*bc)
        _check(lib().oracle_create(nx, ny, Lx, Ly, bcs, ctypes.byref(self.opts), ctypes.byref(self._h)), "create")

    def close(self):
        if self._h:
            lib().oracle_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # shapes -----------------------------------------------------------
    @property
    def nlev(self):
        return lib().oracle_num_levels(self._h)

    def level_shape(self, l):
        a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().oracle_level_shape(self._h, l, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "level")
        return a.value, b.value, c.value

    @staticmethod
    def shapes(nx, ny):
        return {"vx": (ny, nx + 1), "vy": (ny + 1, nx), "p": (ny, nx), "b": (ny + 1, nx + 1)}

    def zeros(self, kind, level=0):
        nx, ny, _ = self.level_shape(level)
        return np.zeros(self.shapes(nx, ny)[kind])

    # setup ------------------------------------------------------------
    def set_viscosity(self, eta_b, eta_p):
        self._eta = (np.ascontiguousarray(eta_b, np.float64), np.ascontiguousarray(eta_p, np.float64))
        _check(lib().oracle_set_viscosity(self._h, _d(self._eta[0]), _d(self._eta[1])), "set_viscosity")

    def set_density(self, rho_b):
        r = np.ascontiguousarray(rho_b, np.float64)
        _check(lib().oracle_set_density(self._h, _d(r)), "set_density")

    def set_gravity(self, gx, gy):
        _check(lib().oracle_set_gravity(self._h, gx, gy), "set_gravity")

    def set_force(self, fx, fy):
        fx = np.ascontiguousarray(fx, np.float64)
        fy = np.ascontiguousarray(fy, np.float64)
        _check(lib().oracle_set_force(self._h, _d(fx), _d(fy)), "set_force")

    def get_viscosity(self, level):
        eb, ep = self.zeros("b", level), self.zeros("p", level)
        _check(lib().oracle_get_viscosity(self._h, level, _d(eb), _d(ep)), "get_viscosity")
        return eb, ep

    def blend_viscosity(self, theta):
        """test hook: computational viscosity (1 - theta) eta_min + theta eta"""
        _check(lib().oracle_blend_viscosity(self._h, ctypes.c_double(theta)), "blend_viscosity")

    def lithostatic(self):
        """p_litho = int_0^y rho g_y dy' at the P nodes, P layout"""
        p = self.zeros("p")
        _check(lib().oracle_lithostatic(self._h, _d(p)), "lithostatic")
        return p

    # operators ----------------------------------------------------------
    def apply_operator(self, vx, vy, p):
        ax, ay, ap = self.zeros("vx"), self.zeros("vy"), self.zeros("p")
        vx, vy, p = (np.ascontiguousarray(a, np.float64) for a in (vx, vy, p))
        _check(lib().oracle_apply_operator(self._h, _d(vx), _d(vy), _d(p), _d(ax), _d(ay), _d(ap)), "apply")
        return ax, ay, ap

    def residual(self, vx, vy, p):
        rx, ry, rp = self.zeros("vx"), self.zeros("vy"), self.zeros("p")
        e = ctypes.c_double()
        vx, vy, p = (np.ascontiguousarray(a, np.float64) for a in (vx, vy, p))
        _check(lib().oracle_residual(self._h, _d(vx), _d(vy), _d(p), _d(rx), _d(ry), _d(rp), ctypes.byref(e)),
               "residual")
        return rx, ry, rp, e.value

    def residual_ld(self, vx, vy, p):
        """The residual and E of residual() evaluated in long double (verification of E near
        convergence at large sizes, reading R34); arrays rounded to FP64."""
        rx, ry, rp = self.zeros("vx"), self.zeros("vy"), self.zeros("p")
        e = ctypes.c_double()
        vx, vy, p = (np.ascontiguousarray(a, np.float64) for a in (vx, vy, p))
        _check(lib().oracle_residual_ld(self._h, _d(vx), _d(vy), _d(p), _d(rx), _d(ry), _d(rp), ctypes.byref(e)),
               "residual_ld")
        return rx, ry, rp, e.value

    def energy_sums(self, vx, vy, p):
        s = np.zeros(3)
        vx, vy, p = (np.ascontiguousarray(a, np.float64) for a in (vx, vy, p))
        _check(lib().oracle_energy_sums(self._h, _d(vx), _d(vy), _d(p), _d(s)), "energy_sums")
        return s

    def vcycle(self, bx, by, vx, vy):
        vx = np.array(vx, np.float64, order="C")
        vy = np.array(vy, np.float64, order="C")
        bx, by = np.ascontiguousarray(bx, np.float64), np.ascontiguousarray(by, np.float64)
        _check(lib().oracle_vcycle(self._h, _d(bx), _d(by), _d(vx), _d(vy)), "vcycle")
        return vx, vy

    def smooth(self, level, bx, by, vx, vy, nsweeps):
        vx = np.array(vx, np.float64, order="C")
        vy = np.array(vy, np.float64, order="C")
        bx, by = np.ascontiguousarray(bx, np.float64), np.ascontiguousarray(by, np.float64)
        _check(lib().oracle_smooth(self._h, level, _d(bx), _d(by), _d(vx), _d(vy), nsweeps), "smooth")
        return vx, vy

    def level_residual(self, level, bx, by, vx, vy):
        rx, ry = self.zeros("vx", level), self.zeros("vy", level)
        args = [np.ascontiguousarray(a, np.float64) for a in (bx, by, vx, vy)]
        _check(lib().oracle_level_residual(self._h, level, *[_d(a) for a in args], _d(rx), _d(ry)), "lres")
        return rx, ry

    def restrict(self, level, kind, fine):
        coarse = self.zeros(kind, level + 1)
        fine = np.ascontiguousarray(fine, np.float64)
        _check(lib().oracle_restrict(self._h, level, self.TYPES[kind], _d(fine), _d(coarse)), "restrict")
        return coarse

    def prolong(self, level, ex, ey, vx, vy):
        vx = np.array(vx, np.float64, order="C")
        vy = np.array(vy, np.float64, order="C")
        ex, ey = np.ascontiguousarray(ex, np.float64), np.ascontiguousarray(ey, np.float64)
        _check(lib().oracle_prolong(self._h, level, _d(ex), _d(ey), _d(vx), _d(vy)), "prolong")
        return vx, vy

    def coarse_solve(self, bx, by):
        l = self.nlev - 1
        vx, vy = self.zeros("vx", l), self.zeros("vy", l)
        bx, by = np.ascontiguousarray(bx, np.float64), np.ascontiguousarray(by, np.float64)
        _check(lib().oracle_coarse_solve(self._h, _d(bx), _d(by), _d(vx), _d(vy)), "coarse_solve")
        return vx, vy

    def solve(self, rtol, vx=None, vy=None, p=None, hist_len=0):
        vx = self.zeros("vx") if vx is None else np.array(vx, np.float64, order="C")
        vy = self.zeros("vy") if vy is None else np.array(vy, np.float64, order="C")
        p = self.zeros("p") if p is None else np.array(p, np.float64, order="C")
        it, e = ctypes.c_int(), ctypes.c_double()
        hist = np.full(max(hist_len, 1), np.nan)
        st = lib().oracle_solve_hist(self._h, rtol, _d(vx), _d(vy), _d(p), ctypes.byref(it),
                                     ctypes.byref(e), _d(hist), hist_len)
        if st < 0 and st != EDIVERGED:
            _check(st, "solve")
        out = {"vx": vx, "vy": vy, "p": p, "iters": it.value, "E": e.value, "status": st}
        if hist_len:
            out["hist"] = hist[: min(it.value, hist_len)]
        return out


# ---------------------------------------------------------------- Krylov / Anderson cores on dense data
def gcr_dense(A, Minv, b, x0, m, max_iter, rtol=0.0, true_restart=1, hist_len=0):
    """The oracle's GCR(m) code (gcr_core, Alg. 4) on a dense system A x = b with explicit
    preconditioner Minv.  Returns dict(x, iters, E, status, W[, hist]); W = the normalised
    w_i of the last cycle (m x n)."""
    A, Minv, b = (np.ascontiguousarray(a, np.float64) for a in (A, Minv, b))
    n = b.size
    x = np.array(x0, np.float64, order="C")
    W = np.zeros((m, n))
    it, e = ctypes.c_int(), ctypes.c_double()
    hist = np.full(max(hist_len, 1), np.nan)
    st = lib().oracle_gcr_dense(n, _d(A), _d(Minv), _d(b), _d(x), m, max_iter, true_restart, rtol,
                                ctypes.byref(it), ctypes.byref(e), _d(hist), hist_len, _d(W))
    if st < 0 and st != EDIVERGED:
        _check(st, "gcr_dense")
    out = {"x": x, "iters": it.value, "E": e.value, "status": st, "W": W}
    if hist_len:
        out["hist"] = hist[: min(it.value, hist_len)]
    return out


def aa_alpha(H):
    """The oracle's Alg. 5 argmin (solve_anderson's aa_alpha) for the Gram matrix H = R^T R."""
    H = np.ascontiguousarray(H, np.float64)
    n = H.shape[0]
    a = np.zeros(n)
    _check(lib().oracle_aa_alpha(n, _d(H), _d(a)), "aa_alpha")
    return a


# ---------------------------------------------------------------- marker-in-cell (NEXT-4)
SCHEMES = {"euler": 0, "heun": 1, "rk4": 2, "lpi2": 3, "lpi3": 4}


def _bc(bc):
    return (ctypes.c_int * 4)(*bc)


def markers_to_grid(nx, ny, Lx, Ly, xm, ym, eta_m, rho_m):
    """PAPER.md:467-495 (R28): returns eta_b, eta_p, rho_b (user layout) and the number of
    empty nodes (zero accumulated weight; written 0)."""
    xm, ym, eta_m, rho_m = (np.ascontiguousarray(a, np.float64) for a in (xm, ym, eta_m, rho_m))
    eta_b = np.zeros((ny + 1, nx + 1))
    rho_b = np.zeros((ny + 1, nx + 1))
    eta_p = np.zeros((ny, nx))
    ne = ctypes.c_longlong()
    _check(lib().oracle_markers_to_grid(nx, ny, Lx, Ly, len(xm), _d(xm), _d(ym), _d(eta_m), _d(rho_m),
                                        _d(eta_b), _d(eta_p), _d(rho_b), ctypes.byref(ne)), "markers_to_grid")
    return eta_b, eta_p, rho_b, ne.value


def grid_to_markers(nx, ny, Lx, Ly, bc, xm, ym, vx, vy):
    """PAPER.md:497-511 (R29): velocity interpolated to the markers."""
    xm, ym, vx, vy = (np.ascontiguousarray(a, np.float64) for a in (xm, ym, vx, vy))
    um, vm = np.zeros_like(xm), np.zeros_like(xm)
    _check(lib().oracle_grid_to_markers(nx, ny, Lx, Ly, _bc(bc), len(xm), _d(xm), _d(ym), _d(vx), _d(vy),
                                        _d(um), _d(vm)), "grid_to_markers")
    return um, vm


def advect_markers(nx, ny, Lx, Ly, bc, xm, ym, vx, vy, dt, scheme="rk4"):
    """PAPER.md:560-578 (R30): one advection step; returns new (xm, ym) and the number of
    markers whose final position was clamped into the box."""
    xm, ym = np.array(xm, np.float64, order="C"), np.array(ym, np.float64, order="C")
    vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
    nc = ctypes.c_longlong()
    _check(lib().oracle_advect_markers(nx, ny, Lx, Ly, _bc(bc), len(xm), _d(xm), _d(ym), _d(vx), _d(vy),
                                       float(dt), SCHEMES[scheme], ctypes.byref(nc)), "advect_markers")
    return xm, ym, nc.value


def marker_timestep(nx, ny, Lx, Ly, vx, vy, cfl, max_dt):
    """R31: dt = min(max_dt, cfl min(dx/max|vx|, dy/max|vy|))."""
    vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
    dt = ctypes.c_double()
    _check(lib().oracle_marker_timestep(nx, ny, Lx, Ly, _d(vx), _d(vy), cfl, max_dt, ctypes.byref(dt)),
           "marker_timestep")
    return dt.value
